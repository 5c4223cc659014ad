set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest.log
QFLASH_LIB=libqflash_fqt.so timeout 300 python tools/fq_timing.py 2>&1 | tee gpurun_out/fq_timing.txt
for m in fused two; do
  timeout 300 python bench.py --no-cpu-baseline --mode $m 2>&1 | tail -1 | tee gpurun_out/bench_a3_$m.log
  timeout 300 python bench.py --workload A4 --batch 8 --steps 2000 --no-cpu-baseline --no-e2e --mode $m 2>&1 | tail -1 | tee gpurun_out/bench_a4_$m.log
  timeout 300 python bench.py --workload A1 --batch 1 --steps 2000 --no-cpu-baseline --no-e2e --mode $m 2>&1 | tail -1 | tee gpurun_out/bench_a1_$m.log
done
