# quick iteration: parity tests, default bench, A1 b1 / A2 b8 / A4 b8 benches, fused timeline
timeout 600 python -m pytest tests -m gpu -q --timeout 200 -x 2>&1 | tail -4 | tee gpurun_out/r2_pytest_gpu.log
for wl in "A3 8" "A1 1" "A2 8" "A4 8"; do set -- $wl
  timeout 120 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --no-e2e --no-extra 2>&1 | tail -1 > gpurun_out/r2_bench_$1b$2.log
  QFLASH_STAGE=0 timeout 120 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --no-e2e --no-extra 2>&1 | tail -1 > gpurun_out/r2_bench_$1b$2_nostage.log
done
QFLASH_LIB=libqflash_fqt.so timeout 200 python tools/fq_timing_graph.py 2>&1 | tail -12 > gpurun_out/r2_fq_timeline.txt
