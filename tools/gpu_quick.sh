# Quick GPU iteration: parity tests (both kernel configurations), timeline, benches.
set -x
for c in 0 1; do
  QFLASH_ATTN_CFG=$c timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 | tee gpurun_out/pytest_cfg$c.log
done
for m in fused two three; do
  timeout 300 python bench.py --no-cpu-baseline --mode $m 2>&1 | tail -1 | tee gpurun_out/bench_a3_$m.log
done
timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | tee gpurun_out/bench_l14.log
for m in fused two; do
timeout 300 python bench.py --workload A4 --batch 8 --steps 2000 --no-cpu-baseline --no-e2e --mode $m 2>&1 | tail -1 | tee gpurun_out/bench_a4_$m.log
done
timeout 300 python bench.py --workload A1 --batch 1 --steps 2000 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | tee gpurun_out/bench_a1.log
