timeout 300 python -m pytest tests -m gpu -q -x --timeout 60 2>&1 | tail -2 | tee gpurun_out/pytest.log
for own in 1 0; do
  QFLASH_FUSED_OWN=$own timeout 120 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_a3_own$own.log
  QFLASH_FUSED_OWN=$own timeout 120 python bench.py --workload A1 --batch 1 --steps 2000 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_a1_own$own.log
done
