timeout 300 python -m pytest tests -m gpu -q -x --timeout 60 2>&1 | tail -2 | tee gpurun_out/pytest.log
for pdl in 15 7; do
  QFLASH_PDL=$pdl timeout 120 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_a3_pdl$pdl.log
  QFLASH_PDL=$pdl timeout 120 python bench.py --workload A1 --batch 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_a1_pdl$pdl.log
  QFLASH_PDL=$pdl timeout 120 python bench.py --workload A4 --batch 8 --steps 2000 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_a4_pdl$pdl.log
done
