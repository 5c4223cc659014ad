for c in 0 1; do QFLASH_ATTN_CFG=$c timeout 400 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -2 | tee -a gpurun_out/pytest.log; done
timeout 120 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --mode two 2>&1 | tail -1 > gpurun_out/bench_qb_l14.log
timeout 120 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_qb_a3.log
timeout 120 python bench.py --workload A4 --batch 8 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_qb_a4.log
timeout 120 python bench.py --no-cpu-baseline --no-e2e --mode two 2>&1 | tail -1 > gpurun_out/bench_qb_a3two.log
