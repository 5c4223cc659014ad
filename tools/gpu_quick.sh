QFLASH_ATTN_CFG=1 timeout 400 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -2 | tee -a gpurun_out/pytest.log
timeout 400 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -2 | tee -a gpurun_out/pytest.log
for v in generic packed; do
  timeout 120 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --mode two --variant $v 2>&1 | tail -1 > gpurun_out/bench_l14_$v.log
done
