./tools/derive_bench | tee gpurun_out/derive.txt
timeout 400 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -2 | tee gpurun_out/pytest.log
timeout 120 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_a3.log
