timeout 300 python -m pytest tests -m gpu -q -x --timeout 60 2>&1 | tail -2 | tee gpurun_out/pytest.log
timeout 200 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.log
timeout 120 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --mode two 2>&1 | tail -1 > gpurun_out/bench_l14_two.log
