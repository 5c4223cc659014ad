mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -3 > gpurun_out/ch_pytest.log
timeout 600 python bench.py > gpurun_out/ch_bench.log 2>&1
timeout 300 python bench.py --workload L14 --batch 64 --steps 24 --warmup 3 --no-cpu-baseline --no-e2e --no-table1 2>&1 | tail -1 > gpurun_out/ch_L14.log
timeout 200 python tools/timeline_gpu.py > gpurun_out/ch_timeline.txt 2>&1
