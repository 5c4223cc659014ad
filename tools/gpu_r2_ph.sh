timeout 600 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -3 | tee gpurun_out/r2_pytest_gpu.log
timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --scales per-head 2>&1 | tail -1 > gpurun_out/ph_l14.log
timeout 200 python bench.py --workload A3 --batch 8 --steps 2000 --no-cpu-baseline --scales per-head 2>&1 | tail -1 > gpurun_out/ph_a3.log
timeout 200 python tools/timeline_gpu.py > gpurun_out/r2_timeline.txt 2>&1
