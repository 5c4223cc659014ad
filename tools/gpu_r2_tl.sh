timeout 600 python -m pytest tests -m gpu -q --timeout 200 2>&1 | tail -4 | tee gpurun_out/r2_pytest_gpu.log
timeout 200 python tools/timeline_gpu.py 2>&1 | tee gpurun_out/r2_timeline.txt
