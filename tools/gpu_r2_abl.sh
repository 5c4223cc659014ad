timeout 600 python -m pytest tests -m gpu -q --timeout 200 2>&1 | tail -4 | tee gpurun_out/r2_pytest_gpu.log
timeout 600 python tools/ablation.py > gpurun_out/r2_ablation.log 2>&1
cp profiles/r2_ablation.md gpurun_out/ 2>/dev/null
