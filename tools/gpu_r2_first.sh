nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python -m pytest tests -m gpu -q --timeout 200 -x 2>&1 | tail -5 | tee gpurun_out/r2_pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/r2_smoke.log
timeout 300 python bench.py 2>&1 | tail -1 > gpurun_out/r2_bench_default.log
lscpu | head -20 > gpurun_out/r2_lscpu.txt
