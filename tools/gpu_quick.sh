# Quick GPU iteration: parity tests, timeline, bench (A3 b8, L14 b64, A4 b8).
set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log
timeout 300 python tests/timeline_gpu.py 2>&1 | tee gpurun_out/timeline.log
timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_default.log
timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | tee gpurun_out/bench_l14.log
timeout 300 python bench.py --workload A4 --batch 8 --steps 2000 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | tee gpurun_out/bench_a4.log
