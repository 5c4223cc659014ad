# One measurement session: parity tests, smoke, benches (default line with cpu_baseline,
# other BASELINE configs), ncu launch list of the default bench command.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 300 python -m pytest tests -m gpu -q --timeout 120 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.log
timeout 300 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.log
timeout 120 python bench.py --workload A1 --batch 1 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_a1b1.log
timeout 120 python bench.py --workload A4 --batch 8 --steps 2000 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_a4b8.log
timeout 120 python bench.py --workload A4 --batch 8 --steps 2000 --no-cpu-baseline --no-e2e --mode two 2>&1 | tail -1 > gpurun_out/bench_a4b8_two.log
timeout 120 python bench.py --workload SwinB-s1 --batch 8 --steps 2000 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_swinb1b8.log
timeout 200 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_l14b64.log
timeout 200 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --mode two 2>&1 | tail -1 > gpurun_out/bench_l14b64_two.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
