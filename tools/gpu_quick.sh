timeout 120 python bench.py --scales per-head --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_a3_ph.log
timeout 120 python bench.py --scales per-head --workload A4 --batch 8 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_a4_ph.log
timeout 120 python bench.py --scales per-head --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_l14_ph.log
