# One GPU session: parity tests, smoke, bench, ncu launch list + full capture.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 | tee gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke.log
timeout 300 python bench.py 2>&1 | tail -3 | tee gpurun_out/bench_default.log
timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -2 | tee gpurun_out/bench_l14.log
timeout 300 python bench.py --workload A4 --batch 8 --steps 2000 --no-cpu-baseline 2>&1 | tail -2 | tee gpurun_out/bench_a4.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_stdout.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qflash_attn -s 6 -c 1 -o gpurun_out/prof_attn_a3b8 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_stdout.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qflash_attn -s 2 -c 1 -o gpurun_out/prof_attn_l14 python bench.py --workload L14 --batch 64 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_l14_stdout.log 2>&1
ls -la gpurun_out
