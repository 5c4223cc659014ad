# Launch list + one full ncu capture of the attention kernel (A3 b8) and L14.
set -x
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 2000 2>&1 | tail -1 | tee gpurun_out/bench_default.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_stdout.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qflash_attn -s 6 -c 1 -o gpurun_out/prof_attn_a3b8 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_stdout.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qflash_attn -s 2 -c 1 -o gpurun_out/prof_attn_l14 python bench.py --workload L14 --batch 64 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_l14_stdout.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:quantize_kernel -s 6 -c 1 -o gpurun_out/prof_quant_a3b8 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_q_stdout.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:amax_kernel -s 6 -c 1 -o gpurun_out/prof_amax_a3b8 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_a_stdout.log 2>&1
