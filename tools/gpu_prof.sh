# ncu: launch list of the default bench (fused step), full capture of the fused step kernel (A3 b8),
# of the two-launch attention kernel (A3 b8) and of L14's attention kernel.
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fused.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_two.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --mode two > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:qflash_attn -s 6 -c 1 -o gpurun_out/prof_fused_a3b8 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:qflash_attn -s 6 -c 1 -o gpurun_out/prof_attn2_a3b8 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --mode two > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:qflash_attn -s 2 -c 1 -o gpurun_out/prof_attn2_l14 python bench.py --workload L14 --batch 64 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --mode two > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
