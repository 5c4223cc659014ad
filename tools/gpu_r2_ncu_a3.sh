# full ncu capture of the fused A3 b8 step (per-PC stall sampling: where no_instructions lands)
mkdir -p gpurun_out/prof
timeout 400 ncu --set full --clock-control none --import-source on -k regex:qflash_attn -s 6 -c 1 -o gpurun_out/prof/r2b_fused_a3b8 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-extra --no-table1 > gpurun_out/prof/ncu_a3.log 2>&1
ncu -i gpurun_out/prof/r2b_fused_a3b8.ncu-rep --page raw --csv > gpurun_out/prof/r2b_fused_a3b8.raw.csv 2>/dev/null
ncu -i gpurun_out/prof/r2b_fused_a3b8.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/r2b_fused_a3b8.sass.csv 2>/dev/null
ncu -i gpurun_out/prof/r2b_fused_a3b8.ncu-rep --page details --csv > gpurun_out/prof/r2b_fused_a3b8.details.csv 2>/dev/null
ls -la gpurun_out/prof
