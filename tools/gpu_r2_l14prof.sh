mkdir -p gpurun_out/prof
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2 > gpurun_out/l14p_pytest.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qflash_attn -s 2 -c 1 -o gpurun_out/prof/r2b_attn_l14 python bench.py --workload L14 --batch 64 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --mode three --no-extra --no-table1 > gpurun_out/prof/ncu_l14.log 2>&1
ncu -i gpurun_out/prof/r2b_attn_l14.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/r2b_attn_l14.sass.csv 2>/dev/null
ncu -i gpurun_out/prof/r2b_attn_l14.ncu-rep --page raw --csv > gpurun_out/prof/r2b_attn_l14.raw.csv 2>/dev/null
rm -f gpurun_out/prof/r2b_attn_l14.ncu-rep
