# r2 ncu evidence: launch list of the default bench command, full captures of the fused A3 b8
# step kernel and of the L14 b64 attention kernel (int8 in), source pages for SASS histograms
mkdir -p gpurun_out/prof
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/r2_launches_default.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:qflash_attn -s 6 -c 1 -o gpurun_out/prof/r2_fused_a3b8 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qflash_attn -s 2 -c 1 -o gpurun_out/prof/r2_attn_l14 python bench.py --workload L14 --batch 64 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --mode three --no-extra > /dev/null 2>&1
for r in r2_fused_a3b8 r2_attn_l14; do
  ncu -i gpurun_out/prof/$r.ncu-rep --page raw --csv > gpurun_out/prof/$r.raw.csv 2>/dev/null
  ncu -i gpurun_out/prof/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/$r.sass.csv 2>/dev/null
  ncu -i gpurun_out/prof/$r.ncu-rep --page details --csv > gpurun_out/prof/$r.details.csv 2>/dev/null
done
ls -la gpurun_out/prof
