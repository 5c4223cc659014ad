export QFLASH_QUANT_FUSED=0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quantize_kernel -s 6 -c 1 -o gpurun_out/prof_quant python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dequantize -s 6 -c 1 -o gpurun_out/prof_dequant python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:amax_kernel -s 6 -c 1 -o gpurun_out/prof_amax python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
