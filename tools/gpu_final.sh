bash tools/sweep.sh
timeout 300 ncu --set full --clock-control none --import-source on -k regex:qflash_attn -s 2 -c 1 -o gpurun_out/prof_l14_final python bench.py --workload L14 --batch 64 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --mode two > /dev/null 2>&1
