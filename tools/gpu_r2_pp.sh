timeout 600 python -m pytest tests -m gpu -q --timeout 200 -x 2>&1 | tail -4 | tee gpurun_out/r2_pytest_gpu.log
for lib in libqflash.so libqflash_nopp.so; do
  QFLASH_LIB=$lib timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/pp_l14_$lib.log
  QFLASH_LIB=$lib timeout 300 python bench.py --workload A4 --batch 8 --steps 2000 --no-cpu-baseline --no-e2e --no-extra 2>&1 | tail -1 > gpurun_out/pp_a4_$lib.log
done
timeout 200 python tools/timeline_gpu.py 2>&1 > gpurun_out/r2_timeline.txt
