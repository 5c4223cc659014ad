timeout 600 python -m pytest tests -m gpu -q --timeout 200 -x 2>&1 | tail -3 | tee gpurun_out/r2_pytest_gpu.log
for lib in libqflash.so libqflash_oldsleep.so; do
  for wl in "A3 8" "A1 1" "A4 8" "SwinB-s1 8"; do set -- $wl
    QFLASH_LIB=$lib timeout 120 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --no-e2e --no-extra 2>&1 | tail -1 > gpurun_out/sl_$1b$2_$lib.log
  done
  QFLASH_LIB=$lib timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/sl_L14_$lib.log
done
