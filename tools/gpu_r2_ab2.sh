timeout 600 python -m pytest tests -m gpu -q --timeout 200 2>&1 | tail -4 | tee gpurun_out/r2_pytest_gpu.log
for lib in libqflash.so libqflash_spin.so; do
  for wl in "A3 8" "A1 1" "A4 8"; do set -- $wl
    QFLASH_LIB=$lib timeout 120 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --no-e2e --no-extra 2>&1 | tail -1 > gpurun_out/ab2_$1b$2_$lib.log
  done
  QFLASH_LIB=$lib timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-extra 2>&1 | tail -1 > gpurun_out/ab2_L14_$lib.log
done
QFLASH_LIB=libqflash_fqt.so timeout 200 python tools/fq_timing_graph.py 2>&1 | tail -12 > gpurun_out/r2_fq_timeline.txt
timeout 600 python tools/tile_sqnr_sweep.py > gpurun_out/r2_tile_sqnr.log 2>&1
cp profiles/r2_tile_sqnr.md gpurun_out/ 2>/dev/null
