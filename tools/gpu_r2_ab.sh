# A/B: L1 no-allocate amax loads; L14 DBG timeline with producer / MMA stamps
for wl in "A3 8" "A1 1" "A4 8"; do set -- $wl
  timeout 120 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --no-e2e --no-extra 2>&1 | tail -1 > gpurun_out/ab_$1b$2_base.log
  QFLASH_LIB=libqflash_na.so timeout 120 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --no-e2e --no-extra 2>&1 | tail -1 > gpurun_out/ab_$1b$2_na.log
done
QFLASH_LIB=libqflash_fqt.so timeout 200 python tools/fq_timing_graph.py 2>&1 | tail -12 > gpurun_out/ab_fq_base.txt
QFLASH_LIB=libqflash_fqtna.so timeout 200 python tools/fq_timing_graph.py 2>&1 | tail -12 > gpurun_out/ab_fq_na.txt
timeout 200 python tools/timeline_gpu.py 2>&1 > gpurun_out/r2_timeline.txt
