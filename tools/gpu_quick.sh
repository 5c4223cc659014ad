for wl in "A1 1" "A3 8" "A1 1" "A3 8"; do
  set -- $wl
  timeout 120 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --no-e2e 2>&1 | tail -1 >> gpurun_out/bench_chk_$1.log
done
QFLASH_FUSED_CLUSTER=0 timeout 120 python bench.py --workload A1 --batch 1 --steps 2000 --no-cpu-baseline --no-e2e 2>&1 | tail -1 >> gpurun_out/bench_chk_A1nocl.log
