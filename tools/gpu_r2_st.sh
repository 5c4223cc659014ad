timeout 600 python -m pytest tests -m gpu -q --timeout 200 2>&1 | tail -6 | tee gpurun_out/r2_pytest_gpu.log
timeout 300 python -m pytest tests -m gpu -q --timeout 200 -k accumulation 2>&1 | grep -E "assert|Error|passed|failed" | head -20 > gpurun_out/r2_acc_fail.log
for lib in libqflash.so libqflash_st2.so libqflash_sp64.so; do
  QFLASH_LIB=$lib timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/st_l14_$lib.log
done
timeout 200 python tools/timeline_gpu.py 2>&1 > gpurun_out/r2_timeline.txt
