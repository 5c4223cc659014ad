QFLASH_ATTN_CFG=2 timeout 240 python -m pytest tests -m gpu -q -x --timeout 60 2>&1 | tail -2 | tee gpurun_out/pytest_cfg2.log
for lib in libqflash.so libqflash_s32.so; do
for c in 0 1 2; do
  QFLASH_LIB=$lib QFLASH_ATTN_CFG=$c timeout 60 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --mode two 2>&1 | tail -1 > gpurun_out/bench_l14_c${c}_$lib.log
  QFLASH_LIB=$lib QFLASH_ATTN_CFG=$c timeout 60 python bench.py --no-cpu-baseline --no-e2e --steps 2000 --mode two 2>&1 | tail -1 > gpurun_out/bench_a3_c${c}_$lib.log
  QFLASH_LIB=$lib QFLASH_ATTN_CFG=$c timeout 60 python bench.py --workload A4 --no-cpu-baseline --no-e2e --steps 2000 --mode two 2>&1 | tail -1 > gpurun_out/bench_a4_c${c}_$lib.log
done; done
