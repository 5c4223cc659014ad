# A/B of library variants (QFLASH_LIB) on L14 b64 (attention with fused DQ, two-launch mode) and A3 b8
for v in v00 v01 v10 v11; do
  QFLASH_LIB=libqflash_$v.so timeout 120 python -m pytest tests/test_gpu_parity.py -q -x --timeout 60 -k "workload or full_size or edge" 2>&1 | tail -1 | sed "s/^/$v /" >> gpurun_out/var_tests.log
  QFLASH_LIB=libqflash_$v.so timeout 60 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --mode two 2>&1 | tail -1 > gpurun_out/bench_l14_$v.log
  QFLASH_LIB=libqflash_$v.so timeout 60 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_a3_$v.log
done
