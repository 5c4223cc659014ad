export QFLASH_LIB=libqflash_smr.so
timeout 120 python -m pytest tests/test_gpu_parity.py -q -x --timeout 60 -k "workload or full_size or edge" 2>&1 | tail -1 | tee gpurun_out/smr_tests.log
QFLASH_ATTN_CFG=1 timeout 120 python -m pytest tests/test_gpu_parity.py -q -x --timeout 60 -k "workload or edge" 2>&1 | tail -1 | tee -a gpurun_out/smr_tests.log
timeout 90 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --mode two 2>&1 | tail -1 > gpurun_out/bench_smr_l14.log
timeout 90 python bench.py --no-cpu-baseline --no-e2e --mode two 2>&1 | tail -1 > gpurun_out/bench_smr_a3.log
unset QFLASH_LIB
timeout 90 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --mode two 2>&1 | tail -1 > gpurun_out/bench_base_l14.log
timeout 90 python bench.py --no-cpu-baseline --no-e2e --mode two 2>&1 | tail -1 > gpurun_out/bench_base_a3.log
