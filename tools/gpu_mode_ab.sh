set -x
QFLASH_ATTN_MODE=2 timeout 900 python -m pytest tests -m gpu -q -x -k "edge or workload or adversarial or full_size" 2>&1 | tail -3
for n in 0 2; do
  QFLASH_ATTN_MODE=$n timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 2000 2>&1 | tail -1 > gpurun_out/bench_a3_m$n.log
  QFLASH_ATTN_MODE=$n timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_l14_m$n.log
done
for n in 1 2; do
  QFLASH_ATTN_MODE=$n timeout 300 python bench.py --workload A4 --no-cpu-baseline --no-e2e --steps 2000 2>&1 | tail -1 > gpurun_out/bench_a4_m$n.log
done
