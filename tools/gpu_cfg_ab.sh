# Parity for both attention kernel configurations, then A/B bench (cfg 0: CS4 x QT1, cfg 1: CS2 x QT2).
set -x
for c in 0 1; do
  QFLASH_ATTN_CFG=$c timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 | tee gpurun_out/pytest_cfg$c.log
done
timeout 300 python tests/timeline_gpu.py 2>&1 | tee gpurun_out/timeline.log
for c in 0 1; do
  QFLASH_ATTN_CFG=$c timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 2000 2>&1 | tail -1 > gpurun_out/bench_a3_c$c.log
  QFLASH_ATTN_CFG=$c timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_l14_c$c.log
  QFLASH_ATTN_CFG=$c timeout 300 python bench.py --workload A4 --no-cpu-baseline --no-e2e --steps 2000 2>&1 | tail -1 > gpurun_out/bench_a4_c$c.log
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qflash_attn -s 2 -c 1 -o gpurun_out/prof_attn_l14_new python bench.py --workload L14 --batch 64 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
