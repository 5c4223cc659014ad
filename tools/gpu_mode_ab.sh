# A/B of the attention kernel modes (QFLASH_ATTN_MODE 0: 1 CTA/SM x 4 softmax WGs; 1: 2 CTAs/SM x 2 WGs)
set -x
QFLASH_ATTN_MODE=1 timeout 900 python -m pytest tests -m gpu -q -x -k "edge or workload or adversarial or full_size" 2>&1 | tail -3
timeout 300 python tests/timeline_gpu.py 2>&1 | tee gpurun_out/timeline.log
for n in 0 1; do
  QFLASH_ATTN_MODE=$n timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 2000 2>&1 | tail -1 > gpurun_out/bench_a3_m$n.log
  QFLASH_ATTN_MODE=$n timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_l14_m$n.log
  QFLASH_ATTN_MODE=$n timeout 300 python bench.py --workload A4 --no-cpu-baseline --no-e2e --steps 2000 2>&1 | tail -1 > gpurun_out/bench_a4_m$n.log
done
QFLASH_ATTN_MODE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:qflash_attn -s 2 -c 1 -o gpurun_out/prof_attn_l14_m1 python bench.py --workload L14 --batch 64 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
