# Bench sweep over the paper's Table 1 workloads (A1-A7) and Swin-B stages at batch 1 and 8,
# plus L14 b64: one bench.py line each (fused one-launch step, cold rotating inputs).
rm -f gpurun_out/sweep_*.json
for wl in A1 A2 A3 A4 A5 A6 A7 SwinB-s1 SwinB-s2 SwinB-s3 SwinB-s4; do
  for b in 1 8; do
    timeout 120 python bench.py --workload $wl --batch $b --steps 2000 --warmup 50 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/sweep_${wl}_b$b.json
  done
done
timeout 200 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/sweep_L14_b64.json
timeout 200 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --mode two 2>&1 | tail -1 > gpurun_out/sweep_L14_b64_two.json
timeout 300 python bench.py 2>&1 | tail -1 > gpurun_out/r2_bench_default_final.json
