# measured roofline denominators + the new bench line (default and L14)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
./tools/peaks_bench > gpurun_out/r2_peaks.json 2> gpurun_out/r2_peaks.err
cat gpurun_out/r2_peaks.json
cp gpurun_out/r2_peaks.json profiles/r2_peaks.json
timeout 400 python bench.py 2>&1 | tail -1 > gpurun_out/r2_bench_default.log
timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2_bench_l14.log
timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --scaling strong 2>&1 | tail -1 > gpurun_out/r2_bench_l14_strong1.log
tail -c 300 gpurun_out/r2_bench_default.log
