# quick iteration: parity tests, timeline, default bench, A1 b1 / A4 b8 benches
timeout 600 python -m pytest tests -m gpu -q --timeout 200 -x 2>&1 | tail -4 | tee gpurun_out/r2_pytest_gpu.log
timeout 200 python tools/timeline_gpu.py 2>&1 | head -40 > gpurun_out/r2_timeline.txt
timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2_bench_a3.log
timeout 120 python bench.py --workload A1 --batch 1 --steps 2000 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/r2_bench_a1b1.log
timeout 120 python bench.py --workload A2 --batch 8 --steps 2000 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/r2_bench_a2b8.log
QFLASH_LIB=libqflash_fqt.so timeout 200 python tools/fq_timing_graph.py 2>&1 | tail -12 > gpurun_out/r2_fq_timeline.txt
