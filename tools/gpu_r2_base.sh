# Round-2 re-entry baseline: GPU suite, default bench line, timelines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -3 | tee gpurun_out/base_pytest_gpu.log
timeout 400 python bench.py > gpurun_out/base_bench.log 2>&1
for wl in "A3 8" "A1 1" "A4 8" "A2 8"; do set -- $wl
  timeout 200 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --no-e2e --no-extra 2>&1 | tail -1 > gpurun_out/base_$1b$2.log
done
timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-extra 2>&1 | tail -1 > gpurun_out/base_L14b64.log
timeout 200 python tools/timeline_gpu.py > gpurun_out/base_timeline.txt 2>&1
timeout 200 python tools/fq_timing_graph.py > gpurun_out/base_fq_timeline.txt 2>&1
