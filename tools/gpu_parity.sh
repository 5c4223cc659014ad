# GPU parity run (fast fail) + graph A/B timing.
set -x
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.log
rm -f gpurun_out/graph_ab.log
for wl in "A3 --batch 8" "A4 --batch 8" "A1 --batch 1" "L14 --batch 64 --steps 30"; do
  timeout 300 python tools/graph_ab.py --workload $wl 2>&1 | grep graph | tee -a gpurun_out/graph_ab.log
done
timeout 300 python tests/timeline_gpu.py 2>&1 | tee gpurun_out/timeline.log
