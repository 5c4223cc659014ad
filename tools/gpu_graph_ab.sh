set -x
for wl in "A3 --batch 8" "A4 --batch 8" "A1 --batch 1" "L14 --batch 64 --steps 30"; do
  timeout 300 python tools/graph_ab.py --workload $wl 2>&1 | grep graph | tee -a gpurun_out/graph_ab.log
done
