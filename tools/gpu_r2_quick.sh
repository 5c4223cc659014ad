# quick A/B: fused-step timeline (timing build), bench lines (A3 b8, A1 b1, A4 b8, A2 b8), GPU suite
# usage: bash tools/gpu_r2_quick.sh TAG [pytest]
TAG=${1:-q}; PYT=$2
mkdir -p gpurun_out
QFLASH_LIB=libqflash_fqt.so timeout 200 python tools/fq_timing_graph.py > gpurun_out/${TAG}_fq_timeline.txt 2>&1
for wl in "A3 8" "A1 1" "A4 8" "A2 8"; do set -- $wl
  timeout 200 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --no-e2e --no-extra --no-table1 2>&1 | tail -1 > gpurun_out/${TAG}_$1b$2.log
done
if [ "$PYT" = "pytest" ]; then timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -3 > gpurun_out/${TAG}_pytest.log; fi
python - <<PY
import json,glob
for f in sorted(glob.glob("gpurun_out/${TAG}_*b*.log")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["ms_per_step"]*1e3,2), "us")
    except Exception as e: print(f, "ERR", e)
PY
