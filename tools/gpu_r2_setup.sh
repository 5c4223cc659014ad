# setup overlapped with the fused prologue's loads: parity + bench + timeline
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -3 > gpurun_out/su_pytest.log
for wl in "A1 1" "A3 1" "A7 1" "A2 8" "A3 8" "A4 8" "A7 8"; do set -- $wl
  timeout 200 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --no-e2e --no-extra --no-table1 2>&1 | tail -1 > gpurun_out/su_$1b$2.log
done
QFLASH_LIB=libqflash_fqt.so timeout 200 python tools/fq_timing_graph.py > gpurun_out/su_fq_timeline.txt 2>&1
python - <<PY
import json,glob
for f in sorted(glob.glob("gpurun_out/su_*b*.log")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["ms_per_step"]*1e3,2), "us step")
    except Exception as e: print(f, "ERR", e)
PY
