# fused-step grid policy A/B (QFLASH_FUSED_GRID=0: one CTA per tile group; default: 16 / all SMs)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -3 > gpurun_out/gr_pytest.log
for g in 0 1; do
for wl in "A1 1" "A3 1" "A7 1" "A5 1" "A2 8" "A3 8" "A4 8" "A7 8"; do set -- $wl
  QFLASH_FUSED_GRID=$g timeout 200 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --no-e2e --no-extra --no-table1 2>&1 | tail -1 > gpurun_out/gr${g}_$1b$2.log
done; done
python - <<PY
import json,glob
for f in sorted(glob.glob("gpurun_out/gr[01]_*.log")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["ms_per_step"]*1e3,2), "us")
    except Exception as e: print(f, "ERR", e)
PY
