# attention configuration A/B on the Swin shapes and A3 (forced QFLASH_ATTN_CFG)
mkdir -p gpurun_out
for c in -1 0 1 2 3; do
for wl in "A4 8" "A7 8" "SwinB-s1 8" "A3 8" "A4 1"; do set -- $wl
  QFLASH_ATTN_CFG=$c timeout 200 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --no-e2e --no-table1 2>&1 | tail -1 > gpurun_out/cfg${c}_$1b$2.log
done; done
python - <<PY
import json,glob
for f in sorted(glob.glob("gpurun_out/cfg*_*.log")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["ms_per_step"]*1e3,2), "us step", round(d["stages"]["attention_int8_us"],2), "us attn")
    except Exception as e: print(f, "ERR", e)
PY
