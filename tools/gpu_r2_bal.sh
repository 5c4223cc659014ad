# balanced key split (cfg 0) + skipped empty P V K-steps + cfg 1 for multi-wave Swin
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -5 > gpurun_out/bal_pytest.log
for wl in "A1 1" "A3 1" "A7 1" "A2 8" "A3 8" "A4 8" "A7 8" "A6 8" "SwinB-s1 8"; do set -- $wl
  timeout 200 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --no-e2e --no-table1 2>&1 | tail -1 > gpurun_out/bal_$1b$2.log
done
timeout 300 python bench.py --workload L14 --batch 64 --steps 24 --warmup 3 --no-cpu-baseline --no-e2e --no-table1 2>&1 | tail -1 > gpurun_out/bal_L14b64.log
timeout 200 python tools/timeline_gpu.py > gpurun_out/bal_timeline.txt 2>&1
python - <<PY
import json,glob
for f in sorted(glob.glob("gpurun_out/bal_*b*.log")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["ms_per_step"]*1e3,2), "us step", round(d["stages"]["attention_int8_us"],2), "us attn")
    except Exception as e: print(f, "ERR", e)
PY
