"""Markdown table from the bench sweep lines (gpurun_out/sweep_*.json)."""
import glob
import json
import sys

rows = []
for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep_*.json")):
    try:
        b = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    r, c = b["roofline"], b["config"]
    rows.append((c["workload"], c["problems"], c["seq_len"], c["head_dim"], b["us_per_call"], b["value"],
                 r["attn_us"], r["frac"], r["hbm"]["frac"], b["gpu_launches"] // b["steps"], b["clocks"]["sm_mhz"] or 0))
print("| workload | P | N | d | step µs | TOPS | dominant kernel µs | ALU frac | HBM frac | launches/step | SM MHz |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for w in rows:
    print("| %s | %d | %d | %d | %.1f | %.2f | %.1f | %.3f | %.3f | %d | %.0f |" % w)
