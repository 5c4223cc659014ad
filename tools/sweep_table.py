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
    st = b.get("stages") or {}
    rows.append((c["workload"], c["problems"], c["seq_len"], c["head_dim"], b["us_per_call"], b["value"],
                 r["frac"], r["hbm"]["frac"], st.get("attention_int8_us", float("nan")),
                 st.get("attention_int8_tops", float("nan")), st.get("quantize_qkv_us", float("nan")),
                 st.get("dequantize_us", float("nan")), b["gpu_launches"] // b["steps"],
                 (b.get("clocks") or {}).get("sm_mhz") or 0))
print("| workload | P | N | d | step µs | TOPS | step ALU frac | step HBM frac | attention (int8) µs | "
      "attention TOPS | quantizer µs | dequantizer µs | launches/step | SM MHz |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for w in rows:
    print("| %s | %d | %d | %d | %.1f | %.2f | %.3f | %.3f | %.1f | %.1f | %.1f | %.1f | %d | %.0f |" % w)
