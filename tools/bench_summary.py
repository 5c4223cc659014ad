"""One line per bench JSON log: us/step, value, roofline frac, stages (gpurun_out helper)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    r = d.get("roofline", {})
    print("%-44s %9.2f us  %8.2f %s  frac %.3f  attn %.2f us  clk %s" % (
        f.split("/")[-1], d.get("us_per_call", d.get("ms_per_step", 0) * 1e3), d["value"], d["unit"],
        r.get("frac", 0), r.get("attn_us", 0), (d.get("clocks") or {}).get("sm_mhz")))
