import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    r = d["roofline"]
    print(f"{f:32s} us/step {d['us_per_call']:9.2f}  TOPS {d['value']:8.2f}  attn_us {r['attn_us']:9.2f}  "
          f"alu_frac {r['frac']:.3f}  tensor {r['tensor']['frac']:.3f}  e2e {d['e2e']['value'] if d['e2e'] else None}")
