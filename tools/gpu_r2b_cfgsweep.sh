# every forced configuration on every Table-1 workload and the Swin-B stages (b1 / b8): is AUTO the best?
mkdir -p gpurun_out/cfgs
for wl in A1 A2 A3 A4 A5 A6 A7 SwinB-s1 SwinB-s2 SwinB-s3 SwinB-s4; do for b in 1 8; do for c in -1 0 1 2 3; do
  QFLASH_ATTN_CFG=$c timeout 120 python bench.py --workload $wl --batch $b --steps 1500 --warmup 20 --no-cpu-baseline --no-e2e --no-table1 2>&1 | tail -1 > gpurun_out/cfgs/${wl}_b${b}_c${c}.json
done; done; done
python - <<PY
import json,glob,collections
res=collections.defaultdict(dict)
for f in glob.glob("gpurun_out/cfgs/*.json"):
    k,c=f.split('/')[-1].rsplit('_c',1); c=int(c[:-5])
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); res[k][c]=(d["ms_per_step"]*1e3, d["stages"]["attention_int8_us"])
    except Exception as e: res[k][c]=None
for k in sorted(res):
    r=res[k]; ok={c:v for c,v in r.items() if v}
    best=min((v[0],c) for c,v in ok.items() if c>=0) if any(c>=0 for c in ok) else None
    print(k, " ".join("c%d %.2f/%.2f"%(c,v[0],v[1]) for c,v in sorted(ok.items())), "| best", best)
PY
