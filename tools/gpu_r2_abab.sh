# same-box ABAB over libraries; usage: LIBS="libqflash_base.so libqflash.so" bash tools/gpu_r2_abab.sh TAG "wl b [env]" ...
TAG=$1; shift
LIBS=${LIBS:-"libqflash_base.so libqflash.so"}
SPECS=("$@")
mkdir -p gpurun_out
for rep in 1 2; do
for lib in $LIBS; do
for spec in "${SPECS[@]}"; do set -- $spec
  env ${3:-X=1} QFLASH_LIB=$lib timeout 200 python bench.py --workload $1 --batch $2 --steps 3000 --no-cpu-baseline --no-e2e --no-extra --no-table1 2>&1 | tail -1 > gpurun_out/${TAG}_${lib}_$1b$2_r$rep.log
done; done; done
python - <<PY
import json,glob,collections
res=collections.defaultdict(list)
for f in sorted(glob.glob("gpurun_out/${TAG}_*.log")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); k=f.split('_r')[0]; res[k].append(round(d["ms_per_step"]*1e3,2))
    except Exception as e: print(f, "ERR", e)
for k,v in sorted(res.items()): print(k, v)
PY
