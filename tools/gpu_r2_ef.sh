# evict-first A/B + hot-L2 timeline (icache-from-HBM hypothesis)
mkdir -p gpurun_out
QFLASH_LIB=libqflash_fqt.so timeout 200 python tools/fq_timing_graph.py > gpurun_out/ef_tl_base.txt 2>&1
FQ_SETS=2 QFLASH_LIB=libqflash_fqt.so timeout 200 python tools/fq_timing_graph.py > gpurun_out/ef_tl_hot.txt 2>&1
QFLASH_LIB=libqflash_fqte.so timeout 200 python tools/fq_timing_graph.py > gpurun_out/ef_tl_ef.txt 2>&1
for lib in libqflash.so libqflash_ef.so; do
for wl in "A3 8" "A1 1" "A4 8" "A2 8"; do set -- $wl
  QFLASH_LIB=$lib timeout 200 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --no-e2e --no-extra --no-table1 2>&1 | tail -1 > gpurun_out/ef_${lib}_$1b$2.log
done; done
python - <<PY
import json,glob
for f in sorted(glob.glob("gpurun_out/ef_lib*.log")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["ms_per_step"]*1e3,2), "us")
    except Exception as e: print(f, "ERR", e)
PY
