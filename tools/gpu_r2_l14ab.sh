timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2 > gpurun_out/pk_pytest.log
for rep in 1 2; do for lib in libqflash_base.so libqflash.so; do
QFLASH_LIB=$lib timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-table1 2>&1 | tail -1 > gpurun_out/pk_${lib}_r$rep.json
done; done
QFLASH_LIB=libqflash.so LIBS="libqflash_base.so libqflash.so" bash tools/gpu_r2_abab.sh pk "A3 8" "A4 8"
python - <<PY
import json,glob
for f in sorted(glob.glob("gpurun_out/pk_lib*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d["ms_per_step"]*1e3,1), round(d["stages"]["attention_int8_us"],1))
PY
