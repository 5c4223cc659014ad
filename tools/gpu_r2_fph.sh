timeout 300 python -m pytest tests -m gpu -q --timeout 300 -k "per_head" 2>&1 | tail -2 | tee gpurun_out/r2_fph_tests.log
for wl in "A3 8" "A4 8" "A1 1"; do set -- $wl
  timeout 200 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --scales per-head 2>&1 | tail -1 > gpurun_out/fph_$1b$2.log
done
timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --scales per-head 2>&1 | tail -1 > gpurun_out/fph_L14b64.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/r2_bench_table1.json
