timeout 400 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -2 | tee gpurun_out/pytest.log
for wl in "A1 1" "A2 1" "A7 1" "SwinB-s4 1" "A3 1" "A6 1"; do
  set -- $wl
  timeout 120 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/bench_cl_$1.log
done
