# round-2b evidence: GPU suite, sweep (chained graphs), default bench line, ncu launch list
mkdir -p gpurun_out/prof
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -3 > gpurun_out/fin_pytest.log
bash tools/sweep.sh
timeout 300 python bench.py --scales per-head --no-cpu-baseline --no-e2e --no-table1 2>&1 | tail -1 > gpurun_out/fin_a3_per_head.json
timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --scales per-head --no-cpu-baseline --no-e2e --no-table1 2>&1 | tail -1 > gpurun_out/fin_l14_per_head.json
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/r2b_launches_default.csv python bench.py --steps 24 --warmup 3 --no-cpu-baseline --no-e2e --no-extra --no-table1 > /dev/null 2>&1
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1
