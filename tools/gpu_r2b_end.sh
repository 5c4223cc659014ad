# end-of-session evidence: GPU suite, smoke, default bench line, L14 line, launch list
mkdir -p gpurun_out/end
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 2>&1 | tail -3 > gpurun_out/end/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/end/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/end/bench_default.log 2>&1
timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-table1 2>&1 | tail -1 > gpurun_out/end/bench_l14.json
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/end/launches_default.csv python bench.py --steps 48 --warmup 3 --no-cpu-baseline --no-e2e --no-extra --no-table1 > /dev/null 2>&1
