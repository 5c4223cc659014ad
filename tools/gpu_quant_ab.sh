set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "quantiz or pipeline or prepare or dscale or sqnr" 2>&1 | tail -3
for f in 1 0; do
  QFLASH_QUANT_FUSED=$f timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 2000 2>&1 | tail -1 > gpurun_out/bench_q$f.log
  QFLASH_QUANT_FUSED=$f timeout 300 python bench.py --workload A4 --no-cpu-baseline --no-e2e --steps 2000 2>&1 | tail -1 > gpurun_out/bench_a4_q$f.log
done
QFLASH_QUANT_FUSED=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q0.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
QFLASH_QUANT_FUSED=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q1.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
