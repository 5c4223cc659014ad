timeout 600 python -m pytest tests -m gpu -q --timeout 300 -k "fused or workload or full_size or sharded or packed_qkv" 2>&1 | tail -2 | tee gpurun_out/r2_pytest_gpu.log
for wl in "A4 8" "SwinB-s1 8" "A5 8" "A3 8"; do set -- $wl
  timeout 200 python bench.py --workload $1 --batch $2 --steps 2000 --no-cpu-baseline --no-e2e --no-extra 2>&1 | tail -1 > gpurun_out/s12_$1b$2.log
done
timeout 300 python bench.py --workload L14 --batch 64 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-extra 2>&1 | tail -1 > gpurun_out/s12_L14b64.log
