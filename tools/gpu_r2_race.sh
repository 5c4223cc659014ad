# racecheck / synccheck of configuration 2 (row owner + correction, named-barrier alpha hand-off)
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -3 | tee gpurun_out/r2_pytest_gpu.log
QFLASH_ATTN_CFG=2 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -k "edge_seq or alignments or workload_parity" 2>&1 | tail -2 > gpurun_out/r2_cfg2_tests.log
QFLASH_ATTN_CFG=2 timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python tools/sanitize.py > gpurun_out/r2_racecheck_cfg2.log 2>&1
QFLASH_ATTN_CFG=2 timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize.py > gpurun_out/r2_synccheck_cfg2.log 2>&1
tail -5 gpurun_out/r2_racecheck_cfg2.log gpurun_out/r2_synccheck_cfg2.log
