for c in 0 1; do echo "== cfg $c"; QFLASH_ATTN_CFG=$c timeout 300 python tools/diag_cfg.py; done 2>&1 | tee gpurun_out/diag.log
for c in 0 1; do
  QFLASH_ATTN_CFG=$c timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -8 | tee gpurun_out/pytest_cfg$c.log
done
