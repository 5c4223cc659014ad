for c in 0 1 2; do
  QFLASH_ATTN_CFG=$c timeout 600 compute-sanitizer --tool racecheck --print-limit 5 python tools/sanitize.py > gpurun_out/sanitize_race_c$c.log 2>&1
  echo "cfg $c rc=$?" >> gpurun_out/sanitize_summary.log
  tail -3 gpurun_out/sanitize_race_c$c.log >> gpurun_out/sanitize_summary.log
done
