timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python tools/sanitize.py > gpurun_out/sanitize_memcheck2.log 2>&1
tail -4 gpurun_out/sanitize_memcheck2.log
