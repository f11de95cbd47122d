timeout 1200 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python tools/sanitize_small.py > gpurun_out/san_memcheck.log 2>&1; echo rc=$? >> gpurun_out/san_memcheck.log
