timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/b2.json 2> gpurun_out/b2.err; echo "rc=$?" >> gpurun_out/b2.err
PDLP_TIMING=1 timeout 300 python tools/c2_variants.py default > gpurun_out/c2t.jsonl 2> gpurun_out/c2t.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2.json 2> gpurun_out/r2.err; echo "rc=$?" >> gpurun_out/r2.err
