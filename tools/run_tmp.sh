python tools/c2_variants.py default tools/variants/gkeep/libpdlp_b200.so > gpurun_out/v7.jsonl 2> gpurun_out/v7.err
bash tools/c2_prof.sh
