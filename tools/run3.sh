python tools/c2_variants.py default tools/variants/segnoef/libpdlp_b200.so > gpurun_out/v3.jsonl 2> gpurun_out/v3.err
PDLP_PANEL_SEG=1 python tools/c2_variants.py default >> gpurun_out/v3.jsonl 2>> gpurun_out/v3.err
