# C2 schedule sweeps (column-pass threshold, panel budget, variant builds); tuning only.
# column-pass threshold sweep (panels on) and panel budget sweep
for t in 16 32 64 128 256 512 2048; do PDLP_SHORT_MAX=$t python tools/c2_variants.py default >> gpurun_out/sw.jsonl 2>> gpurun_out/sw.err; echo "T=$t" >> gpurun_out/sw.jsonl; done
for b in 2688 3600; do PDLP_PANEL_BUDGET=$b python tools/c2_variants.py default >> gpurun_out/sw.jsonl 2>> gpurun_out/sw.err; echo "B=$b" >> gpurun_out/sw.jsonl; done
python tools/c2_variants.py tools/variants/mb2g8/libpdlp_b200.so tools/variants/mb2g16/libpdlp_b200.so >> gpurun_out/sw.jsonl 2>> gpurun_out/sw.err
