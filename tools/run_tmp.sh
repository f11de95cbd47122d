timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_split.log 2>&1; echo rc=$? >> gpurun_out/t_split.log
python tools/c2_variants.py default tools/variants/nosplit/libpdlp_b200.so > gpurun_out/v10.jsonl 2> gpurun_out/v10.err
