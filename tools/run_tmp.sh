timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "segmented or skewed or spmv" > gpurun_out/t_seg.log 2>&1; echo rc=$? >> gpurun_out/t_seg.log
python tools/c2_variants.py default tools/variants/nostaged/libpdlp_b200.so > gpurun_out/v6.jsonl 2> gpurun_out/v6.err
