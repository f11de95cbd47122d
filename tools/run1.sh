timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/t_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_parity.log
python tools/c2_variants.py default > gpurun_out/seg1.jsonl 2> gpurun_out/seg1.err
PDLP_SEG=0 python tools/c2_variants.py default >> gpurun_out/seg1.jsonl 2>> gpurun_out/seg1.err
