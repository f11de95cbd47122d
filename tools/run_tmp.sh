timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "multi or segmented or panels" > gpurun_out/t_multi.log 2>&1; echo rc=$? >> gpurun_out/t_multi.log
python tools/cadence_c2.py > gpurun_out/cad3.log 2>&1
PDLP_MULTI=0 python tools/cadence_c2.py > gpurun_out/cad3b.log 2>&1
