timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_schedule.py -q -m gpu -x > gpurun_out/t_e2e.log 2>&1; echo rc=$? >> gpurun_out/t_e2e.log
python tools/e2e_c2.py > gpurun_out/e2e2.log 2>&1
