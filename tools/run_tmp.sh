timeout 1100 python -m pytest tests/ -q -m gpu -x -k "not scale" > gpurun_out/t_e2e.log 2>&1; echo rc=$? >> gpurun_out/t_e2e.log
python tools/e2e_c2.py > gpurun_out/e2e2.log 2>&1
