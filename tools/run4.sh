timeout 1100 python -m pytest tests/ -q -m gpu -x --durations=8 > gpurun_out/gpu_all2.log 2>&1; echo rc=$? >> gpurun_out/gpu_all2.log
python tools/cadence_c2.py > gpurun_out/cad2.log 2>&1
