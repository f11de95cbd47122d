timeout 1100 python -m pytest tests/ -q -m gpu -x -k "not scale" > gpurun_out/t_lp.log 2>&1; echo rc=$? >> gpurun_out/t_lp.log
timeout 1500 python tools/c1_seeds.py > gpurun_out/c1_seeds.jsonl 2> gpurun_out/c1_seeds.err
