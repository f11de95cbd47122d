timeout 900 python tools/bench_configs.py c3 --steps 128 --warmup 8 --ttt-limit 30 > gpurun_out/cfg3.jsonl 2> gpurun_out/cfg3.err
PDLP_STAGE_BUDGET=2016 timeout 900 python tools/bench_configs.py c3 --steps 128 --warmup 8 --ttt-limit 1 >> gpurun_out/cfg3.jsonl 2>> gpurun_out/cfg3.err
PDLP_STAGE_BUDGET=1344 timeout 900 python tools/bench_configs.py c3 --steps 128 --warmup 8 --ttt-limit 1 >> gpurun_out/cfg3.jsonl 2>> gpurun_out/cfg3.err
PDLP_SHORT_MAX=256 timeout 900 python tools/bench_configs.py c3 --steps 128 --warmup 8 --ttt-limit 1 >> gpurun_out/cfg3.jsonl 2>> gpurun_out/cfg3.err
