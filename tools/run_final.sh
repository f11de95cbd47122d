# Round-end measurements (one GPU): the driver-shaped bench, the reference
# arm, a 64-iteration window, C3 / C4-shard configs, and the C2 launch list.
set -x
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/final_b20.json 2> gpurun_out/final_b20.err
timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final_ref20.json 2> gpurun_out/final_ref20.err
timeout 1200 python bench.py --steps 64 --warmup 8 --no-cpu-baseline --no-c1 --ttt-limit 300 > gpurun_out/final_b64.json 2> gpurun_out/final_b64.err
timeout 1500 python tools/bench_configs.py c3 c4w --steps 128 --warmup 8 --ttt-limit 60 > gpurun_out/final_cfg.jsonl 2> gpurun_out/final_cfg.err
timeout 300 python tools/c2_steps.py > gpurun_out/c2l_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/c2_launches_r2.csv python tools/c2_steps.py > gpurun_out/c2l_ncu.log 2>&1
echo done
