# C2 (full size) step kernels: CUDA-event split, then one ncu --set full
# capture of each step kernel (after the plain command exits 0).
set -x
export PDLP_TIMING=1
timeout 600 python tools/bench_configs.py c2 --steps 128 --warmup 8 --ttt-limit 1 > gpurun_out/c2_cfg.jsonl 2> gpurun_out/c2_cfg.err
echo rc=$?
timeout 300 python tools/c2_steps.py > gpurun_out/c2_plain.log 2>&1
echo rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"row_pass|col_pass|primal_pass" --launch-skip 6 -c 3 -o gpurun_out/c2_full -f python tools/c2_steps.py > gpurun_out/c2_ncu.log 2>&1
echo rc=$?
