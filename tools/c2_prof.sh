# C2 (full size) step kernels: one ncu --set full capture of each step kernel
# (after the plain command exits 0).  Skips the first attempt (5 launches:
# primal pass, two column-panel row passes, the split column pass).
timeout 300 python tools/c2_steps.py > gpurun_out/c2_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"row_pass|col_pass|primal_pass|col_product|col_epi_decide" --launch-skip 5 -c 5 -o gpurun_out/c2_full_r2 -f python tools/c2_steps.py > gpurun_out/c2_ncu.log 2>&1
echo rc=$?
