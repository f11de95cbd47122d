L=tools/spmv_lab/lab
$L 5000000 10000000 0 "row vec G=8" > gpurun_out/labq.txt 2>&1 && \
ncu --set full --clock-control none -k regex:vec_kernel -c 1 -o gpurun_out/lab_vec8 -f $L 5000000 10000000 0 "row vec G=8" > gpurun_out/labn1.txt 2>&1
$L 5000000 10000000 0 "row panels P=2" >> gpurun_out/labq.txt 2>&1 && \
ncu --set full --clock-control none -k regex:panel_kernel -c 2 -o gpurun_out/lab_p2 -f $L 5000000 10000000 0 "row panels P=2" > gpurun_out/labn2.txt 2>&1
$L 5000000 10000000 0 "col item=256 seq=128" >> gpurun_out/labq.txt 2>&1 && \
ncu --set full --clock-control none -k regex:wb_kernel -c 1 -o gpurun_out/lab_wbcol -f $L 5000000 10000000 0 "col item=256 seq=128" > gpurun_out/labn3.txt 2>&1
