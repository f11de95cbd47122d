L=tools/spmv_lab/lab
$L 5000000 10000000 1 "row vec G=8" > gpurun_out/labq2.txt 2>&1 && \
ncu --set full --clock-control none -k regex:vec_kernel -c 1 -o gpurun_out/lab_vec8s -f $L 5000000 10000000 1 "row vec G=8" > gpurun_out/labn4.txt 2>&1
