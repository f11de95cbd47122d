L=tools/spmv_lab/lab
F="col seg2 U=8 span=1024 minb=3"
$L 5000000 10000000 0 "$F" > gpurun_out/labq3.txt 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:seg2_kernel -c 1 -o gpurun_out/lab_seg2 -f $L 5000000 10000000 0 "$F" > gpurun_out/labn5.txt 2>&1
