# Every kernel launch of a 12-iteration C2 solve (setup, cadences, attempts)
timeout 300 python tools/c2_steps.py > gpurun_out/c2l_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/c2_launches.csv python tools/c2_steps.py > gpurun_out/c2l_ncu.log 2>&1
echo rc=$?
