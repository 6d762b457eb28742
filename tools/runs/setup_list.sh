timeout 120 python tools/setmask_target.py
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/setup_launches.csv python tools/setmask_target.py > /dev/null 2>&1; echo ncu $?
