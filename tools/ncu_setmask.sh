for cfg in C1 C3; do
NPSD_SETUP_SERIAL=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sm_launch_$cfg.csv python tools/setmask_target.py --config $cfg --reps 2 > gpurun_out/sm_ncu_$cfg.log 2>&1
done
