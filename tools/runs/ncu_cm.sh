ncu --set full --import-source on --clock-control none -k regex:"k_classify_march" -c 1 -f -o gpurun_out/cm python tools/setmask_target.py > /dev/null 2>&1; echo ncu $?
ncu -i gpurun_out/cm.ncu-rep --page raw --csv > gpurun_out/cm_raw.csv 2>&1
ncu -i gpurun_out/cm.ncu-rep --page source --csv --print-source sass > gpurun_out/cm_src.csv 2>&1
