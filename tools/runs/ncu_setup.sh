ncu --set full --import-source on --clock-control none -k regex:"k_setup_l0_march|k_zsums_rows|k_classify" -c 6 -f -o gpurun_out/setup python tools/setmask_target.py > gpurun_out/ncu_setup.log 2>&1; echo ncu $?
ncu -i gpurun_out/setup.ncu-rep --page raw --csv > gpurun_out/setup_raw.csv 2>&1
for id in 0 1; do ncu -i gpurun_out/setup.ncu-rep --page source --csv --print-source sass --launch-skip $id --launch-count 1 > gpurun_out/setup_src_$id.csv 2>&1; done
