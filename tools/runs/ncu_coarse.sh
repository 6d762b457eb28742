# ncu --set full of the z-marching coarse kernels (L1 down and up at C3 256^3)
ncu --set full --import-source on --clock-control none -k regex:"k_cdownz|k_cupz" -c 6 -f -o gpurun_out/coarse python tools/ncu_target.py --iters 1 > gpurun_out/ncu_coarse.log 2>&1; echo ncu $?
ncu -i gpurun_out/coarse.ncu-rep --page raw --csv > gpurun_out/coarse_raw.csv 2>&1
for id in 0 1 2 3 4 5; do ncu -i gpurun_out/coarse.ncu-rep --page source --csv --print-source sass --launch-skip $id --launch-count 1 > gpurun_out/coarse_src_$id.csv 2>&1; done
ls -la gpurun_out/
