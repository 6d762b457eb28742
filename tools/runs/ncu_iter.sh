# ncu --set full of one PSDO iteration's kernels (direct launches), C3 256^3
ncu --set full --import-source on --clock-control none -k regex:"k_ortho2|k_update2|k_down_l0|k_up_l0|k_mixed_down0|k_mixed_up0" -c 6 -f -o gpurun_out/iter python tools/ncu_target.py --iters 1 > gpurun_out/ncu_iter.log 2>&1; echo ncu $?
ncu -i gpurun_out/iter.ncu-rep --page raw --csv > gpurun_out/iter_raw.csv 2>&1
for id in 0 1 2 3 4 5; do ncu -i gpurun_out/iter.ncu-rep --page source --csv --print-source sass --launch-skip $id --launch-count 1 > gpurun_out/iter_src_$id.csv 2>&1; done
