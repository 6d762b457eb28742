# full ncu captures of set_mask's slowest kernels (classifier at C3, one-block scan at C1)
ncu --set full --clock-control none --import-source on -k "regex:k_classify_simd" -s 1 -c 1 -o gpurun_out/sm_classify python tools/setmask_target.py --config C3 --reps 2 > gpurun_out/sm_full1.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_scan_small" -s 5 -c 1 -o gpurun_out/sm_scan python tools/setmask_target.py --config C1 --reps 2 > gpurun_out/sm_full2.log 2>&1
