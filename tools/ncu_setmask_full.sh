# full ncu captures of set_mask's heaviest level-0 kernels at C3 (classifier, window keys, dedup insert)
ncu --set full --clock-control none --import-source on -k "regex:k_classify_simd|k_window_keys|k_dedup_insert" -s 3 -c 3 -o gpurun_out/sm_full python tools/setmask_target.py --config C3 --reps 2 > gpurun_out/sm_full.log 2>&1
