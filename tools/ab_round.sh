python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "spmv or psdo or solve or ortho" > gpurun_out/v19_tests.log 2>&1; echo rc=$? >> gpurun_out/v19_tests.log
VARIANTS="ctr0" bash tools/ab_variants.sh > gpurun_out/v19_ab.txt 2>&1
python tools/ncu_target.py --iters 1 > /dev/null 2>&1; ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_ortho2|k_update2" -c 4 --csv python tools/ncu_target.py --iters 1 > gpurun_out/v19_ncu.csv 2>&1
NPSD_B200_LIB=$PWD/variants/libnpsd_b200_ctr0.so ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_ortho2|k_update2" -c 4 --csv python tools/ncu_target.py --iters 1 > gpurun_out/v19_ncu0.csv 2>&1
