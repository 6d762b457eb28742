python -m pytest tests/test_gpu_parity.py tests/test_gpu_00_bench_configs.py -q -x -p no:cacheprovider > gpurun_out/v24_tests.log 2>&1; echo rc=$? >> gpurun_out/v24_tests.log
VARIANTS="mixold mix5" bash tools/ab_variants.sh > gpurun_out/v24_ab.txt 2>&1
python tools/ncu_target.py --iters 1 > /dev/null 2>&1; ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_mixed_down0" -c 2 --csv python tools/ncu_target.py --iters 1 > gpurun_out/v24_ncu.csv 2>&1
NPSD_B200_LIB=$PWD/variants/libnpsd_b200_mixold.so ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_mixed_down0" -c 2 --csv python tools/ncu_target.py --iters 1 > gpurun_out/v24_ncu_old.csv 2>&1
