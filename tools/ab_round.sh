python -m pytest tests/test_gpu_parity.py tests/test_gpu_00_bench_configs.py tests/test_gpu_slab.py -q -x -p no:cacheprovider > gpurun_out/v12_tests.log 2>&1; echo rc=$? >> gpurun_out/v12_tests.log
python tools/env_ab.py NPSD_PDL_COARSE 0 1 > gpurun_out/v12_ab_pdl.txt 2>&1
VARIANTS="mixold mx4" bash tools/ab_variants.sh > gpurun_out/v12_ab_mix.txt 2>&1
python tools/ncu_target.py --iters 1 > /dev/null 2>&1; ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k "regex:k_mixed_down0" -c 2 --csv python tools/ncu_target.py --iters 1 > gpurun_out/v12_ncu.csv 2>&1
