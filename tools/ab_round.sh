python -m pytest tests/test_gpu_parity.py tests/test_gpu_00_bench_configs.py -q -x -p no:cacheprovider > gpurun_out/v25_tests.log 2>&1; echo rc=$? >> gpurun_out/v25_tests.log
VARIANTS="upold" bash tools/ab_variants.sh > gpurun_out/v25_ab.txt 2>&1
NPSD_MERGE_UP0=0 python tools/ncu_target.py --iters 5 > gpurun_out/v25_split.txt 2>&1
