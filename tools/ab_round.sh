python -m pytest tests/test_gpu_parity.py tests/test_gpu_00_bench_configs.py tests/test_gpu_slab.py -q -x -p no:cacheprovider > gpurun_out/v16_tests.log 2>&1; echo rc=$? >> gpurun_out/v16_tests.log
python tools/env_ab.py NPSD_COARSE_SKIP 0 1 > gpurun_out/v16_ab_skip.txt 2>&1
python tools/env_ab.py NPSD_COARSE_SKIP 1 0 >> gpurun_out/v16_ab_skip.txt 2>&1
