python -m pytest tests/test_gpu_parity.py tests/test_gpu_00_bench_configs.py -q -x -p no:cacheprovider > gpurun_out/v26_tests.log 2>&1; echo rc=$? >> gpurun_out/v26_tests.log
bash tools/setmask_ab.sh > gpurun_out/v26_setmask.log 2>&1
bash tools/ncu_setmask.sh
