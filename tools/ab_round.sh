python -m pytest tests/test_gpu_parity.py tests/test_gpu_00_bench_configs.py tests/test_gpu_slab.py tests/test_gpu_boundary.py tests/test_gpu_dropin.py -q -x -p no:cacheprovider > gpurun_out/v17_tests.log 2>&1; echo rc=$? >> gpurun_out/v17_tests.log
bash tools/setmask_ab.sh > gpurun_out/v17_setmask.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v17_bench.json 2> gpurun_out/v17_bench.err
