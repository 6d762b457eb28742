# targeted GPU checks of the latest set_mask changes, then set_mask timing and a short bench
python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -q -x -p no:cacheprovider > gpurun_out/val_tests.log 2>&1; echo "rc=$?" >> gpurun_out/val_tests.log
bash tools/setmask_ab.sh > gpurun_out/val_setmask.log 2>&1
bash tools/ncu_setmask.sh
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/val_bench.json 2> gpurun_out/val_bench.err; echo "rc=$?" >> gpurun_out/val_bench.err
python -m pytest tests/test_gpu_00_bench_configs.py -q -x -p no:cacheprovider > gpurun_out/val_cfg.log 2>&1; echo "rc=$?" >> gpurun_out/val_cfg.log
