timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_dropin.py -q -x -p no:cacheprovider --timeout 120 2>&1 | tail -3
bash tools/runs/setup_list.sh
