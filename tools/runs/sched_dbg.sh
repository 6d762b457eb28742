timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -q -x -p no:cacheprovider --timeout 120 2>&1 | grep -E "^E |FAILED|Error" | head -20
