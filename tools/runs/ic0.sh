timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "ic0 or pcg" 2>&1 | tail -15
