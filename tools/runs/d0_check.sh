timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 120 -k "precond or psdo or trained" 2>&1 | tail -3
timeout 120 python tools/ncu_target.py --iters 5
