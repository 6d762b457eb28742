timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/gpu_tests.log
for v in "NPSD_COARSE_ZC=8" "NPSD_COARSE_ZC=4" "NPSD_COARSE_ZC=2"; do
  echo "== $v"; env $v timeout 120 python tools/ncu_target.py --iters 5 | grep -E "L1|L2|L3|total"
done
