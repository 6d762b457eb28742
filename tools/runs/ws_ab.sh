timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -q -x -p no:cacheprovider --timeout 120 2>&1 | tail -1
for i in 1 2; do for v in "NPSD_B200_LIB=variants/lib_base.so" "NPSD_B200_LIB=variants/lib_wsearch.so"; do
  echo "== $v"; env $v timeout 120 python tools/ncu_target.py --iters 5 | grep -E "L0|ortho|update|total" | awk '{print $1, $2}' | tr '\n' ' '; echo
done; done
