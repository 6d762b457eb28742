for v in "" "NPSD_B200_LIB=variants/lib_d0a2.so" "NPSD_B200_LIB=variants/lib_d0a6.so"; do
  echo "== $v"; env $v timeout 120 python tools/ncu_target.py --iters 5 | grep -E "down_L0|total" | tr '\n' ' '; echo
done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 120 -k "precond or psdo" 2>&1 | tail -2
