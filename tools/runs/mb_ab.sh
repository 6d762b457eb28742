for i in 1 2; do for v in "X=1" "NPSD_B200_LIB=variants/lib_mb.so"; do
  echo "== $v"; env $v timeout 120 python tools/ncu_target.py --iters 5 | grep -E "L0|total" | awk '{print $1, $2}' | tr '\n' ' '; echo
done; done
