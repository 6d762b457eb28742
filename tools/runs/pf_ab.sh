# A/B: stencil prefetch depths (ortho 3 -> 2, update 2 -> 3) against the default build
for i in 1 2; do for v in "X=1" "NPSD_B200_LIB=variants/lib_o2.so" "NPSD_B200_LIB=variants/lib_u3.so"; do
  echo "== $v"; env $v timeout 120 python tools/ncu_target.py --iters 5 | grep -E "ortho|update|total" | awk '{print $1, $2}' | tr '\n' ' '; echo
done; done
