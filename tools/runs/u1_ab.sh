# A/B: update with a 1-plane prefetch (43 KB) uncapped (lib_u1b) and capped at 5 blocks/SM (lib_u1a)
for i in 1 2; do for v in "X=1" "NPSD_B200_LIB=variants/lib_u1a.so" "NPSD_B200_LIB=variants/lib_u1b.so"; do
  echo "== $v"; env $v timeout 120 python tools/ncu_target.py --iters 5 | grep -E "update|total" | awk '{print $1, $2}' | tr '\n' ' '; echo
done; done
