# A/B: k_down_l0 at 4 blocks/SM (D0_MINB=4, lib_d4) vs 3
for i in 1 2; do for v in "X=1" "NPSD_B200_LIB=variants/lib_d4.so"; do
  echo "== $v"; env $v timeout 120 python tools/ncu_target.py --iters 5 | grep -E "down_L0|total" | awk '{print $1, $2}' | tr '\n' ' '; echo
done; done
