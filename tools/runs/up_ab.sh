# A/B: k_up_l0 register caps (UP0_MINB 1 default / 4 / 5)
for i in 1 2; do for v in "X=1" "NPSD_B200_LIB=variants/lib_up4.so" "NPSD_B200_LIB=variants/lib_up5.so"; do
  echo "== $v"; env $v timeout 120 python tools/ncu_target.py --iters 5 | grep -E "up_L0|total" | awk '{print $1, $2}' | tr '\n' ' '; echo
done; done
