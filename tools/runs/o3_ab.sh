# A/B: ortho with r read into registers and 2-plane prefetch (70 KB, lib_o2d), plus a 3-blocks/SM register cap (lib_o3)
for i in 1 2; do for v in "X=1" "NPSD_B200_LIB=variants/lib_o2d.so" "NPSD_B200_LIB=variants/lib_o3.so"; do
  echo "== $v"; env $v timeout 120 python tools/ncu_target.py --iters 5 | grep -E "ortho|total" | awk '{print $1, $2}' | tr '\n' ' '; echo
done; done
