# per-iteration solve time (graph) per library variant (tools/build_variant.sh), C1/C2/C3
for v in default ${VARIANTS} default; do
  if [ $v = default ]; then unset NPSD_B200_LIB; else export NPSD_B200_LIB=$PWD/variants/libnpsd_b200_$v.so; fi
  echo "== $v"
  python tools/env_ab.py NPSD_DUMMY 0 2>&1
done
