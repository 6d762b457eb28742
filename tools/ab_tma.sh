# A/B of compile-time variants (tools/build_variant.sh) on the per-kernel profile of C3 256^3
python -m pytest tests/test_gpu_parity.py tests/test_gpu_00_bench_configs.py -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/r2_gputest5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gputest5.log
for v in default ${VARIANTS:-tmapf1 tmapf3 notma} default; do
  if [ $v = default ]; then unset NPSD_B200_LIB; else export NPSD_B200_LIB=$PWD/variants/libnpsd_b200_$v.so; fi
  echo "== $v" >> gpurun_out/r2_ab.log
  python tools/ncu_target.py --iters 5 | grep -E "ortho|update|total" >> gpurun_out/r2_ab.log 2>&1
done
