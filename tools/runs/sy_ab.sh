# A/B: ortho/update tile rows 16 (default build) vs 8 (variants/lib_sy8.so)
for i in 1 2; do for v in "X=1" "NPSD_B200_LIB=variants/lib_sy8.so"; do
  echo "== $v"; env $v timeout 120 python tools/ncu_target.py --iters 5 | grep -E "ortho|update|total" | awk '{print $1, $2}' | tr '\n' ' '; echo
done; done
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/gpu_tests.log
for v in "X=1" "NPSD_B200_LIB=variants/lib_sy8.so"; do
  env $v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$v.json 2> gpurun_out/bench.err; echo "$v bench $?"
  python -c "import json;d=json.load(open('gpurun_out/bench_$v.json'));print(d['value'],d['per_iter_ms'],d['setup_ms'],d['e2e']['value'],d['roofline'])"
done
