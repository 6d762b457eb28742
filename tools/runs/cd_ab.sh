# A/B: update's b read into registers (default) vs staged in the cp.async ring (variants/lib_cd0.so)
for i in 1 2; do for v in "X=1" "NPSD_B200_LIB=variants/lib_cd0.so"; do
  echo "== $v"; env $v timeout 120 python tools/ncu_target.py --iters 5 | grep -E "update|total" | awk '{print $1, $2}' | tr '\n' ' '; echo
done; done
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/gpu_tests.log
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['per_iter_ms'],d['setup_ms'],d['e2e']['value'],d['clocks']);print(d['baselines_same_gpu']['gpu_cg'])"
