timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/gpu_tests.log
for v in "NPSD_COARSE_OLD=1" "NPSD_COARSE_ZC=8" "NPSD_COARSE_ZC=4"; do
  env $v timeout 300 python bench.py --no-cpu-baseline --no-sequence --steps 5 > gpurun_out/b_$v.json 2>gpurun_out/b_$v.err; echo "$v $?"
  python -c "import json,sys;d=json.load(open('gpurun_out/b_$v.json'));print(round(d['value'],3),round(d['per_iter_ms'],4),{k:round(v*1e3,1) for k,v in d['kernel_ms'].items()})"
done
