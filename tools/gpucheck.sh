timeout 400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/gpu_tests.log
timeout 120 python tools/ncu_target.py > gpurun_out/target.txt 2>&1; cat gpurun_out/target.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['per_iter_ms'],d['e2e']['value'])"
