# HEAD verification + round-1 profile set v13: gpu tests, smoke, bench, then ncu captures
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/gpu_tests.log
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['per_iter_ms'],d['setup_ms'],d['e2e']['value'],d['clocks'])"
bash tools/runs/profiles_v13.sh
