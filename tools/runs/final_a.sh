timeout 800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/gpu_tests.log
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['per_iter_ms'],d['setup_ms'],d['e2e']['value'],d['clocks'])"
timeout 600 python bench.py --slab --no-cpu-baseline --no-sequence > gpurun_out/bench_slab.json 2> gpurun_out/bench_slab.err; echo slab $?; head -c 600 gpurun_out/bench_slab.json
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref $?; head -c 300 gpurun_out/bench_ref.json
