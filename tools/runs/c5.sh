timeout 1200 python bench.py --config C5 --no-cpu-baseline --no-sequence --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5 $?
python -c "import json;d=json.load(open('gpurun_out/bench_c5.json'));print(d['value'],d['per_iter_ms'],d['setup_ms'],d['config']['iterations'],d['iteration_roofline']['frac'],d['e2e']['value']);print(d['baselines_same_gpu']);print(d['identity_weights_same_gpu'])"
tail -3 gpurun_out/bench_c5.err
