timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?; tail -3 gpurun_out/bench.err
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['per_iter_ms'],d['setup_ms'],d['e2e']['value'],d['clocks']);print(d['baselines_same_gpu']);print(d['sequence_c4'])"
