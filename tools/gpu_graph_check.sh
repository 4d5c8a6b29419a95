mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gather.py tests/test_gpu_manager.py -x -q 2>&1 | tail -2
timeout 300 python tools/decode_split_sweep.py
timeout 600 python bench.py --no-extras > gpurun_out/bench_graph.json 2> gpurun_out/bench_graph.err; tail -2 gpurun_out/bench_graph.err
python -c "import json;d=json.loads(open('gpurun_out/bench_graph.json').read().splitlines()[-1]);print('graph', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
timeout 600 python bench.py --no-extras --eager > gpurun_out/bench_eager.json 2> gpurun_out/bench_eager.err; tail -2 gpurun_out/bench_eager.err
python -c "import json;d=json.loads(open('gpurun_out/bench_eager.json').read().splitlines()[-1]);print('eager', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
