# Eight ranks on ONE GPU (gloo for host collectives): the N = 8 bench path end to end
# (KV-head shards of 1 head, CUDA IPC between 8 processes, fused gather); timings are meaningless.
export VATTN_BENCH_ONE_GPU=1 VATTN_DIST_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --gpus 8 --steps 3 --warmup 3 > gpurun_out/mp8.json 2> gpurun_out/mp8.err
echo "rc=$?"; grep -iE "error|Traceback" gpurun_out/mp8.err | head -5
python -c "import json;d=json.loads(open('gpurun_out/mp8.json').read().splitlines()[-1]);print(d['n_gpus'], d['config']['parallelism'], d.get('head_gather'), d['gpu_launches'])"
