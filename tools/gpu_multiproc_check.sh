# Two ranks on ONE GPU (gloo for host collectives): exercises the N>1 bench path, CUDA IPC setup and
# the cross-process fused head gather the way an 8-GPU torchrun job does (timings are not N-GPU numbers).
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gather.py -x -q 2>&1 | tail -2
export VATTN_BENCH_ONE_GPU=1 VATTN_DIST_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 5 --warmup 3 --gather fused > gpurun_out/mp_bench_fused.json 2> gpurun_out/mp_bench_fused.err
echo "rc=$?"; tail -3 gpurun_out/mp_bench_fused.err; cut -c1-600 gpurun_out/mp_bench_fused.json
python -c "import json;d=json.loads(open('gpurun_out/mp_bench_fused.json').read().splitlines()[-1]);print(d.get('head_gather'), d['value'], d['gpu_launches'])"
