# Two ranks on ONE GPU (gloo for host collectives): exercises the N>1 bench path, CUDA IPC setup and
# the cross-process fused head gather the way an 8-GPU torchrun job does (timings are not N-GPU numbers).
mkdir -p gpurun_out
export VATTN_BENCH_ONE_GPU=1 VATTN_DIST_BACKEND=gloo
for g in none fused; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 5 --warmup 3 --gather $g > gpurun_out/mp_bench_$g.json 2> gpurun_out/mp_bench_$g.err
echo "gather=$g rc=$?"; grep -i "error\|Traceback" gpurun_out/mp_bench_$g.err | head -3
python -c "import json;d=json.loads(open('gpurun_out/mp_bench_$g.json').read().splitlines()[-1]);print(d.get('head_gather'), d['value'], d['gpu_launches'], d['head_gather_mode'])"
done
