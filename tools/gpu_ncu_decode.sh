#!/bin/bash
# one ncu --set full capture of the fused decode kernel inside the default bench (1 GPU)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 100 -c 1 \
    -o gpurun_out/prof_decode_fused python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --eager > gpurun_out/ncu_decode.log 2>&1
tail -1 gpurun_out/ncu_decode.log
ncu --set full --clock-control none --import-source on -k regex:kv_append -s 0 -c 1 \
    -o gpurun_out/prof_append python -c "
import sys; sys.path.insert(0,'.')
import torch
from paper_2405_04437_b200.attention import kv_append_raw
S=16384; dev=torch.device('cuda')
kc=torch.empty(1,S,4,128,device=dev,dtype=torch.bfloat16); vc=torch.empty_like(kc)
kn=torch.randn(1,S,4,128,device=dev,dtype=torch.bfloat16); vn=torch.randn_like(kn)
kv_append_raw(kc,vc,kn,vn,torch.zeros(1,dtype=torch.int32,device=dev)); torch.cuda.synchronize()
" > gpurun_out/ncu_append.log 2>&1
tail -1 gpurun_out/ncu_append.log
