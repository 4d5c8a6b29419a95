#!/bin/bash
# phys_chunk_groups 2 (4 MiB) vs 4 (8 MiB) vs the paged loop, 128 requests, back to back
mkdir -p gpurun_out/serving_c2
O=gpurun_out/serving_c2/srv
R=128
ST="--prefetch 256 --spec-slots 4 --spec-tokens 3072 --lazy-unmap --stage 32 --hold"
for C in 2 4; do
  timeout 900 python tools/serving_trace.py --mode overlapped --requests $R --dense-proxy --chunk $C --out $O > /dev/null
  timeout 900 python tools/serving_trace.py --mode overlapped --requests $R --dense-proxy $ST --chunk $C --out $O > /dev/null
done
timeout 900 python tools/serving_trace.py --mode paged --requests $R --dense-proxy --out $O > /dev/null
ls gpurun_out/serving_c2
