#!/bin/bash
# BASELINE config 5 on the whole 512-request trace (wall clock, real kernels, dense layers as bf16
# GEMMs sized to the reference IterationModel): sync and reference-style overlap with 2 MiB
# handles and with 8 MiB physical chunks (phys_chunk_groups 4), the staged B200 loop (chunk 4,
# layered and sliced), and the paged-layout loop.  Outputs: gpurun_out/serving512/*.{csv,json}
mkdir -p gpurun_out/serving512
O=gpurun_out/serving512/srv
R=512
ST="--prefetch 256 --spec-slots 4 --spec-tokens 3072 --lazy-unmap --stage 32 --hold"
timeout 1200 python tools/serving_trace.py --mode sync --requests $R --dense-proxy --out $O | cut -c1-300
timeout 1200 python tools/serving_trace.py --mode overlapped --requests $R --dense-proxy --out $O | cut -c1-300
timeout 1200 python tools/serving_trace.py --mode sync --requests $R --dense-proxy --chunk 4 --out $O | cut -c1-300
timeout 1200 python tools/serving_trace.py --mode overlapped --requests $R --dense-proxy --chunk 4 --out $O | cut -c1-300
timeout 1200 python tools/serving_trace.py --mode overlapped --requests $R --dense-proxy $ST --chunk 4 --out $O | cut -c1-300
timeout 1200 python tools/serving_trace.py --mode overlapped --requests $R --dense-proxy $ST --chunk 4 --sliced --out $O | cut -c1-300
timeout 1200 python tools/serving_trace.py --mode paged --requests $R --dense-proxy --out $O | cut -c1-300
ls gpurun_out/serving512
