#!/bin/bash
# BASELINE config 5 on the whole 512-request trace (wall clock, real kernels, dense layers as bf16
# GEMMs sized to the reference IterationModel): sync, reference-style overlap, the staged B200
# loop (layered and sliced), and the paged-layout loop.  Outputs: gpurun_out/serving512/*.{csv,json}
mkdir -p gpurun_out/serving512
O=gpurun_out/serving512/srv
R=512
timeout 900 python tools/serving_trace.py --mode sync --requests $R --dense-proxy --out $O
timeout 900 python tools/serving_trace.py --mode overlapped --requests $R --dense-proxy --out $O
timeout 900 python tools/serving_trace.py --mode overlapped --requests $R --dense-proxy --prefetch 256 --spec-slots 4 --spec-tokens 3072 --lazy-unmap --stage 32 --hold --out $O
timeout 900 python tools/serving_trace.py --mode overlapped --requests $R --dense-proxy --prefetch 256 --spec-slots 4 --spec-tokens 3072 --lazy-unmap --stage 32 --hold --sliced --out $O
timeout 900 python tools/serving_trace.py --mode paged --requests $R --dense-proxy --out $O
ls gpurun_out/serving512
