#!/bin/bash
# Config-5, whole 512-request trace: the chunked (8 MiB) loops and the paged loop, back to back
mkdir -p gpurun_out/serving512b
O=gpurun_out/serving512b/srv
R=512
ST="--prefetch 256 --spec-slots 4 --spec-tokens 3072 --lazy-unmap --stage 32 --hold"
timeout 1200 python tools/serving_trace.py --mode overlapped --requests $R --dense-proxy --chunk 4 --out $O | cut -c1-200
timeout 1200 python tools/serving_trace.py --mode sync --requests $R --dense-proxy --chunk 4 --out $O | cut -c1-200
timeout 1200 python tools/serving_trace.py --mode overlapped --requests $R --dense-proxy $ST --chunk 4 --sliced --out $O | cut -c1-200
timeout 1200 python tools/serving_trace.py --mode paged --requests $R --dense-proxy --out $O | cut -c1-200
