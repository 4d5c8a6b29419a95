#!/bin/bash
# Physical chunks (phys_chunk_groups 4 = 8 MiB handles) vs 2 MiB handles on the config-5 trace:
# GPU chunk tests, then the serving loop (wall clock, real kernels, GEMM dense proxy) for
# sync / reference-style overlap / staged B200 loop at chunk 1 and 4, and the paged loop.
R=${R:-128}
mkdir -p gpurun_out/serving_chunk
O=gpurun_out/serving_chunk/srv
timeout 600 python -m pytest tests/test_gpu_manager.py -q -x -k "chunk" -p no:cacheprovider 2>&1 | tail -3
ST="--prefetch 256 --spec-slots 4 --spec-tokens 3072 --lazy-unmap --stage 32 --hold"
for C in 1 4; do
  timeout 900 python tools/serving_trace.py --mode sync --requests $R --dense-proxy --chunk $C --out $O | tail -1 | cut -c1-600
  timeout 900 python tools/serving_trace.py --mode overlapped --requests $R --dense-proxy --chunk $C --out $O | tail -1 | cut -c1-600
  timeout 900 python tools/serving_trace.py --mode overlapped --requests $R --dense-proxy $ST --chunk $C --out $O | tail -1 | cut -c1-600
done
timeout 900 python tools/serving_trace.py --mode paged --requests $R --dense-proxy --out $O | tail -1 | cut -c1-600
