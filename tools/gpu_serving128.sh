# config-5 serving trace, first 128 requests, real kernels + dense-layer proxy: sync, reference overlap,
# + prefetch/speculative eager, + lazy unmap + staged admission, and the paged-layout loop
mkdir -p gpurun_out/serving128
for v in "--mode sync" "--mode overlapped" "--mode overlapped --prefetch 256 --spec-slots 4 --spec-tokens 3072" \
         "--mode overlapped --prefetch 256 --spec-slots 4 --spec-tokens 3072 --lazy-unmap --stage 32" "--mode paged"; do
  echo "== $v"
  timeout 900 python tools/serving_trace.py $v --requests 128 --pool-gib 40 --dense-proxy --out gpurun_out/serving128/srv 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:(round(d[k],3) if isinstance(d[k],float) else d[k]) for k in ('iterations','tokens_per_s','exposed_map_ms_per_iter','exposed_map_ms_p99','exposed_map_ms_max','preemptions') if k in d})"
done
