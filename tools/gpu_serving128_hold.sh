# config-5 serving, first 128 requests: the staged + lazy variant with and without the held
# prefetch worker, against the paged-layout loop, interleaved twice on one box
mkdir -p gpurun_out/serving128h
for rep in 1 2; do
for v in "--mode overlapped --prefetch 256 --spec-slots 4 --spec-tokens 3072 --lazy-unmap --stage 32" \
         "--mode overlapped --prefetch 256 --spec-slots 4 --spec-tokens 3072 --lazy-unmap --stage 32 --hold" "--mode paged"; do
  echo "== rep $rep $v"
  timeout 900 python tools/serving_trace.py $v --requests 128 --pool-gib 40 --dense-proxy --out gpurun_out/serving128h/srv_r$rep 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:(round(d[k],3) if isinstance(d[k],float) else d[k]) for k in ('iterations','tokens_per_s','exposed_map_ms_per_iter','exposed_map_ms_p99','compute_ms_per_iter','driver_set_access_ms_total') if k in d})"
done
done
