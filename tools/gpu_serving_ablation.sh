# config-5 serving, 128 requests: staged + lazy with / without holding the prefetch worker during launches; paged reference
for v in "--mode overlapped --prefetch 256 --spec-slots 4 --spec-tokens 3072 --lazy-unmap --stage 32" \
         "--mode overlapped --prefetch 256 --spec-slots 4 --spec-tokens 3072 --lazy-unmap --stage 32 --hold" "--mode paged"; do
  echo "== $v"
  timeout 900 python tools/serving_trace.py $v --requests 128 --pool-gib 40 --dense-proxy 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(d.get(k,0),2) for k in ('iterations','tokens_per_s','kernel_ms_total','exposed_map_ms_per_iter','exposed_map_ms_p99','driver_set_access_ms_total')}, 'kernel ms/iter', round(d['kernel_ms_total']/d['iterations'],2))"
done
