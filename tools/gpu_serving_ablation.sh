# config-5 serving, 48 requests: staged admission with and without speculative eager (hints alone)
for v in "--prefetch 256 --spec-slots 4 --spec-tokens 3072 --lazy-unmap --stage 32 --hold" \
         "--prefetch 256 --lazy-unmap --stage 32 --hold" "--prefetch 64 --lazy-unmap --stage 32 --hold"; do
  echo "== $v"
  timeout 900 python tools/serving_trace.py --mode overlapped $v --requests 48 --pool-gib 24 --dense-proxy 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(d.get(k,0),2) for k in ('iterations','tokens_per_s','exposed_map_ms_per_iter','exposed_map_ms_p99','driver_set_access_ms_total','driver_maps_total')}, 'kernel ms/iter', round(d['kernel_ms_total']/d['iterations'],2))"
done
