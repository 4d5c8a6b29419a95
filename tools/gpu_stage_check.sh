# serving config 5 (48 requests, dense proxy): prefetch + speculative eager, then + lazy unmap, then + staged admission
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_manager.py -x -q 2>&1 | tail -1
for v in "" "--lazy-unmap" "--lazy-unmap --stage 8" "--lazy-unmap --stage 32"; do
  echo "== $v"
  timeout 600 python tools/serving_trace.py --mode overlapped --requests 48 --pool-gib 24 --dense-proxy --prefetch 256 \
     --spec-slots 4 --spec-tokens 3072 $v --out gpurun_out/srv_stage 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print({k:(round(d[k],3) if isinstance(d[k],float) else d[k]) for k in ('iterations','tokens_per_s','p50_iteration_ms','p99_iteration_ms','exposed_map_ms_per_iter','exposed_map_ms_p99','exposed_map_ms_max','exposed_map_ms_median','driver_set_access_ms_total','driver_maps_total','exposed_breakdown_ms')})"
done
