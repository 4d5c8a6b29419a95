mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_manager.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
timeout 900 python tools/growth_probe.py 2>&1 | grep -v "^$" | sed 's/bursts_us_per_call.*//'
timeout 600 python tools/serving_trace.py --mode overlapped --requests 48 --pool-gib 24 --dense-proxy --prefetch 256 --spec-slots 4 --spec-tokens 3072 --out gpurun_out/srv_pf 2>&1 | tail -5
