#!/bin/bash
# compute-sanitizer passes over the GPU suite (run under gpurun).  memcheck over everything;
# racecheck / synccheck over the kernel parity files (slow).  initcheck is not used: it does not
# see TMA (async-proxy) stores, so it reports every prefill output as uninitialised.
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --target-processes all --print-limit 20 \
    --log-file gpurun_out/memcheck.%p.log python -m pytest tests -m gpu -q -p no:cacheprovider \
    > gpurun_out/memcheck_pytest.log 2>&1
echo "memcheck rc=$?"; tail -1 gpurun_out/memcheck_pytest.log; tail -qn 1 gpurun_out/memcheck.*.log
for t in racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $t --print-limit 10 --log-file gpurun_out/$t.log \
      python -m pytest tests/test_gpu_kernels.py tests/test_gpu_prefill.py -q -p no:cacheprovider -k "not serving" \
      > gpurun_out/${t}_pytest.log 2>&1
  echo "$t rc=$?"; tail -1 gpurun_out/${t}_pytest.log; tail -1 gpurun_out/$t.log
done
