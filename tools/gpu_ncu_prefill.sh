#!/bin/bash
# one ncu --set full capture of the tcgen05 prefill kernel at Yi-6B 16K (BASELINE config 3)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 2 -c 1 \
    -o gpurun_out/prof_prefill python tools/prefill_once.py > gpurun_out/ncu_prefill.log 2>&1
tail -2 gpurun_out/ncu_prefill.log
