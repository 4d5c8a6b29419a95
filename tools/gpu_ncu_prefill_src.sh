#!/bin/bash
# ncu --set full with source correlation for the Y6 16K prefill kernel (one launch), exported
# as per-SASS-instruction stall samples (source page) + raw metrics.  Run under gpurun.
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 2 -c 1 \
  -o gpurun_out/ncu/prefill_src -f python tools/ncu_targets.py prefill > gpurun_out/ncu/prefill_src.log 2>&1
ncu -i gpurun_out/ncu/prefill_src.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/prefill_src.sass.csv 2>&1
ncu -i gpurun_out/ncu/prefill_src.ncu-rep --page details --csv > gpurun_out/ncu/prefill_src.details.csv 2>&1
ncu -i gpurun_out/ncu/prefill_src.ncu-rep --page raw --csv > gpurun_out/ncu/prefill_src.raw.csv 2>&1
ls -la gpurun_out/ncu
