#!/bin/bash
# ncu --set full of one Yi-6B causal prefill launch at 16K and 64K (why long prompts run slower
# per FLOP): L2 hit rate, DRAM traffic, tensor-pipe activity, SM clock.  One GPU.
set -u
mkdir -p gpurun_out/ncu_long
N="ncu --set full --clock-control none --import-source on"
for S in 16384 65536; do
  PF_S=$S timeout 900 $N -k regex:prefill_kernel -s 2 -c 1 -o gpurun_out/ncu_long/prefill_y6_$S -f python tools/prefill_once.py > gpurun_out/ncu_long/$S.log 2>&1
  ncu -i gpurun_out/ncu_long/prefill_y6_$S.ncu-rep --page raw --csv > gpurun_out/ncu_long/prefill_y6_$S.raw.csv 2>/dev/null
  ncu -i gpurun_out/ncu_long/prefill_y6_$S.ncu-rep --page details --csv > gpurun_out/ncu_long/prefill_y6_$S.details.csv 2>/dev/null
  rm -f gpurun_out/ncu_long/prefill_y6_$S.ncu-rep
done
ls -la gpurun_out/ncu_long
