#!/bin/bash
# ncu --set full of the Yi-6B 16K prefill (config 3) under both single-request tilings: head pairs
# (the default) and row tiles (VATTN_PF_HEADPAIR=0).  One GPU; numbers under ncu are never bench
# values.  Summarise with: python tools/ncu_summarize.py gpurun_out/ncu_hp r02c
set -u
mkdir -p gpurun_out/ncu_hp
N="ncu --set full --clock-control none --import-source on"
timeout 600 $N -k regex:prefill_kernel -s 2 -c 1 -o gpurun_out/ncu_hp/prefill_y6_heads -f python tools/ncu_targets.py prefill > gpurun_out/ncu_hp/heads.log 2>&1
VATTN_PF_HEADPAIR=0 timeout 600 $N -k regex:prefill_kernel -s 2 -c 1 -o gpurun_out/ncu_hp/prefill_y6_rows -f python tools/ncu_targets.py prefill > gpurun_out/ncu_hp/rows.log 2>&1
for f in gpurun_out/ncu_hp/*.ncu-rep; do
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}.raw.csv" 2>/dev/null
  ncu -i "$f" --page details --csv > "${f%.ncu-rep}.details.csv" 2>/dev/null
done
ls -la gpurun_out/ncu_hp
