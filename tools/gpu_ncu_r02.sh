#!/bin/bash
# Round-2 ncu captures (one GPU): `ncu --set full` of one launch per hot kernel at every contract
# shape (decode L8 shards G=1/2/4/8, Yi-34B shards, Yi-6B 16K prefill, KV append > L2), exported
# to CSV for profiles/ (tools/ncu_summarize.py).  Numbers under ncu are never bench values.
set -u
mkdir -p gpurun_out/ncu
N="ncu --set full --clock-control none --import-source on"
for G in 1 2 4 8; do
  timeout 600 $N -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/ncu/decode_l8_G$G -f python tools/ncu_targets.py decode $G > gpurun_out/ncu/decode_l8_G$G.log 2>&1
  timeout 600 $N -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/ncu/decode_y34_G$G -f python tools/ncu_targets.py y34 $G > gpurun_out/ncu/decode_y34_G$G.log 2>&1
done
timeout 600 $N -k regex:prefill_kernel -s 2 -c 1 -o gpurun_out/ncu/prefill_y6 -f python tools/ncu_targets.py prefill > gpurun_out/ncu/prefill_y6.log 2>&1
timeout 600 $N -k regex:kv_append -s 2 -c 1 -o gpurun_out/ncu/append_4x16k -f python tools/ncu_targets.py append > gpurun_out/ncu/append_4x16k.log 2>&1
for f in gpurun_out/ncu/*.ncu-rep; do
  ncu -i "$f" --page raw --csv > "${f%.ncu-rep}.raw.csv" 2>/dev/null
  ncu -i "$f" --page details --csv > "${f%.ncu-rep}.details.csv" 2>/dev/null
done
ls -la gpurun_out/ncu | head -40
