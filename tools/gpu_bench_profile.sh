#!/bin/bash
# bench + launch list + one ncu --set full capture of the decode kernel (run under gpurun)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|kv_append|combine" -c 200 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 100 -c 1 \
    -o gpurun_out/prof_decode python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
