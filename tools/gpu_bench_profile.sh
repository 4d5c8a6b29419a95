#!/bin/bash
# bench + launch list (timed steps only) for the default workload (run under gpurun)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
# launches: skip the 256 cache-fill appends + 3 warm-up steps x 64 launches; keep 2 timed steps
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|kv_append|combine" -s 448 -c 128 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --eager > /dev/null 2>&1
tail -2 gpurun_out/launches.csv
