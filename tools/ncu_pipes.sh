#!/bin/bash
# usage: tools/ncu_pipes.sh <name> <kernel-regex> <cmd...>   (run under gpurun)
name=$1; kre=$2; shift 2
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:$kre -s 2 -c 1 --csv "$@" 2>/dev/null | grep -E "^\"[0-9]" | awk -F'","' -v n=$name '{print n, $(NF-2), $NF}'
