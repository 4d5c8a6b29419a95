#!/bin/bash
# A/B of prefill variants (regular build), then per-variant timelines (trace build).  Run under gpurun.
VARS=${VARS:-"0 3 16 19"}
python tools/pf_var_ab.py $VARS
VATTN_EXTRA_NVCC=-DVATTN_PF_TRACE python -m paper_2405_04437_b200.build --force > /dev/null
for v in $VARS; do
  echo "== VATTN_PF_VAR=$v"; VATTN_PF_VAR=$v python tools/prefill_trace2.py
done
python -m paper_2405_04437_b200.build --force > /dev/null
