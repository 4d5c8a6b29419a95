#!/bin/bash
# Timelines (trace build) of the single-CTA vs the CTA-pair prefill kernel (leader CTA of head 0)
VATTN_EXTRA_NVCC=-DVATTN_PF_TRACE python -m paper_2405_04437_b200.build --force > /dev/null
for m in 0 1; do echo "== VATTN_PF_PAIR=$m"; VATTN_PF_PAIR=$m timeout 120 python tools/prefill_trace2.py; done
python -m paper_2405_04437_b200.build --force > /dev/null
