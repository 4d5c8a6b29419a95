#!/bin/bash
# Timelines (trace build) of the prefill kernel with one vs two softmax warps per TMEM lane quarter
VATTN_EXTRA_NVCC=-DVATTN_PF_TRACE python -m paper_2405_04437_b200.build --force > /dev/null
for smw in 4 8; do echo "== VATTN_PF_SMW=$smw"; VATTN_PF_SMW=$smw python tools/prefill_trace2.py; done
python -m paper_2405_04437_b200.build --force > /dev/null
