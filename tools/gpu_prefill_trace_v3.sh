#!/bin/bash
# Timeline (trace build) of the v3 prefill kernel (one tile per CTA, double-buffered S / P)
VATTN_EXTRA_NVCC=-DVATTN_PF_TRACE python -m paper_2405_04437_b200.build --force > /dev/null
echo "== VATTN_PF_V3=1"; VATTN_PF_V3=1 timeout 120 python tools/prefill_trace2.py
python -m paper_2405_04437_b200.build --force > /dev/null
