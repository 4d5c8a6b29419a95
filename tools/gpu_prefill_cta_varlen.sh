#!/bin/bash
VATTN_EXTRA_NVCC=-DVATTN_PF_TRACE python -m paper_2405_04437_b200.build --force > /dev/null
timeout 120 python tools/prefill_cta_timeline_varlen.py
python -m paper_2405_04437_b200.build --force > /dev/null
