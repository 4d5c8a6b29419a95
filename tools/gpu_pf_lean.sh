# lean converged MMA issue x exp2 offload (each in its own process) + timelines
for cfg in "0 0" "0 1" "1 1" "2 1"; do set -- $cfg
  echo "== POLY=$1 LEAN=$2"; VATTN_PF_POLY=$1 VATTN_PF_LEAN=$2 python tools/pf_var_ab.py 0 2>&1 | grep -v bit-equal
done
VATTN_EXTRA_NVCC=-DVATTN_PF_TRACE python -m paper_2405_04437_b200.build --force > /dev/null
for cfg in "0 1" "1 1"; do set -- $cfg
  echo "== trace POLY=$1 LEAN=$2"; VATTN_PF_POLY=$1 VATTN_PF_LEAN=$2 timeout 120 python tools/prefill_trace2.py
done
python -m paper_2405_04437_b200.build --force > /dev/null
