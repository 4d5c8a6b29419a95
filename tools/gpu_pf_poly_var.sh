# POLY x VAR A/B (each in its own process)
for cfg in "0 0" "0 3" "0 19" "1 3" "1 19" "2 19"; do set -- $cfg
  echo "== POLY=$1 VAR=$2"; VATTN_PF_POLY=$1 VATTN_PF_VAR=$2 python tools/pf_var_ab.py $2 2>&1 | grep -v bit-equal
done
