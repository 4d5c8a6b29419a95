"""Small-grid decode: bench.py's l8_shards (32-layer graph-replayed step at the G = 1/2/4/8 shard
shapes) and long_decode extras, for A/B of decode changes (e.g. VATTN_DEC_CLUSTER=0/1)."""
import json, os, sys
sys.path.insert(0, ".")
import bench
out = {"cluster_env": os.environ.get("VATTN_DEC_CLUSTER", "default")}
out["l8_shards"] = {k: round(v["ms_per_step"], 4) for k, v in bench.extra_l8_shards(0).items()}
ld = bench.extra_long_decode(0) if hasattr(bench, "extra_long_decode") else {}
out["long_decode_us"] = {k: round(v["us"], 2) for k, v in ld.items() if isinstance(v, dict) and "us" in v}
print(json.dumps(out))
