"""Run one bench.py extra by name on cuda:0 and print its JSON (e.g. l8_shards, decode_growth)."""
import json, sys
sys.path.insert(0, ".")
import bench
print(json.dumps(getattr(bench, "extra_" + sys.argv[1])(0), indent=1))
