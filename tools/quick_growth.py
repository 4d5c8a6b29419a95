"""Run only bench.extra_decode_growth (exposed map ms/iter under decode growth) and print it."""
import json, sys
sys.path.insert(0, ".")
import bench
print(json.dumps(bench.extra_decode_growth(0), indent=1))
