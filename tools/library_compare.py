import sys, json; sys.path.insert(0, ".")
import bench
print(json.dumps(bench.extra_libraries(0), indent=1))
