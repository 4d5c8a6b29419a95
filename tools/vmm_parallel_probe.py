import ctypes as C, json, sys
sys.path.insert(0, ".")
from paper_2405_04437_b200._abi import check, lib
for rep in range(2):
    for t in (1, 2, 4, 8, 16):
        out = (C.c_double * 3)()
        check(lib().vattn_vmm_parallel_probe(0, 512, t, out))
        print(json.dumps({"threads": t, "us_per_page": round(out[0], 1), "total_ms": round(out[1], 1), "unmap_us": round(out[2], 1)}), flush=True)
