"""B200 analog of the paper's Table 2: µs per cuMem* call at 2 MiB."""
import ctypes as C
import json
import sys

sys.path.insert(0, ".")
from paper_2405_04437_b200._abi import check, lib

NAMES = ["cuMemAddressReserve", "cuMemCreate", "cuMemMap", "cuMemSetAccess", "cuMemUnmap",
         "cuMemRelease", "cuMemAddressFree", "cuMemSetAccess_batched_per_page"]
res = {}
for run in (1, 4, 16, 64):
    out = (C.c_double * 8)()
    check(lib().vattn_vmm_microbench(0, 2 * 1024 * 1024, 1024, run, out))
    res[f"run{run}"] = dict(zip(NAMES, [round(x, 2) for x in out]))
print(json.dumps(res, indent=1))
