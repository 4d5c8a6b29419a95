"""B200 analog of the paper's Table 2: µs per cuMem* call, one process per
configuration so driver state does not leak between rows."""
import ctypes as C
import json
import subprocess
import sys

sys.path.insert(0, ".")

NAMES = ["cuMemAddressReserve", "cuMemCreate", "cuMemMap", "cuMemSetAccess", "cuMemUnmap",
         "cuMemRelease", "cuMemAddressFree", "cuMemSetAccess_batched_per_page",
         "cuMemMap_recycled", "cuMemSetAccess_recycled"]

if len(sys.argv) > 1 and sys.argv[1] == "one":
    from paper_2405_04437_b200._abi import check, lib
    page, n, run = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    out = (C.c_double * 10)()
    check(lib().vattn_vmm_microbench(0, page, n, run, out))
    print(json.dumps(dict(zip(NAMES, [round(x, 2) for x in out]))))
    sys.exit(0)

res = {}
for page_mb, n, run in [(2, 256, 1), (2, 256, 1), (2, 256, 16), (8, 64, 1), (32, 16, 1)]:
    r = subprocess.run([sys.executable, __file__, "one", str(page_mb << 20), str(n), str(run)],
                       capture_output=True, text=True)
    key = f"page{page_mb}MiB_n{n}_run{run}"
    res.setdefault(key, []).append(json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-300:])
print(json.dumps(res, indent=1))
