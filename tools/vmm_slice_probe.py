import ctypes as C, json, subprocess, sys
sys.path.insert(0, ".")
if len(sys.argv) > 1:
    from paper_2405_04437_b200._abi import check, lib
    out = (C.c_double * 3)()
    check(lib().vattn_vmm_slice_probe(0, int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), out))
    print(json.dumps({"n": int(sys.argv[1]), "big": int(sys.argv[2]), "extra": int(sys.argv[3]),
                      "map_us": round(out[0], 2), "set_access_us": round(out[1], 1), "unmap_us": round(out[2], 1)}))
    sys.exit(0)
for args in [(256, 0, 0), (256, 0, 1000), (256, 0, 4000), (256, 0, 12000), (256, 0, 0)]:
    r = subprocess.run([sys.executable, __file__, *map(str, args)], capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-300:], flush=True)
