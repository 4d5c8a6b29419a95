"""The C ABI from C: examples/c_host.c (gcc, linked against libvattn.so, shadow backend) makes the
reference API calls (alloc_reqid / step / free_reqid / eager_prepare / reclaim, manager.py:163-372)
and the Python facade replays them; every printed result must agree, including the status code
of a double free (DoubleFreeError, manager.py:32)."""

import shutil
import subprocess

import pytest

from conftest import ROOT


def test_c_host_matches_python_facade(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry
    from paper_2405_04437_b200._abi import LIB_PATH, lib
    from paper_2405_04437_b200.errors import DoubleFreeError

    lib()                                   # builds the library if needed
    exe = tmp_path / "c_host"
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", str(ROOT / "include"),
                    str(ROOT / "examples" / "c_host.c"), "-L", str(LIB_PATH.parent), "-lvattn",
                    f"-Wl,-rpath,{LIB_PATH.parent}", "-o", str(exe)], check=True)
    got = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines()

    g = ModelGeometry(2, 2, 64, 2, max_context=8192, max_batch=4)
    m = KVCacheManager(g, ManagerConfig(page_group_size=64 * 1024, pool_bytes=64 << 20, reclaim_threshold=0.1,
                                        pre_create_fraction=1.0, eager_groups=2), backend="shadow")
    want = []
    r0, r1, r2 = m.alloc_reqid(), m.alloc_reqid(), m.alloc_reqid()
    want.append(f"alloc {r0} {r1} {r2}")
    seq = [0] * 4
    seq[r0], seq[r1], seq[r2] = 1000, 3000, 10
    r = m.step(seq)
    want.append(f"step {int(r.ok)} {r.sync_us:.3f}")
    m.free_reqid(r1)
    seq[r1] = 0
    want.append(f"eager {m.eager_prepare():.3f}")
    r3 = m.alloc_reqid()
    want.append(f"realloc {r3}")
    seq[r3], seq[r0], seq[r2] = 500, 1001, 11
    r = m.step(seq)
    want.append(f"step {int(r.ok)} {r.sync_us:.3f}")
    freed, us = m.reclaim()
    want.append(f"reclaim {freed} {us:.3f}")
    c = m._counters()
    want.append(f"counters {c.created} {c.mapped} {c.total_mapped_bytes} {c.eager_slot}")
    m.free_reqid(r3)
    with pytest.raises(DoubleFreeError):
        m.free_reqid(r3)
    want.append("double_free 2")
    m.close()
    assert got == want
