"""Resource budget of the hot kernels, read from ptxas's report of the in-tree build (CPU only).

The decode ring relies on 2 CTAs/SM when the grid exceeds one CTA per SM (3 stages, 160
threads): that needs <= 168 registers per thread (10 warps -> 3 per sub-partition of 16K
registers).  A regression to 217 registers once cost 11 % of decode bandwidth; no hot kernel may
spill."""

import re

from conftest import ROOT


def _report():
    from paper_2405_04437_b200.build import LIB, build

    build()
    log = (LIB.parent / "ptxas.log").read_text()
    out = {}
    name = None
    for line in log.splitlines():
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            name = m.group(1)
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and name:
            out.setdefault(name, {})["spill"] = int(m.group(1)) + int(m.group(2))
        m = re.search(r"Used (\d+) registers", line)
        if m and name:
            out.setdefault(name, {})["regs"] = int(m.group(1))
    return out


def test_decode_kernels_fit_two_ctas_per_sm_without_spills():
    rep = _report()
    dec = {k: v for k, v in rep.items() if "decode_kernel" in k}
    assert len(dec) >= 6, sorted(rep)
    for k, v in dec.items():
        assert v["regs"] <= 168, (k, v)
        assert v.get("spill", 0) == 0, (k, v)


def test_prefill_and_append_kernels_do_not_spill():
    rep = _report()
    hot = {k: v for k, v in rep.items() if ("prefill_kernel" in k and "ILi0E" in k) or "kv_append" in k}
    assert hot
    for k, v in hot.items():
        assert v.get("spill", 0) == 0, (k, v)
        assert v["regs"] <= 168, (k, v)     # 320-thread prefill CTA / 256-thread append
