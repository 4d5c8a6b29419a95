"""CPU checks of the attention oracle's internal consistency (oracle/attention.py).

The reference has no attention code, so the oracle is pinned on the GPU against flash-attn
2.8.3 (tests/test_gpu_flash_attn_crosscheck.py).  These CPU tests tie its functions to each
other: the batched equal-length decode used by the CPU baseline equals the per-row restatement,
decode over n tokens equals the last row of a causal prefill over the same n tokens, and the
bottom-right causal alignment matches an explicit triple loop on a tiny case.
"""

import math

import torch

from oracle.attention import (decode_ref, decode_ref_equal, elem_rel_err, err_report, kv_append_ref, max_rel_err,
                              prefill_ref)


def _r(shape, gen):
    return torch.randn(shape, generator=gen).to(torch.bfloat16)


def test_decode_ref_equal_matches_per_row_decode():
    gen = torch.Generator().manual_seed(0)
    q, k, v = _r((11, 8, 64), gen), _r((11, 300, 2, 64), gen), _r((11, 300, 2, 64), gen)
    for n in (1, 37, 300):
        a = decode_ref(q, k, v, torch.full((11,), n, dtype=torch.int32))
        b = decode_ref_equal(q, k, v, n, rows_per_chunk=4)
        assert torch.allclose(a, b, atol=1e-5, rtol=1e-5)
    assert decode_ref_equal(q, k, v, 0).abs().max() == 0


def test_decode_is_last_row_of_causal_prefill():
    gen = torch.Generator().manual_seed(1)
    n, hq, hkv, d = 90, 8, 2, 64
    k, v = _r((n, hkv, d), gen), _r((n, hkv, d), gen)
    qp = _r((n, hq, d), gen)
    pre = prefill_ref(qp, k, v, causal=True)
    dec = decode_ref(qp[-1:], k.unsqueeze(0), v.unsqueeze(0), torch.tensor([n], dtype=torch.int32))
    assert torch.allclose(pre[-1:], dec, atol=1e-5)
    # a 5-row query block over 90 keys: bottom-right alignment -> row i sees keys <= 85 + i
    pre5 = prefill_ref(qp[-5:], k, v, causal=True)
    for i in range(5):
        m = 85 + i + 1
        di = decode_ref(qp[85 + i:86 + i], k.unsqueeze(0), v.unsqueeze(0), torch.tensor([m], dtype=torch.int32))
        assert torch.allclose(pre5[i:i + 1], di, atol=1e-5)


def test_prefill_ref_matches_explicit_loop():
    gen = torch.Generator().manual_seed(2)
    sq, sk, hq, hkv, d = 3, 6, 4, 2, 16
    q, k, v = _r((sq, hq, d), gen), _r((sk, hkv, d), gen), _r((sk, hkv, d), gen)
    got = prefill_ref(q, k, v, causal=True)
    want = torch.zeros(sq, hq, d)
    for i in range(sq):
        for h in range(hq):
            kh = h // (hq // hkv)
            lim = i + sk - sq
            s = torch.tensor([float(q[i, h].float() @ k[j, kh].float()) / math.sqrt(d) for j in range(lim + 1)])
            p = torch.softmax(s, 0)
            want[i, h] = sum(p[j] * v[j, kh].float() for j in range(lim + 1))
    assert torch.allclose(got, want, atol=1e-5)


def test_kv_append_ref_and_metrics():
    gen = torch.Generator().manual_seed(3)
    kc, vc = torch.zeros(3, 10, 2, 8), torch.zeros(3, 10, 2, 8)
    kn, vn = _r((2, 4, 2, 8), gen), _r((2, 4, 2, 8), gen)
    k2, v2 = kv_append_ref(kc, vc, kn, vn, torch.tensor([1, 6]), torch.tensor([2, 0]))
    assert torch.equal(k2[2, 1:5], kn[0].float()) and torch.equal(v2[0, 6:10], vn[1].float())
    assert k2[1].abs().max() == 0
    ref = torch.tensor([1.0, -2.0, 0.0])
    out = torch.tensor([1.0, -2.0, 0.001])
    assert abs(max_rel_err(out, ref) - 0.001 / 2.0) < 1e-9
    assert abs(elem_rel_err(out, ref) - 1.0) < 1e-4        # 0.001 / (0 + 1e-3)
    assert set(err_report(out, ref)) == {"max_rel_err", "elem_rel_err", "elements"}
