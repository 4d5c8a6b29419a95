"""Layer-sliced layout at the real model shapes (VERDICT r1 "missing 1").

With `ManagerConfig(sliced=True)` the reference keeps two buffers (K, V) whose page-groups span
all layers of their tokens (`kvsim/manager.py:93-96`), i.e. the cache is [B, L, N, H, D] and
one 2 MiB page-group holds 2 MiB / (N * row) tokens: 32 at Llama-3-8B, 17.07 at Yi-34B (TP 1),
136.5 at Yi-34B/8.  A 64-token decode tile can then reach past a row's mapped page-groups, so
the decode kernels load each row's last, partial tile with per-row loads bounded by its length
(kernels.cu, CacheView::tail_guard).  Every length class below is checked against the fp32
oracle for decode, fused append + decode (split and unsplit), and causal prefill.
"""

import pytest
import torch

from oracle.attention import decode_ref, err_report, max_rel_err, prefill_ref

pytestmark = pytest.mark.gpu
MB2 = 2 * 1024 * 1024
TOL = 2e-2


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch.device("cuda")


CASES = {
    # name: (n_layers, hkv_total, hq_total, tp, max_context, lens, layers)
    "llama3_8b": (32, 8, 32, 1, 4096, [1, 31, 32, 33, 63, 64, 65, 1100], [0, 13, 31]),
    "yi34b_tp1": (60, 8, 56, 1, 2048, [1, 17, 18, 34, 35, 69, 700], [0, 59]),
    "yi34b_tp8": (60, 8, 56, 8, 4096, [1, 136, 137, 138, 273, 2000], [7, 59]),
}


@pytest.mark.parametrize("name", list(CASES))
def test_sliced_decode_prefill_match_oracle(name):
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
    from paper_2405_04437_b200.attention import (decode_attention, decode_attention_append, kv_append,
                                                 prefill_attention)
    from paper_2405_04437_b200.geometry import ModelGeometry

    dev = _cuda()
    n_layers, hkv_t, hq_t, tp, ctx, lens, layers = CASES[name]
    B = len(lens)
    g = ModelGeometry(n_layers, hkv_t, 128, 2, max_context=ctx, max_batch=B, tp_degree=tp, n_q_heads_total=hq_t)
    hkv, hq = g.kv_heads_per_worker, g.q_heads_per_worker
    tok_bytes = n_layers * g.per_token_layer_bytes
    groups = sum(-(-(n + 1) * tok_bytes // MB2) for n in lens)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=(2 * groups + 8) * MB2, sliced=True))
    rids = [mgr.alloc_reqid() for _ in range(B)]
    seq_all = [0] * B
    for r, n in zip(rids, lens):
        seq_all[r] = n + 1                       # room for the fused-append token
    assert mgr.step(seq_all).ok
    idx = torch.tensor(rids, dtype=torch.int32, device=dev)
    pos = torch.tensor(lens, dtype=torch.int32, device=dev)
    gen = torch.Generator().manual_seed(7)
    L = max(lens) + 1
    zero = torch.zeros(1, dtype=torch.int32, device=dev)
    report = {}
    for layer in layers:
        k_host = torch.randn(B, L, hkv, 128, generator=gen).to(torch.bfloat16)
        v_host = torch.randn(B, L, hkv, 128, generator=gen).to(torch.bfloat16)
        for b, (r, n) in enumerate(zip(rids, lens)):
            kv_append(mgr, layer, k_host[b:b + 1, :n].to(dev), v_host[b:b + 1, :n].to(dev), zero,
                      torch.tensor([r], dtype=torch.int32, device=dev))
        q = torch.randn(B, hq, 128, generator=gen).to(torch.bfloat16)
        seq = torch.tensor(lens, dtype=torch.int32)
        ref = decode_ref(q, k_host, v_host, seq)
        for splits in (1, 0, 3):
            out = decode_attention(mgr, layer, q.to(dev), pos, idx, num_splits=splits)
            torch.cuda.synchronize()
            rep = err_report(out.cpu(), ref)
            assert rep["max_rel_err"] <= TOL, (name, layer, splits, rep)
            report[(layer, splits)] = rep
        # the cache views see the same rows (strided [B, L, N, H, D] layout)
        kc = mgr.k_cache(layer)
        for b, (r, n) in enumerate(zip(rids, lens)):
            assert torch.equal(kc[r, :n].cpu(), k_host[b, :n])
        # fused append + decode: the new token lands at row lens[b], possibly a new page-group
        k1 = torch.randn(B, hkv, 128, generator=gen).to(torch.bfloat16)
        v1 = torch.randn(B, hkv, 128, generator=gen).to(torch.bfloat16)
        k_ref, v_ref = k_host.clone(), v_host.clone()
        for b, n in enumerate(lens):
            k_ref[b, n], v_ref[b, n] = k1[b], v1[b]
        ref1 = decode_ref(q, k_ref, v_ref, seq + 1)
        out1 = decode_attention_append(mgr, layer, q.to(dev), k1.to(dev), v1.to(dev), pos, idx, num_splits=2)
        torch.cuda.synchronize()
        assert max_rel_err(out1.cpu(), ref1) <= TOL
        # causal prefill of the longest request's rows (tcgen05 kernel, per-call tensor maps)
        b = lens.index(max(lens))
        n = lens[b] + 1
        qp = torch.randn(n, hq, 128, generator=gen).to(torch.bfloat16)
        outp = prefill_attention(mgr, layer, qp.to(dev), rids[b], kv_len=n)
        torch.cuda.synchronize()
        refp = prefill_ref(qp, k_ref[b, :n], v_ref[b, :n])
        assert max_rel_err(outp.cpu(), refp) <= TOL
    mgr.close()
    print(name, {str(k): v for k, v in report.items()})
