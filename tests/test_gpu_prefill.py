"""GPU parity of the tcgen05 causal prefill kernel against the fp32 CPU oracle.

Tolerance (north_star): max|o - o_ref| / max|o_ref| <= 2e-2 (bf16 in, fp32 accumulate)."""

import pytest
import torch

from oracle.attention import max_rel_err, prefill_ref

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch.device("cuda")


CASES = [
    # n_q, kv_len, Hq, Hkv, causal, slot, slots
    (256, 256, 8, 1, True, 0, 1),          # one CTA pair, MHA-in-group
    (384, 384, 32, 4, True, 1, 2),         # partial second pair, Y6 GQA group 8
    (1000, 1000, 56, 8, True, 0, 1),       # ragged, Yi-34B group 7
    (200, 1224, 32, 8, True, 2, 3),        # chunked prefill: q_off = 1024
    (129, 1, 8, 2, True, 0, 1),            # kv shorter than the query block (rows see nothing)
    (300, 700, 16, 4, False, 0, 1),        # non-causal
    (2048, 2048, 32, 4, True, 0, 1),
    # <= 128 query rows (row tiling, tile B empty) and an even GQA group; the multi-tile cases
    # above with an even group run the head-pair tiling (two query heads per CTA)
    (1, 1, 8, 4, True, 0, 1),
    (77, 900, 32, 8, True, 1, 2),          # chunk over a longer prefix
    (128, 128, 32, 4, False, 0, 1),
    (100, 50, 8, 2, True, 0, 1),           # rows that see no key
    (300, 100, 8, 2, True, 0, 1),          # head pairs with rows that see no key
    (64, 3000, 56, 8, True, 0, 1),         # odd group (7): row tiles
]


@pytest.mark.parametrize("d", [128, 64])
@pytest.mark.parametrize("case", CASES, ids=[str(i) for i in range(len(CASES))])
def test_prefill_raw_matches_oracle(case, d):
    from paper_2405_04437_b200.attention import prefill_attention_raw

    dev = _cuda()
    n_q, kv_len, hq, hkv, causal, slot, slots = case
    gen = torch.Generator().manual_seed(11)
    L = (kv_len + 127) // 128 * 128 + 128
    k = torch.randn(slots, L, hkv, d, generator=gen).to(torch.bfloat16)
    v = torch.randn(slots, L, hkv, d, generator=gen).to(torch.bfloat16)
    k[:, kv_len:] = float("nan")          # rows past kv_len must never be read into the result
    v[:, kv_len:] = float("nan")
    q = torch.randn(n_q, hq, d, generator=gen).to(torch.bfloat16)
    ref = prefill_ref(q, k[slot, :kv_len], v[slot, :kv_len], causal=causal)
    out = prefill_attention_raw(q.to(dev), k.to(dev), v.to(dev), slot, kv_len, causal=causal)
    torch.cuda.synchronize()
    out = out.cpu()
    assert torch.isfinite(out.float()).all()
    err = max_rel_err(out, ref)
    assert err <= TOL, err


def test_prefill_tiles_without_keys_write_exact_zeros():
    """Bottom-right causal alignment with kv_len < n_q: query rows that see no key output 0
    (flash-attn convention).  A tile with no keys must not stage its zeros in its Q buffer (the
    Q load may still be landing there): many heads and repeats to widen the race window."""
    from paper_2405_04437_b200.attention import prefill_attention_raw

    dev = _cuda()
    gen = torch.Generator().manual_seed(5)
    n_q, kv_len, hq, hkv = 129, 1, 64, 8
    k = torch.randn(1, 128, hkv, 128, generator=gen).to(torch.bfloat16).to(dev)
    v = torch.randn(1, 128, hkv, 128, generator=gen).to(torch.bfloat16).to(dev)
    q = torch.randn(n_q, hq, 128, generator=gen).to(torch.bfloat16).to(dev)
    for _ in range(20):
        out = prefill_attention_raw(q, k, v, 0, kv_len, causal=True)
        torch.cuda.synchronize()
        assert torch.count_nonzero(out[:128]).item() == 0
        # the last row sees key 0 only: its output is V row 0 of its KV head
        ref = v[0, 0].repeat_interleave(hq // hkv, dim=0)
        assert torch.equal(out[128], ref)


def test_prefill_full_size_y6_sampled_heads():
    """BASELINE config 3 at full size (16K causal, 32 Q / 4 KV heads): heads checked against
    the oracle on CPU (2 of 32), all heads checked for finiteness."""
    from paper_2405_04437_b200.attention import prefill_attention_raw

    dev = _cuda()
    S, hq, hkv = 16384, 32, 4
    g = torch.Generator(device=dev).manual_seed(3)
    k = torch.randn(1, S, hkv, 128, generator=g, device=dev, dtype=torch.bfloat16)
    v = torch.randn(1, S, hkv, 128, generator=g, device=dev, dtype=torch.bfloat16)
    q = torch.randn(S, hq, 128, generator=g, device=dev, dtype=torch.bfloat16)
    out = prefill_attention_raw(q, k, v, 0, S, causal=True)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    for h in (0, 31):
        kv = h // (hq // hkv)
        ref = prefill_ref(q[:, h:h + 1].cpu(), k[0, :, kv:kv + 1].cpu(), v[0, :, kv:kv + 1].cpu())
        assert max_rel_err(out[:, h:h + 1].cpu(), ref) <= TOL


def test_prefill_through_manager_after_append():
    """Append a prompt into a request slot of the virtual cache, then prefill over it."""
    _cuda()
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry
    from paper_2405_04437_b200.attention import kv_append, prefill_attention

    dev = torch.device("cuda")
    g = ModelGeometry(2, 4, 128, 2, max_context=4096, max_batch=2, n_q_heads_total=32)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=2 * 1024 * 1024, pool_bytes=64 * 2 * 1024 * 1024))
    r0, r1 = mgr.alloc_reqid(), mgr.alloc_reqid()
    S = 3000
    lens = [0, 0]
    lens[r1] = S
    assert mgr.step(lens).ok
    gen = torch.Generator().manual_seed(7)
    kn = torch.randn(1, S, 4, 128, generator=gen).to(torch.bfloat16)
    vn = torch.randn(1, S, 4, 128, generator=gen).to(torch.bfloat16)
    q = torch.randn(S, 32, 128, generator=gen).to(torch.bfloat16)
    kv_append(mgr, 1, kn.to(dev), vn.to(dev), torch.zeros(1, dtype=torch.int32, device=dev),
              torch.tensor([r1], dtype=torch.int32, device=dev))
    out = prefill_attention(mgr, 1, q.to(dev), r1)
    torch.cuda.synchronize()
    ref = prefill_ref(q, kn[0], vn[0])
    assert max_rel_err(out.cpu(), ref) <= TOL
    mgr.close()


@pytest.mark.parametrize("block_size", [16, 128, 256])
def test_prefill_paged_matches_contiguous(block_size):
    """The paged-layout comparison kernel computes the same attention as the contiguous one."""
    from paper_2405_04437_b200.attention import prefill_attention_paged, prefill_attention_raw

    dev = _cuda()
    gen = torch.Generator().manual_seed(12)
    S, hq, hkv = 1000, 32, 4
    nb = (S + block_size - 1) // block_size
    k = torch.randn(1, nb * block_size, hkv, 128, generator=gen).to(torch.bfloat16)
    v = torch.randn(1, nb * block_size, hkv, 128, generator=gen).to(torch.bfloat16)
    q = torch.randn(S, hq, 128, generator=gen).to(torch.bfloat16)
    perm = torch.randperm(nb + 5, generator=gen)[:nb]
    kp = torch.randn(nb + 5, block_size, hkv, 128, generator=gen).to(torch.bfloat16)
    vp = torch.randn(nb + 5, block_size, hkv, 128, generator=gen).to(torch.bfloat16)
    kp[perm] = k[0].view(nb, block_size, hkv, 128)
    vp[perm] = v[0].view(nb, block_size, hkv, 128)
    ref = prefill_ref(q, k[0, :S], v[0, :S])
    out_p = prefill_attention_paged(q.to(dev), kp.to(dev), vp.to(dev), perm.to(torch.int32).to(dev), S)
    out_c = prefill_attention_raw(q.to(dev), k.to(dev), v.to(dev), 0, S)
    torch.cuda.synchronize()
    assert max_rel_err(out_p.cpu(), ref) <= TOL
    assert torch.equal(out_p.cpu(), out_c.cpu())


def test_prefill_max_jumps_take_the_rescale_paths():
    """Keys with large norms late in the sequence make the running row max jump by far more than
    2^8 inside a tile's second half and first half: the single-pass softmax must rescale O, l and
    the already-stored P correctly."""
    from paper_2405_04437_b200.attention import prefill_attention_raw

    dev = _cuda()
    gen = torch.Generator().manual_seed(31)
    S, hq, hkv = 1024, 16, 2
    k = torch.randn(1, S, hkv, 128, generator=gen)
    v = torch.randn(1, S, hkv, 128, generator=gen)
    q = torch.randn(S, hq, 128, generator=gen)
    for pos in (200, 300, 357, 700, 1000):      # second halves and first halves of 128-key tiles
        k[0, pos] *= 12.0
    k, v, q = k.to(torch.bfloat16), v.to(torch.bfloat16), q.to(torch.bfloat16)
    ref = prefill_ref(q, k[0], v[0])
    out = prefill_attention_raw(q.to(dev), k.to(dev), v.to(dev), 0, S)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    assert max_rel_err(out.cpu(), ref) <= TOL


def test_tiny_config_serving_loop_on_gpu():
    """BASELINE config 1 geometry (1 layer, 8 Q / 2 KV heads, D 64, 2 MiB pages) through the
    wall-clock Algorithm-1 loop: prefill (tcgen05, D 64) + fused decode on the virtual cache."""
    _cuda()
    from paper_2405_04437_b200.geometry import tiny
    from paper_2405_04437_b200.serving import run

    g = tiny()
    recs = [(0, 128, 5), (0, 400, 3), (1, 300, 4), (2, 200, 2)]
    m = run(recs, g, mode="overlapped", clock="wall", pool_bytes=64 << 20, eager_groups=1)
    s = m.summary()
    assert s["completed_requests"] == 4 and s["generated_tokens"] == 14


@pytest.mark.parametrize("d,rd,inter,n_q,kv_len", [(128, 128, False, 1000, 1000), (128, 64, True, 200, 1224),
                                                   (64, 64, True, 384, 384), (64, 32, False, 129, 700)])
def test_rotary_append_and_prefill_match_oracle(d, rd, inter, n_q, kv_len):
    """Rotary at append (k row i cached rotated at cache_seqlens + i) and inside the tcgen05
    prefill (query row i rotated in shared memory at kv_len - n_q + i) vs the fp32 oracle."""
    from oracle.attention import rotary_ref
    from paper_2405_04437_b200.attention import kv_append_raw, prefill_attention_raw

    dev = _cuda()
    hq, hkv = 16, 4
    gen = torch.Generator().manual_seed(21)
    kn = torch.randn(1, kv_len, hkv, d, generator=gen).to(torch.bfloat16)
    vn = torch.randn(1, kv_len, hkv, d, generator=gen).to(torch.bfloat16)
    q = torch.randn(n_q, hq, d, generator=gen).to(torch.bfloat16)
    ang = torch.arange(2048, dtype=torch.float32)[:, None] / (10000 ** (torch.arange(0, rd, 2) / rd))[None, :]
    cos, sin = ang.cos(), ang.sin()
    L = (kv_len + 127) // 128 * 128 + 128
    kc = torch.zeros(2, L, hkv, d, dtype=torch.bfloat16, device=dev)
    vc = torch.zeros_like(kc)
    kv_append_raw(kc, vc, kn.to(dev), vn.to(dev), torch.zeros(1, dtype=torch.int32, device=dev),
                  torch.tensor([1], dtype=torch.int32, device=dev), rotary_cos=cos.to(dev), rotary_sin=sin.to(dev),
                  rotary_interleaved=inter)
    out = prefill_attention_raw(q.to(dev), kc, vc, 1, kv_len, rotary_cos=cos.to(dev), rotary_sin=sin.to(dev),
                                rotary_interleaved=inter)
    torch.cuda.synchronize()
    pos_k = torch.arange(kv_len, dtype=torch.int32)
    kr = rotary_ref(kn[0], cos, sin, pos_k, inter).to(torch.bfloat16)        # [kv_len, hkv, d]
    assert torch.allclose(kc[1, :kv_len].cpu().float(), kr.float(), rtol=1e-2, atol=1e-2)
    assert torch.equal(vc[1, :kv_len].cpu(), vn[0])
    qr = rotary_ref(q, cos, sin, torch.arange(kv_len - n_q, kv_len, dtype=torch.int32), inter).to(torch.bfloat16)
    ref = prefill_ref(qr, kr, vn[0])
    assert max_rel_err(out.cpu(), ref) <= TOL


def test_rotary_manager_backed_prefill_then_decode():
    """Rotary through the manager (VMM cache): prompt appended rotated, prefill rotates q inside
    the kernel, then the fused decode appends + rotates the next token; both checked vs oracle."""
    from oracle.attention import decode_ref, rotary_ref
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry
    from paper_2405_04437_b200.attention import decode_attention_append, kv_append, prefill_attention

    dev = _cuda()
    g = ModelGeometry(1, 4, 128, 2, max_context=4096, max_batch=2, n_q_heads_total=32)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=2 << 20, pool_bytes=64 << 20))
    r = mgr.alloc_reqid()
    S = 777
    lens = [0, 0]
    lens[r] = S + 1
    assert mgr.step(lens).ok
    gen = torch.Generator().manual_seed(22)
    kn = torch.randn(1, S, 4, 128, generator=gen).to(torch.bfloat16)
    vn = torch.randn(1, S, 4, 128, generator=gen).to(torch.bfloat16)
    q = torch.randn(S, 32, 128, generator=gen).to(torch.bfloat16)
    ang = torch.arange(4096, dtype=torch.float32)[:, None] / (10000 ** (torch.arange(0, 128, 2) / 128))[None, :]
    cos, sin = ang.cos(), ang.sin()
    rot = dict(rotary_cos=cos.to(dev), rotary_sin=sin.to(dev))
    idx = torch.tensor([r], dtype=torch.int32, device=dev)
    kv_append(mgr, 0, kn.to(dev), vn.to(dev), torch.zeros(1, dtype=torch.int32, device=dev), idx, **rot)
    out = prefill_attention(mgr, 0, q.to(dev), r, **rot)
    pos = torch.arange(S, dtype=torch.int32)
    kr = rotary_ref(kn[0], cos, sin, pos).to(torch.bfloat16)
    qr = rotary_ref(q, cos, sin, pos).to(torch.bfloat16)
    torch.cuda.synchronize()
    assert max_rel_err(out.cpu(), prefill_ref(qr, kr, vn[0])) <= TOL
    q1 = torch.randn(1, 32, 128, generator=gen).to(torch.bfloat16)
    k1 = torch.randn(1, 4, 128, generator=gen).to(torch.bfloat16)
    v1 = torch.randn(1, 4, 128, generator=gen).to(torch.bfloat16)
    o1 = decode_attention_append(mgr, 0, q1.to(dev), k1.to(dev), v1.to(dev),
                                 torch.tensor([S], dtype=torch.int32, device=dev), idx, **rot)
    p1 = torch.tensor([S], dtype=torch.int32)
    kc = torch.cat([kr, rotary_ref(k1, cos, sin, p1).to(torch.bfloat16)], 0).unsqueeze(0)
    vc = torch.cat([vn[0], v1], 0).unsqueeze(0)
    ref = decode_ref(rotary_ref(q1, cos, sin, p1).to(torch.bfloat16), kc, vc, torch.tensor([S + 1], dtype=torch.int32))
    torch.cuda.synchronize()
    assert max_rel_err(o1.cpu(), ref) <= TOL
    mgr.close()


@pytest.mark.parametrize("d", [128, 64])
def test_varlen_prefill_equals_per_request_prefill(d):
    """One launch over several requests (packed queries, ragged lengths, chunked-prefill offsets,
    an empty request) is bit-identical to per-request launches and within tolerance of the oracle."""
    from paper_2405_04437_b200.attention import prefill_attention_raw, prefill_attention_varlen_raw

    dev = _cuda()
    hq, hkv = 16, 4
    q_lens = [300, 1, 0, 1000, 129, 256]
    kv_lens = [300, 700, 5, 1000, 2000, 256]
    slots = [2, 0, 1, 4, 3, 5]
    gen = torch.Generator().manual_seed(31)
    L = 2048 + 128
    k = torch.randn(6, L, hkv, d, generator=gen).to(torch.bfloat16)
    v = torch.randn(6, L, hkv, d, generator=gen).to(torch.bfloat16)
    q = torch.randn(sum(q_lens), hq, d, generator=gen).to(torch.bfloat16)
    kd, vd, qd = k.to(dev), v.to(dev), q.to(dev)
    out = prefill_attention_varlen_raw(qd, kd, vd, q_lens, slots, kv_lens)
    torch.cuda.synchronize()
    o = 0
    for m, kl, sl in zip(q_lens, kv_lens, slots):
        if m:
            one = prefill_attention_raw(qd[o:o + m].contiguous(), kd, vd, sl, kl)
            torch.cuda.synchronize()
            # a lone launch on a grid below half the SMs with >= 16 KV tiles splits its KV range
            # (split-KV, a different fp32 summation); every other launch is bit-identical
            split = (kl + 127) // 128 >= 16 and hq * ((m + 255) // 256) * 2 <= torch.cuda.get_device_properties(dev).multi_processor_count
            if split:
                assert max_rel_err(one.cpu(), out[o:o + m].float().cpu()) <= 1e-2
            else:
                assert torch.equal(out[o:o + m].cpu(), one.cpu())
            ref = prefill_ref(q[o:o + m], k[sl, :kl], v[sl, :kl])
            assert max_rel_err(out[o:o + m].cpu(), ref) <= TOL
        o += m


def test_varlen_prefill_manager_backed():
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry
    from paper_2405_04437_b200.attention import kv_append, prefill_attention, prefill_attention_varlen

    dev = _cuda()
    g = ModelGeometry(1, 4, 128, 2, max_context=4096, max_batch=4, n_q_heads_total=32)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=2 << 20, pool_bytes=128 << 20))
    rids = [mgr.alloc_reqid() for _ in range(3)]
    lens = [0] * 4
    prompts = [500, 3000, 64]
    for r, n in zip(rids, prompts):
        lens[r] = n
    assert mgr.step(lens).ok
    gen = torch.Generator(device=dev).manual_seed(5)
    zero = torch.zeros(1, dtype=torch.int32, device=dev)
    for r, n in zip(rids, prompts):
        kn = torch.randn(1, n, 4, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        kv_append(mgr, 0, kn, kn * 0.5, zero, torch.tensor([r], dtype=torch.int32, device=dev))
    q = torch.randn(sum(prompts), 32, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    out = prefill_attention_varlen(mgr, 0, q, prompts, rids)
    o = 0
    for r, n in zip(rids, prompts):
        one = prefill_attention(mgr, 0, q[o:o + n].contiguous(), r)
        torch.cuda.synchronize()
        assert torch.equal(out[o:o + n], one)
        o += n
    mgr.close()


_HEADPAIR_CHILD = r"""
import sys, json, torch
sys.path.insert(0, ".")
from paper_2405_04437_b200.attention import prefill_attention_raw
from oracle.attention import max_rel_err, prefill_ref
dev = torch.device("cuda")
out = {}
for n_q, kv, hq, hkv, causal in ((1000, 1000, 32, 8, True), (512, 2048, 16, 2, True), (384, 384, 8, 4, False)):
    g = torch.Generator().manual_seed(n_q + kv)
    k = torch.randn(1, kv + 128, hkv, 128, generator=g).to(torch.bfloat16)
    v = torch.randn(1, kv + 128, hkv, 128, generator=g).to(torch.bfloat16)
    q = torch.randn(n_q, hq, 128, generator=g).to(torch.bfloat16)
    o = prefill_attention_raw(q.to(dev), k.to(dev), v.to(dev), 0, kv, causal=causal).cpu()
    ref = prefill_ref(q, k[0, :kv], v[0, :kv], causal=causal)
    out[f"{n_q}_{kv}_{hq}_{hkv}_{causal}"] = [max_rel_err(o, ref), o.view(torch.int16).to(torch.int64).sum().item(),
                                               (o.view(torch.int16).to(torch.int64) * torch.arange(o.numel()).view_as(o).remainder(997)).sum().item()]
print("RESULT " + json.dumps(out))
"""


def test_prefill_head_pair_tiling_matches_row_tiling():
    """The two single-request tilings (VATTN_PF_HEADPAIR=0: two consecutive 128-row tiles of one
    head per CTA; =1: the same 128 rows of two query heads of one GQA group) run each tile's
    arithmetic in the same order, so their outputs are bit-identical; both are within the
    oracle tolerance on multi-tile prompts (causal, chunked, non-causal)."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    _cuda()
    root = Path(__file__).resolve().parents[1]
    res = {}
    for mode in ("0", "1"):
        r = subprocess.run([sys.executable, "-c", _HEADPAIR_CHILD], cwd=root, capture_output=True, text=True,
                           timeout=600, env=dict(os.environ, VATTN_PF_HEADPAIR=mode))
        line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
        assert line, r.stderr[-2000:]
        res[mode] = json.loads(line[0][7:])
    for key, (err, s1, s2) in res["1"].items():
        assert err <= TOL, (key, err)
        assert [s1, s2] == res["0"][key][1:], key


_EARLYPV_CHILD = r"""
import sys, json, torch
sys.path.insert(0, ".")
from paper_2405_04437_b200.attention import prefill_attention_raw
from oracle.attention import max_rel_err, prefill_ref
dev = torch.device("cuda")
out = {}
# (n_q, kv, hq, hkv, causal, spikes): spikes = key rows whose scores jump far above the running
# max (> 2^8 in the exp2 domain) - in the second half of a later tile (the rare path where keys
# 0..63 of P were already released at the old max) and in a first half (two-pass path)
for n_q, kv, hq, hkv, causal, spikes in ((1000, 1000, 32, 8, True, ()), (512, 2048, 16, 2, True, (1800, 1930)),
                                         (384, 384, 8, 4, False, (200, 330)), (700, 700, 8, 2, True, (640, 200))):
    g = torch.Generator().manual_seed(n_q + kv)
    k = torch.randn(1, kv + 128, hkv, 128, generator=g)
    v = torch.randn(1, kv + 128, hkv, 128, generator=g).to(torch.bfloat16)
    q = torch.randn(n_q, hq, 128, generator=g)
    for r in spikes:
        k[0, r] = q[-1].view(hkv, hq // hkv, 128).mean(1) * 4.0
    k = k.to(torch.bfloat16)
    q = q.to(torch.bfloat16)
    o = prefill_attention_raw(q.to(dev), k.to(dev), v.to(dev), 0, kv, causal=causal).cpu()
    ref = prefill_ref(q, k[0, :kv], v[0, :kv], causal=causal)
    out[f"{n_q}_{kv}_{hq}_{hkv}_{causal}_{len(spikes)}"] = [max_rel_err(o, ref), bool(torch.isfinite(o.float()).all())]
print("RESULT " + json.dumps(out))
"""


def test_prefill_early_pv_matches_oracle():
    """VATTN_PF_EARLYPV=1 (keys 0..63 of P go to the tensor core before keys 64..127 are done):
    within the oracle tolerance, including rows whose running max jumps in the second half of a
    tile after the first half was already released (O is rescaled once that PV retired)."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    _cuda()
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, "-c", _EARLYPV_CHILD], cwd=root, capture_output=True, text=True,
                       timeout=600, env=dict(os.environ, VATTN_PF_EARLYPV="1"))
    line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
    assert line, r.stderr[-2000:]
    for key, (err, finite) in json.loads(line[0][7:]).items():
        assert finite and err <= TOL, (key, err)


_SPLITKV_CHILD = r"""
import sys, json, torch
sys.path.insert(0, ".")
from paper_2405_04437_b200.attention import prefill_attention_raw
from oracle.attention import max_rel_err, prefill_ref
dev = torch.device("cuda")
out = {}
for n_q, kv, hq, hkv, causal, d in ((128, 4000, 32, 8, True, 128), (1, 3000, 8, 2, True, 128),
                                    (200, 2500, 16, 4, False, 128), (300, 100, 8, 2, True, 128),
                                    (128, 16384, 32, 4, True, 128), (96, 2100, 8, 4, True, 64)):
    g = torch.Generator().manual_seed(n_q * 3 + kv)
    k = torch.randn(1, kv + 128, hkv, d, generator=g).to(torch.bfloat16)
    v = torch.randn(1, kv + 128, hkv, d, generator=g).to(torch.bfloat16)
    k[:, kv:] = float("nan")
    v[:, kv:] = float("nan")
    q = torch.randn(n_q, hq, d, generator=g).to(torch.bfloat16)
    o = prefill_attention_raw(q.to(dev), k.to(dev), v.to(dev), 0, kv, causal=causal).cpu()
    ref = prefill_ref(q, k[0, :kv], v[0, :kv], causal=causal)
    out[f"{n_q}_{kv}_{hq}_{hkv}_{causal}_{d}"] = [max_rel_err(o, ref), bool(torch.isfinite(o.float()).all())]
print("RESULT " + json.dumps(out))
"""


@pytest.mark.parametrize("mode", ["0", "1", "3", "7"])
def test_prefill_split_kv_matches_oracle(mode):
    """Split-KV prefill (VATTN_PF_SPLITKV: 0 off, 1 automatic - on for grids below half the SMs
    with >= 16 KV tiles -, N forced): each CTA runs a slice of the KV tiles, writes fp32 partials
    and a log2-domain LSE, and the combine kernel merges them.  Within the oracle tolerance for
    chunks over long prefixes, a single query row, non-causal, rows that see no key (their
    splits are all empty) and D 64; NaN rows past kv_len are never read."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    _cuda()
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, "-c", _SPLITKV_CHILD], cwd=root, capture_output=True, text=True,
                       timeout=600, env=dict(os.environ, VATTN_PF_SPLITKV=mode))
    line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
    assert line, r.stderr[-2000:]
    for key, (err, finite) in json.loads(line[0][7:]).items():
        assert finite and err <= TOL, (key, err)
