"""GPU parity of the sm_100a kernels against the fp32 CPU oracle (oracle/attention.py).

Tolerance (north_star): bf16 inputs, fp32 accumulation, max relative error
max|o - o_ref| / max|o_ref| <= 2e-2.  KV append is byte work: bit-exact.
"""

import pytest
import torch

from oracle.attention import decode_ref, kv_append_ref, max_rel_err

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch.device("cuda")


def _rand(shape, gen, scale=1.0):
    return (torch.randn(shape, generator=gen) * scale).to(torch.bfloat16)


def _mk_cache(slots, L, hkv, d, gen, fill_nan=False):
    k = _rand((slots, L, hkv, d), gen)
    v = _rand((slots, L, hkv, d), gen)
    return k, v


DECODE_CASES = [
    # B, Hq, Hkv, D, seqlens, idx permutation?, splits
    (2, 8, 2, 64, [128, 512], False, 0),                       # config 1 (tiny)
    (2, 8, 2, 64, [128, 512], False, 3),
    (6, 32, 8, 128, [1, 63, 64, 65, 1000, 4096], True, 0),     # L8 shape, ragged
    (6, 32, 8, 128, [1, 63, 64, 65, 1000, 4096], False, 1),
    (6, 32, 8, 128, [1, 63, 64, 65, 1000, 4096], False, 5),
    (3, 56, 8, 128, [8192, 777, 4097], True, 0),                # Y34 group of 7
    (2, 32, 4, 128, [2048, 31], False, 0),                      # Y6 group of 8
    (3, 7, 1, 128, [300, 0, 129], False, 2),                    # Y34/8 shard: 1 KV head, empty row
    (4, 16, 1, 64, [64, 65, 127, 1], True, 0),                  # group of 16
    (1, 32, 8, 128, [8192], False, 64),                         # 64 splits: 4 combine batches
    (2, 32, 8, 128, [8000, 1000], False, 40),                   # row 2: splits 16-39 empty
]


@pytest.mark.parametrize("case", DECODE_CASES, ids=[str(i) for i in range(len(DECODE_CASES))])
def test_decode_raw_matches_oracle(case):
    from paper_2405_04437_b200.attention import decode_attention_raw

    dev = _cuda()
    B, hq, hkv, d, lens, perm, splits = case
    gen = torch.Generator().manual_seed(0)
    L = max(max(lens), 1)
    L = (L + 63) // 64 * 64
    slots = B + 2
    k, v = _mk_cache(slots, L, hkv, d, gen)
    q = _rand((B, hq, d), gen)
    idx = torch.randperm(slots, generator=gen)[:B].to(torch.int32) if perm else torch.arange(B, dtype=torch.int32)
    seq = torch.tensor(lens, dtype=torch.int32)
    ref = decode_ref(q, k, v, seq, idx)
    out = decode_attention_raw(q.to(dev), k.to(dev), v.to(dev), seq.to(dev), idx.to(dev), num_splits=splits)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    err = max_rel_err(out.cpu(), ref)
    assert err <= TOL, err
    for b, n in enumerate(lens):
        if n == 0:
            assert out[b].abs().max().item() == 0.0


def test_decode_ignores_stale_rows_past_seqlen():
    """Rows past seqlen inside the last tile may hold NaN/Inf left in a reused physical page."""
    from paper_2405_04437_b200.attention import decode_attention_raw

    dev = _cuda()
    gen = torch.Generator().manual_seed(1)
    B, hq, hkv, d, L = 3, 32, 8, 128, 256
    k, v = _mk_cache(B, L, hkv, d, gen)
    lens = [5, 100, 191]
    for b, n in enumerate(lens):
        k[b, n:] = float("nan")
        v[b, n:] = float("inf")
    q = _rand((B, hq, d), gen)
    seq = torch.tensor(lens, dtype=torch.int32)
    ref = decode_ref(q, k, v, seq)
    for splits in (1, 2):
        out = decode_attention_raw(q.to(dev), k.to(dev), v.to(dev), seq.to(dev), num_splits=splits)
        assert torch.isfinite(out.float()).all()
        assert max_rel_err(out.cpu(), ref) <= TOL


@pytest.mark.parametrize("d", [128, 64])
@pytest.mark.parametrize("block_size", [16, 64, 256])
@pytest.mark.parametrize("small_grid", [False, True])
def test_decode_paged_matches_oracle(block_size, d, small_grid):
    """small_grid: 2 rows x 8 KV heads x auto splits <= 148 CTAs, the two-consumer-group kernel;
    otherwise 5 rows (> 148 CTAs, 3-stage ring, one group)."""
    from paper_2405_04437_b200.attention import decode_attention_paged

    dev = _cuda()
    gen = torch.Generator().manual_seed(2)
    B, hq, hkv = (2, 32, 8) if small_grid else (5, 32, 8)
    lens = [1000, 2049] if small_grid else [1, 300, 1024, 17, 2049]
    maxb = (max(lens) + block_size - 1) // block_size
    nblocks = B * maxb + 3
    kp, vp = _mk_cache(nblocks, block_size, hkv, d, gen)
    perm = torch.randperm(nblocks, generator=gen)[: B * maxb].view(B, maxb).to(torch.int32)
    # gather the oracle's contiguous view of each sequence
    kc = kp[perm.long()].reshape(B, maxb * block_size, hkv, d)
    vc = vp[perm.long()].reshape(B, maxb * block_size, hkv, d)
    q = _rand((B, hq, d), gen)
    seq = torch.tensor(lens, dtype=torch.int32)
    ref = decode_ref(q, kc, vc, seq)
    out = decode_attention_paged(q.to(dev), kp.to(dev), vp.to(dev), perm.to(dev), seq.to(dev))
    assert max_rel_err(out.cpu(), ref) <= TOL


def test_kv_append_raw_bit_exact():
    from paper_2405_04437_b200.attention import kv_append_raw

    dev = _cuda()
    gen = torch.Generator().manual_seed(3)
    slots, L, hkv, d = 5, 300, 8, 128
    k, v = _mk_cache(slots, L, hkv, d, gen)
    for B, T in ((4, 1), (2, 37), (1, 256)):
        kn = _rand((B, T, hkv, d), gen)
        vn = _rand((B, T, hkv, d), gen)
        seq = torch.randint(0, L - T, (B,), generator=gen, dtype=torch.int32)
        idx = torch.randperm(slots, generator=gen)[:B].to(torch.int32)
        kr, vr = kv_append_ref(k, v, kn, vn, seq, idx)
        kd, vd = k.to(dev), v.to(dev)
        kv_append_raw(kd, vd, kn.to(dev), vn.to(dev), seq.to(dev), idx.to(dev))
        assert torch.equal(kd.cpu(), kr) and torch.equal(vd.cpu(), vr)
        k, v = kr, vr


@pytest.mark.parametrize("splits", [0, 1, 3])
def test_fused_append_decode_matches_append_then_decode(splits):
    """flash-attn k=/v= semantics: the new row is written at cache_seqlens[b] and attended to."""
    from paper_2405_04437_b200.attention import decode_attention_append_raw

    dev = _cuda()
    gen = torch.Generator().manual_seed(21)
    B, hq, hkv, d, L = 5, 56, 8, 128, 1024
    k, v = _mk_cache(B + 1, L, hkv, d, gen)
    lens = torch.tensor([0, 63, 64, 500, 1023], dtype=torch.int32)   # lengths BEFORE the token
    idx = torch.tensor([5, 0, 3, 1, 2], dtype=torch.int32)
    q = _rand((B, hq, d), gen)
    kn, vn = _rand((B, hkv, d), gen), _rand((B, hkv, d), gen)
    kr, vr = kv_append_ref(k, v, kn.unsqueeze(1), vn.unsqueeze(1), lens, idx)
    ref = decode_ref(q, kr, vr, lens + 1, idx)
    kd, vd = k.to(dev), v.to(dev)
    out = decode_attention_append_raw(q.to(dev), kd, vd, kn.to(dev), vn.to(dev), lens.to(dev), idx.to(dev),
                                      num_splits=splits)
    torch.cuda.synchronize()
    assert max_rel_err(out.cpu(), ref) <= TOL
    assert torch.equal(kd.cpu(), kr) and torch.equal(vd.cpu(), vr)


def test_kv_append_paged_bit_exact():
    from paper_2405_04437_b200.attention import kv_append_paged

    dev = _cuda()
    gen = torch.Generator().manual_seed(8)
    bs, hkv, d, nb = 16, 8, 128, 40
    kp, vp = _mk_cache(nb, bs, hkv, d, gen)
    B, T = 3, 20
    table = torch.randperm(nb, generator=gen)[: B * 6].view(B, 6).to(torch.int32)
    seq = torch.tensor([0, 17, 70], dtype=torch.int32)
    kn, vn = _rand((B, T, hkv, d), gen), _rand((B, T, hkv, d), gen)
    kr, vr = kp.clone(), vp.clone()
    for b in range(B):
        for i in range(T):
            pos = int(seq[b]) + i
            kr[table[b, pos // bs], pos % bs] = kn[b, i]
            vr[table[b, pos // bs], pos % bs] = vn[b, i]
    kd, vd = kp.to(dev), vp.to(dev)
    kv_append_paged(kd, vd, kn.to(dev), vn.to(dev), table.to(dev), seq.to(dev))
    assert torch.equal(kd.cpu(), kr) and torch.equal(vd.cpu(), vr)


@pytest.mark.parametrize("d,rd,inter,splits", [(128, 128, False, 0), (128, 64, False, 3), (128, 128, True, 0),
                                               (64, 32, True, 2), (64, 64, False, 0)])
def test_fused_decode_rotary_matches_oracle(d, rd, inter, splits):
    """Rotary at append (flash_attn_with_kvcache rotary_cos/sin): q and k_new rotated at position
    cache_seqlens[b]; k cached rotated; attention over the rotated cache."""
    from oracle.attention import rotary_ref
    from paper_2405_04437_b200.attention import decode_attention_append_raw

    dev = _cuda()
    gen = torch.Generator().manual_seed(7)
    B, hq, hkv, L = 4, 16, 4, 1024
    lens = [0, 63, 500, 1000]
    k, v = _mk_cache(B, L, hkv, d, gen)
    q = _rand((B, hq, d), gen)
    kn, vn = _rand((B, hkv, d), gen), _rand((B, hkv, d), gen)
    pos = torch.arange(L, dtype=torch.float32)
    inv = 1.0 / (10000 ** (torch.arange(0, rd, 2, dtype=torch.float32) / rd))
    ang = pos[:, None] * inv[None, :]
    cos, sin = ang.cos(), ang.sin()
    seq = torch.tensor(lens, dtype=torch.int32)
    qr = rotary_ref(q, cos, sin, seq, inter).to(torch.bfloat16)
    kr = rotary_ref(kn, cos, sin, seq, inter).to(torch.bfloat16)
    k_ref, v_ref = k.clone(), v.clone()
    for b, n in enumerate(lens):
        k_ref[b, n], v_ref[b, n] = kr[b], vn[b]
    ref = decode_ref(qr, k_ref, v_ref, seq + 1)
    kd, vd = k.to(dev), v.to(dev)
    out = decode_attention_append_raw(q.to(dev), kd, vd, kn.to(dev), vn.to(dev), seq.to(dev), num_splits=splits,
                                      rotary_cos=cos.to(dev), rotary_sin=sin.to(dev), rotary_interleaved=inter)
    torch.cuda.synchronize()
    assert max_rel_err(out.cpu(), ref) <= TOL
    got = kd.cpu()
    for b, n in enumerate(lens):      # the cached row is the rotated k (one bf16 rounding of fp32 math)
        assert torch.allclose(got[b, n].float(), kr[b].float(), rtol=1e-2, atol=1e-2)
        assert torch.equal(vd.cpu()[b, n], vn[b])


@pytest.mark.parametrize("batch,ctx,splits", [(2, 65536, 8), (3, 32768, 6), (8, 4096, 2)])
def test_split_decode_where_unit_clusters_cannot_all_coreside(batch, ctx, splits):
    """Split counts whose per-unit clusters (one cluster of `splits` CTAs per (row, KV head))
    would not all fit on the GPU at once fall back to the combine kernel (B 2 x 64K at 8 splits
    ran as two waves, 1.56x slower); every split count agrees with the oracle and with the
    unsplit kernel, ragged lengths included."""
    from paper_2405_04437_b200.attention import decode_attention_raw

    dev = _cuda()
    hq, hkv, d = 32, 8, 128
    gen = torch.Generator(device=dev).manual_seed(batch * 131 + ctx)
    k = torch.randn(batch, ctx, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)
    v = torch.randn(batch, ctx, hkv, d, device=dev, generator=gen, dtype=torch.bfloat16)
    q = torch.randn(batch, hq, d, device=dev, generator=gen, dtype=torch.bfloat16)
    seq = torch.tensor([ctx - 37 * b for b in range(batch)], dtype=torch.int32, device=dev)
    o_split = decode_attention_raw(q, k, v, seq, num_splits=splits)
    o_one = decode_attention_raw(q, k, v, seq, num_splits=1)
    torch.cuda.synchronize()
    assert torch.isfinite(o_split.float()).all()
    assert (o_split.float() - o_one.float()).abs().max().item() <= 2e-2 * o_one.float().abs().max().item()
    rows = [0, batch - 1]
    ref = decode_ref(q[rows].cpu(), k[rows].cpu(), v[rows].cpu(), seq[rows].cpu())
    assert max_rel_err(o_split[rows].cpu(), ref) <= TOL
