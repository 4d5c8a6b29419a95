"""BASELINE configs 2 and 4 at their stated sizes against the fp32 oracle (VERDICT r1 "missing 2",
"weak 2"): many rows, both error metrics of SURVEY §8(c).

* config 2: Llama-3-8B layer, B 64, context 4096 (+1 appended), fused append + decode through
  the VMM manager; ALL 64 rows are checked against oracle/attention.py.
* config 4: Yi-34B layer, B 128, context 8192 (+1), KV heads sharded over G = 1/2/4/8: one
  rank's shard (geometry.with_tp(G): 8/G KV heads, 56/G query heads; every rank runs the same
  shapes on its own heads) through its own manager; 16 sampled rows + the first and last row
  per shard against the oracle.

Tolerance: north_star max|o - o_ref| / max|o_ref| <= 2e-2.  The elementwise metric
max |o - o_ref| / (|o_ref| + 1e-3) is reported and bounded by ELEM_BOUND (it is dominated by
near-zero outputs, see oracle.attention.elem_rel_err).
"""

import json
import os

import pytest
import torch

from oracle.attention import decode_ref, err_report

pytestmark = pytest.mark.gpu
MB2 = 2 * 1024 * 1024
TOL = 2e-2
ELEM_BOUND = 2.0


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch.device("cuda")


def _record(name, rep):
    out = os.environ.get("VATTN_ERR_LOG")
    if out:
        with open(out, "a") as f:
            f.write(json.dumps({"case": name, **rep}) + "\n")
    print(name, rep)


def _run_layer(geom, B, ctx, rows, seed, name):
    """Fill one layer of a manager with `geom` (B slots at ctx tokens), run fused append+decode,
    compare `rows` against the oracle."""
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
    from paper_2405_04437_b200.attention import decode_attention_append, kv_append

    dev = _cuda()
    hkv, hq = geom.kv_heads_per_worker, geom.q_heads_per_worker
    groups_per_row = -(-(ctx + 1) * geom.per_token_layer_bytes // MB2)
    mgr = KVCacheManager(geom, ManagerConfig(page_group_size=MB2, pool_bytes=(2 * B * groups_per_row + 4) * MB2))
    rids = [mgr.alloc_reqid() for _ in range(B)]
    assert mgr.step([ctx + 1] * B).ok
    gen = torch.Generator(device=dev).manual_seed(seed)
    idx = torch.tensor(rids, dtype=torch.int32, device=dev)
    chunk = 1024
    for c0 in range(0, ctx, chunk):
        n = min(chunk, ctx - c0)
        kn = torch.randn(B, n, hkv, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        vn = torch.randn(B, n, hkv, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        kv_append(mgr, 0, kn, vn, torch.full((B,), c0, dtype=torch.int32, device=dev), idx)
    q = torch.randn(B, hq, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    k1 = torch.randn(B, hkv, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    v1 = torch.randn(k1.shape, device=dev, generator=gen, dtype=torch.bfloat16)
    pos = torch.full((B,), ctx, dtype=torch.int32, device=dev)
    out = decode_attention_append(mgr, 0, q, k1, v1, pos, idx)
    # idempotent and deterministic: appending the same token again gives the same bits
    again = decode_attention_append(mgr, 0, q, k1, v1, pos, idx)
    torch.cuda.synchronize()
    assert torch.equal(out, again)
    kc, vc = mgr.k_cache(0), mgr.v_cache(0)
    sel = torch.tensor([rids[b] for b in rows], dtype=torch.long, device=dev)
    k_rows = kc[sel, : ctx + 1].cpu()
    v_rows = vc[sel, : ctx + 1].cpu()
    # the appended token landed at row ctx of each slot
    assert torch.equal(k_rows[:, ctx], k1[rows].cpu()) and torch.equal(v_rows[:, ctx], v1[rows].cpu())
    ref = decode_ref(q[rows].cpu(), k_rows, v_rows, torch.full((len(rows),), ctx + 1, dtype=torch.int32))
    rep = err_report(out[rows].cpu(), ref)
    rep["rows_checked"] = len(rows)
    _record(name, rep)
    mgr.close()
    return rep


def test_config2_l8_all_64_rows():
    from paper_2405_04437_b200.geometry import llama3_8b

    g = llama3_8b(max_context=4160, max_batch=64)
    g = g.__class__(**{**g.to_dict(), "n_layers": 1})
    rep = _run_layer(g, 64, 4096, list(range(64)), 21, "config2_l8_b64_ctx4096")
    assert rep["max_rel_err"] <= TOL
    assert rep["elem_rel_err"] <= ELEM_BOUND


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_config4_y34_b128_shards(G):
    from paper_2405_04437_b200.geometry import ModelGeometry

    g = ModelGeometry(1, 8, 128, 2, max_context=8256, max_batch=128, tp_degree=G, n_q_heads_total=56)
    rows = sorted(set(torch.randperm(128, generator=torch.Generator().manual_seed(G))[:16].tolist()) | {0, 127})
    rep = _run_layer(g, 128, 8192, rows, 40 + G, f"config4_y34_b128_ctx8192_G{G}")
    assert rep["max_rel_err"] <= TOL
    assert rep["elem_rel_err"] <= ELEM_BOUND
