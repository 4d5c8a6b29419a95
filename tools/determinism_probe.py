"""Determinism probe: the config-2 layer (fused append + decode through the VMM manager) built
twice from the same seeds in one process; prints bit-equality and a checksum to compare across
processes."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
from paper_2405_04437_b200.attention import decode_attention_append, kv_append
from paper_2405_04437_b200.geometry import llama3_8b

MB2 = 2 << 20


def run(seed=21, B=64, ctx=4096):
    dev = torch.device("cuda")
    g = llama3_8b(max_context=4160, max_batch=B)
    g = g.__class__(**{**g.to_dict(), "n_layers": 1})
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=(2 * B * 5 + 4) * MB2))
    rids = [mgr.alloc_reqid() for _ in range(B)]
    assert mgr.step([ctx + 1] * B).ok
    gen = torch.Generator(device=dev).manual_seed(seed)
    idx = torch.tensor(rids, dtype=torch.int32, device=dev)
    for c0 in range(0, ctx, 1024):
        kn = torch.randn(B, 1024, 8, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        vn = torch.randn(B, 1024, 8, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        kv_append(mgr, 0, kn, vn, torch.full((B,), c0, dtype=torch.int32, device=dev), idx)
    q = torch.randn(B, 32, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    k1 = torch.randn(B, 8, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    v1 = torch.randn(k1.shape, device=dev, generator=gen, dtype=torch.bfloat16)
    pos = torch.full((B,), ctx, dtype=torch.int32, device=dev)
    out = decode_attention_append(mgr, 0, q, k1, v1, pos, idx)
    torch.cuda.synchronize()
    kc = mgr.k_cache(0)[:, :ctx + 1].float().sum().item()
    res = (out.clone(), q.float().sum().item(), kc)
    mgr.close()
    return res


a = run()
b = run()
print("same-process equal:", torch.equal(a[0], b[0]), "q sums", a[1], b[1], "k sums", a[2], b[2])
d = (a[0].float() - b[0].float()).abs()
rows = (d.amax(dim=(1, 2)) > 0).nonzero().flatten().tolist()
heads = (d.amax(dim=(0, 2)) > 0).nonzero().flatten().tolist()
print("rows differing", len(rows), rows[:20], "heads", heads, "max diff", d.max().item())
for name in ("VATTN_DEC_STAGES", "VATTN_DEC_CW"):
    pass
print("checksum", a[0].float().sum().item(), a[0].float().abs().sum().item())
