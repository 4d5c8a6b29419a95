"""One launch of each hot kernel at a contract shape, for `ncu --set full` captures
(tools/gpu_ncu_r02.sh).  Not a benchmark: numbers under ncu are never bench values.

    python tools/ncu_targets.py decode G      # Llama-3-8B layer shard at G GPUs (B 64, ctx 4096+1)
    python tools/ncu_targets.py y34 G         # Yi-34B layer shard (B 128, ctx 8192+1)
    python tools/ncu_targets.py prefill       # Yi-6B 16K causal prefill
    python tools/ncu_targets.py append        # KV append, 4 requests x 16K tokens (> L2)
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
from paper_2405_04437_b200.attention import decode_attention_append, kv_append, prefill_attention
from paper_2405_04437_b200.geometry import llama3_8b, yi_34b, yi_6b

MB2 = 2 << 20
dev = torch.device("cuda")
what = sys.argv[1]
gen = torch.Generator(device=dev).manual_seed(0)


def decode(g, ctx, reps=3):
    g = g.__class__(**{**g.to_dict(), "n_layers": 1})
    B, hq, hkv = g.max_batch, g.q_heads_per_worker, g.kv_heads_per_worker
    groups = -(-(ctx + 2) * g.per_token_layer_bytes // MB2)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=(2 * B * groups + 4) * MB2))
    rids = [mgr.alloc_reqid() for _ in range(B)]
    assert mgr.step([ctx + 1] * B).ok
    idx = torch.tensor(rids, dtype=torch.int32, device=dev)
    for c0 in range(0, ctx, 1024):
        kn = torch.randn(B, 1024, hkv, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        kv_append(mgr, 0, kn, kn, torch.full((B,), c0, dtype=torch.int32, device=dev), idx)
    q = torch.randn(B, hq, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    k1 = torch.randn(B, hkv, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    pos = torch.full((B,), ctx, dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    for _ in range(reps):      # ncu -s skips the warm-up launches
        decode_attention_append(mgr, 0, q, k1, k1, pos, idx)
    torch.cuda.synchronize()
    mgr.close()


if what == "decode":
    decode(llama3_8b(max_context=4160, max_batch=64).with_tp(int(sys.argv[2])), 4096)
elif what == "y34":
    decode(yi_34b(max_context=8256, max_batch=128).with_tp(int(sys.argv[2])), 8192)
elif what == "prefill":
    S = 16384
    g = yi_6b(max_context=S, max_batch=1)
    g = g.__class__(**{**g.to_dict(), "n_layers": 1})
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=64 * MB2))
    r = mgr.alloc_reqid()
    assert mgr.step([S]).ok
    kn = torch.randn(1, S, 4, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    kv_append(mgr, 0, kn, kn, torch.zeros(1, dtype=torch.int32, device=dev), torch.tensor([r], dtype=torch.int32, device=dev))
    q = torch.randn(S, 32, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    for _ in range(3):
        prefill_attention(mgr, 0, q, r)
    torch.cuda.synchronize()
    mgr.close()
elif what == "append":
    S, R = 16384, 4
    g = yi_6b(max_context=S, max_batch=R)
    g = g.__class__(**{**g.to_dict(), "n_layers": 1})
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=(2 * R * 8 + 4) * MB2))
    rids = [mgr.alloc_reqid() for _ in range(R)]
    assert mgr.step([S] * R).ok
    kn = torch.randn(R, S, 4, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    vn = torch.randn(R, S, 4, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    idx = torch.tensor(rids, dtype=torch.int32, device=dev)
    z = torch.zeros(R, dtype=torch.int32, device=dev)
    for _ in range(3):
        kv_append(mgr, 0, kn, vn, z, idx)
    torch.cuda.synchronize()
    mgr.close()
else:
    raise SystemExit(__doc__)
