"""Fused decode + output-head all-gather over peer memory, on one GPU.

`HeadGather.local_group(G)` places G ranks' full-output buffers on one device; each simulated
rank runs the decode kernel over its own KV-head shard with the gather sink, exactly as a rank
of a torchrun job would (the only difference is that peer pointers are local instead of
IPC-mapped).  Every rank's full output must equal the fp32 oracle on the whole head set, and be
bit-identical to the same kernel writing its shard locally.
"""

import pytest
import torch

from oracle.attention import decode_ref, max_rel_err

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch.device("cuda")


def _rand(shape, gen):
    return torch.randn(shape, generator=gen).to(torch.bfloat16)


CASES = [
    # world, B, Hq, Hkv, D, seqlens, splits, fused_append
    (1, 3, 8, 2, 64, [128, 512, 1], 0, False),
    (2, 6, 32, 8, 128, [1, 63, 64, 65, 1000, 4096], 0, False),     # L8 shape over 2 ranks
    (4, 6, 32, 8, 128, [1, 63, 64, 65, 1000, 4096], 0, True),
    (8, 5, 56, 8, 128, [8192, 777, 4097, 1, 200], 0, False),       # Y34/8: 1 KV head per rank
    (2, 4, 32, 8, 128, [3000, 129, 64, 2048], 4, False),           # split-K: combine stores remotely
    (4, 4, 32, 8, 128, [3000, 129, 64, 2048], 3, True),
]


@pytest.mark.parametrize("case", CASES, ids=[str(i) for i in range(len(CASES))])
def test_fused_gather_matches_oracle_on_every_rank(case):
    from paper_2405_04437_b200.attention import decode_attention_append_raw, decode_attention_gather_raw
    from paper_2405_04437_b200.attention import decode_attention_raw
    from paper_2405_04437_b200.parallel import HeadGather

    dev = _cuda()
    G, B, hq, hkv, d, lens, splits, fused = case
    gen = torch.Generator().manual_seed(1)
    L = (max(lens) + 1 + 63) // 64 * 64
    k = _rand((B, L, hkv, d), gen)
    v = _rand((B, L, hkv, d), gen)
    q = _rand((B, hq, d), gen)
    kn, vn = _rand((B, hkv, d), gen), _rand((B, hkv, d), gen)
    seq = torch.tensor(lens, dtype=torch.int32)
    if fused:      # the new token lands at row seqlens[b] and is attended to
        k_ref, v_ref = k.clone(), v.clone()
        for b, n in enumerate(lens):
            k_ref[b, n], v_ref[b, n] = kn[b], vn[b]
        ref = decode_ref(q, k_ref, v_ref, seq + 1)
    else:
        ref = decode_ref(q, k, v, seq)
    gathers = HeadGather.local_group(G, B, hq, d, device=dev.index or 0)
    hk, hh = hkv // G, hq // G
    shards = []
    for r in range(G):
        kc = k[:, :, r * hk:(r + 1) * hk].contiguous().to(dev)
        vc = v[:, :, r * hk:(r + 1) * hk].contiguous().to(dev)
        shards.append((kc, vc, q[:, r * hh:(r + 1) * hh].contiguous().to(dev),
                       kn[:, r * hk:(r + 1) * hk].contiguous().to(dev), vn[:, r * hk:(r + 1) * hk].contiguous().to(dev)))
    seq_d = seq.to(dev)
    for rep in range(3):                      # epochs advance; the completion counter re-arms
        for r in range(G):                    # every rank launches, then every rank waits
            kc, vc, qr, knr, vnr = shards[r]
            if fused and rep > 0:             # appended row already in place: plain decode over +1
                decode_attention_gather_raw(qr, kc, vc, gathers[r], seq_d + 1, num_splits=splits, wait=False)
            elif fused:
                decode_attention_gather_raw(qr, kc, vc, gathers[r], seq_d, k_new=knr, v_new=vnr,
                                            num_splits=splits, wait=False)
            else:
                decode_attention_gather_raw(qr, kc, vc, gathers[r], seq_d, num_splits=splits, wait=False)
        for r in range(G):
            gathers[r].wait()
        torch.cuda.synchronize()
        for r in range(G):
            out = gathers[r].output(B).cpu()
            assert torch.isfinite(out.float()).all()
            assert max_rel_err(out, ref) <= TOL
            assert torch.equal(out, gathers[0].output(B).cpu())
    # bit-identical to the same kernel writing each shard locally
    full0 = gathers[0].output(B).cpu()
    for r in range(G):
        kc, vc, qr, _, _ = shards[r]
        loc = decode_attention_raw(qr, kc, vc, seq_d + (1 if fused else 0), num_splits=splits)
        torch.cuda.synchronize()
        assert torch.equal(loc.cpu(), full0[:, r * hh:(r + 1) * hh])
    assert all(g.timed_out_ranks() == [] for g in gathers)
    for g in gathers:
        g.close()


def test_manager_backed_gather_equals_plain_decode():
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
    from paper_2405_04437_b200.attention import decode_attention_append, decode_attention_gather, kv_append
    from paper_2405_04437_b200.geometry import ModelGeometry
    from paper_2405_04437_b200.parallel import HeadGather

    dev = _cuda()
    g = ModelGeometry(2, 8, 128, 2, max_context=4096, max_batch=4, n_q_heads_total=32)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=2 << 20, pool_bytes=1 << 30), backend="cuda",
                         device=dev.index or 0)
    rids = [mgr.alloc_reqid() for _ in range(3)]
    lens = [0] * 4
    for r, n in zip(rids, (700, 64, 2049)):
        lens[r] = n + 1
    assert mgr.step(lens).ok
    gen = torch.Generator(device=dev).manual_seed(0)
    idx = torch.tensor(rids, dtype=torch.int32, device=dev)
    before = torch.tensor([lens[r] - 1 for r in rids], dtype=torch.int32, device=dev)
    zero = torch.zeros(1, dtype=torch.int32, device=dev)
    for layer in range(2):
        for r in rids:       # only the stepped (mapped) rows of each slot
            kv = torch.randn(1, lens[r] - 1, 8, 128, device=dev, generator=gen, dtype=torch.bfloat16)
            kv_append(mgr, layer, kv, kv * 0.5, zero, torch.tensor([r], dtype=torch.int32, device=dev))
    q = torch.randn(3, 32, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    kn = torch.randn(3, 8, 128, device=dev, generator=gen, dtype=torch.bfloat16)
    (hg,) = HeadGather.local_group(1, 4, 32, 128, device=dev.index or 0)
    full = decode_attention_gather(mgr, 1, q, hg, before, idx, k_new=kn, v_new=kn * 2).clone()
    plain = decode_attention_append(mgr, 1, q, kn, kn * 2, before, idx)
    torch.cuda.synchronize()
    assert torch.equal(full, plain)
    hg.close()
    mgr.close()


def test_wait_times_out_when_a_rank_skips_its_launch(monkeypatch):
    from paper_2405_04437_b200.attention import decode_attention_gather_raw
    from paper_2405_04437_b200.parallel import HeadGather

    dev = _cuda()
    monkeypatch.setenv("VATTN_GATHER_TIMEOUT_MS", "200")
    gen = torch.Generator().manual_seed(2)
    k = _rand((2, 128, 1, 64), gen).to(dev)
    q = _rand((2, 4, 64), gen).to(dev)
    g0, g1 = HeadGather.local_group(2, 2, 8, 64, device=dev.index or 0)
    decode_attention_gather_raw(q, k, k, g0, torch.tensor([100, 5], dtype=torch.int32, device=dev))   # rank 1 never runs
    torch.cuda.synchronize()
    assert g0.timed_out_ranks() == [1]
    g0.close()
    g1.close()


def _ipc_worker(rank, world, port, q):
    import os
    import sys

    from conftest import ROOT
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2405_04437_b200.attention import decode_attention_gather_raw
        from paper_2405_04437_b200.parallel import HeadGather

        dev = torch.device("cuda", 0)        # both ranks on one GPU: same IPC + signalling path
        torch.cuda.set_device(dev)
        B, hq, hkv, d, lens = 4, 16, 4, 128, [700, 1, 64, 2049]
        gen = torch.Generator().manual_seed(3)
        k = _rand((B, 2112, hkv, d), gen)
        v = _rand((B, 2112, hkv, d), gen)
        qq = _rand((B, hq, d), gen)
        seq = torch.tensor(lens, dtype=torch.int32)
        ref = decode_ref(qq, k, v, seq)
        hg = HeadGather.create(B, hq, d, device=0)
        hk, hh = hkv // world, hq // world
        kc = k[:, :, rank * hk:(rank + 1) * hk].contiguous().to(dev)
        vc = v[:, :, rank * hk:(rank + 1) * hk].contiguous().to(dev)
        qr = qq[:, rank * hh:(rank + 1) * hh].contiguous().to(dev)
        for _ in range(3):
            out = decode_attention_gather_raw(qr, kc, vc, hg, seq.to(dev))
        torch.cuda.synchronize()
        err = max_rel_err(out.cpu(), ref)
        bad = hg.timed_out_ranks()
        dist.barrier()
        hg.close()
        q.put((rank, "ok" if err <= TOL and not bad else f"err={err} timed_out={bad}"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)[:300]))
    finally:
        dist.destroy_process_group()


def test_two_processes_gather_through_cuda_ipc():
    """Two processes (ranks) share one GPU: the CUDA IPC handle exchange, peer mapping and
    cross-process flag signalling of HeadGather.create run exactly as on two GPUs."""
    import socket

    import torch.multiprocessing as mp

    _cuda()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == [(0, "ok"), (1, "ok")], res


def test_gather_and_manager_decode_replay_from_a_cuda_graph():
    """The gather epoch lives on the device and mark_use records an external event node, so a
    captured step (manager-backed fused decode + fused gather of 2 simulated ranks) replays
    correctly many times."""
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
    from paper_2405_04437_b200.attention import decode_attention_append, decode_attention_gather_raw
    from paper_2405_04437_b200.geometry import ModelGeometry
    from paper_2405_04437_b200.parallel import HeadGather

    dev = _cuda()
    gen = torch.Generator().manual_seed(5)
    # manager-backed fused decode, captured
    g = ModelGeometry(2, 8, 128, 2, max_context=2048, max_batch=2, n_q_heads_total=32)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=2 << 20, pool_bytes=64 << 20), backend="cuda",
                         device=dev.index or 0)
    rids = [mgr.alloc_reqid(), mgr.alloc_reqid()]
    assert mgr.step([1100, 1100]).ok
    q = _rand((2, 32, 128), gen).to(dev)
    kn = _rand((2, 8, 128), gen).to(dev)
    idx = torch.tensor(rids, dtype=torch.int32, device=dev)
    pos = torch.tensor([1000, 1000], dtype=torch.int32, device=dev)
    out = torch.empty_like(q)
    # 2 simulated gather ranks over caller-owned caches
    k = _rand((3, 256, 4, 64), gen).to(dev)
    qg = _rand((3, 8, 64), gen).to(dev)
    seq = torch.tensor([200, 17, 256], dtype=torch.int32, device=dev)
    gs = HeadGather.local_group(2, 3, 8, 64, device=dev.index or 0)
    shards = [(k[:, :, 2 * r:2 * r + 2].contiguous(), qg[:, 4 * r:4 * r + 4].contiguous()) for r in range(2)]

    def body():
        decode_attention_append(mgr, 1, q, kn, kn, pos, idx, out=out)
        pos.add_(1)
        for r in range(2):
            decode_attention_gather_raw(shards[r][1], shards[r][0], shards[r][0], gs[r], seq, wait=False)
        for r in range(2):
            gs[r].wait()

    body()                       # warm-up (workspace, tensor maps)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s, capture_error_mode="thread_local"):
        body()
    for _ in range(5):
        graph.replay()
    torch.cuda.synchronize()
    assert pos.tolist() == [1006, 1006]
    got_dec = out.clone()
    assert all(x.timed_out_ranks() == [] for x in gs)
    # eager reference of the last replay: rows 1005 appended, attention over 1006 rows
    ref = decode_attention_append(mgr, 1, q, kn, kn, pos - 1, idx)
    torch.cuda.synchronize()
    assert torch.equal(got_dec, ref)
    from paper_2405_04437_b200.attention import decode_attention_raw
    full = gs[1].output(3).clone()
    for r in range(2):
        loc = decode_attention_raw(shards[r][1], shards[r][0], shards[r][0], seq)
        torch.cuda.synchronize()
        assert torch.equal(full[:, 4 * r:4 * r + 4], loc.cpu().to(full.device))
    for x in gs:
        x.close()
    mgr.close()
