"""Multi-process (gloo, world_size 2) coverage of the KV-head-sharded path on CPU:
each rank's allocator (C++ core, shadow backend) over geometry.with_tp(2) matches the oracle, and
the output-head all-gather reassembles the full head dimension."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.allocator import Geometry, OracleManager
        from paper_2405_04437_b200 import KVCacheManager, ManagerConfig
        from paper_2405_04437_b200.geometry import yi_34b
        from paper_2405_04437_b200.parallel import gather_heads, head_ranges, shard_geometry

        full = yi_34b(max_context=8192, max_batch=8)
        g = shard_geometry(full, world)
        mgr = KVCacheManager(g, ManagerConfig(page_group_size=2 << 20, pool_bytes=1 << 34), backend="shadow")
        og = Geometry(g.n_layers, g.kv_heads_total, g.head_dim, g.bytes_per_elem, g.max_context, g.max_batch, g.tp_degree)
        om = OracleManager(og, 2 << 20, pool_bytes=1 << 34)
        seq = [0] * 8
        for step in range(40):
            if step % 7 == 0 and 0 in seq:
                r1, r2 = mgr.alloc_reqid(), om.alloc_reqid()
                assert r1 == r2
                seq[r1] = 1000 + 900 * step
            seq = [min(s + 97, 8192) if s else 0 for s in seq]
            ok, us = om.step(seq)
            res = mgr.step(seq)
            assert (res.ok, res.sync_us) == (ok, us)
        st = mgr.parity_state()
        assert st["mapped"] == om.dev.mapped and st["slots"] == [[int(s[0]), s[1], s[2], s[3], s[4]] for s in om.slots]
        # every rank computes the same bookkeeping
        t = torch.tensor([st["mapped"], st["created"]], dtype=torch.int64)
        ts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(ts, t)
        assert all(torch.equal(x, t) for x in ts)
        # head all-gather: rank r holds query heads [r*Hq/G, (r+1)*Hq/G)
        (_, _), (qlo, qhi) = head_ranges(full, rank, world)
        local = torch.arange(qlo, qhi, dtype=torch.float32).view(1, -1, 1).expand(3, -1, 4).contiguous()
        out = gather_heads(local)
        assert out.shape == (3, full.q_heads_total, 4)
        assert torch.equal(out[0, :, 0], torch.arange(full.q_heads_total, dtype=torch.float32))
        # fused-gather setup: IPC handles are exchanged in rank order; creating the device
        # buffers without a GPU fails loudly (no host fallback for the gather)
        from paper_2405_04437_b200.parallel import HeadGather, exchange_handles
        blobs = exchange_handles(bytes([rank + 1]) * 64)
        assert blobs == [bytes([r + 1]) * 64 for r in range(world)]
        try:      # every rank fails (no GPU) but still completes the exchange: no rank hangs
            HeadGather.create(4, full.q_heads_total, 128, device=0)
            raise AssertionError("HeadGather.create succeeded without a GPU")
        except AssertionError:
            raise
        except Exception:
            pass
        dist.barrier()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_kv_head_sharding_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, "ok") for r in range(world)], res
