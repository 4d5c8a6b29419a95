"""GPU: the unmap fence (SURVEY §7 hard part 3) with lazily recorded use events.

Manager-backed launches only flag their stream (a per-launch event record between two decode
launches would cancel their programmatic dependent launch); the fence records the flagged
streams' events when it has to unmap.  A captured graph is covered by one explicit
`mark_use()` at the end of the captured region (an external event node), or, without it, by a
device-wide sync.  Each case queues a decode of slot r behind a 100 ms sleep kernel, then frees
r and reclaims its pages on the host: the reclaim must wait for the decode, and the decode must
read the data it was launched on."""

import ctypes as C
import time

import pytest
import torch

pytestmark = pytest.mark.gpu
MB2 = 2 << 20
SLEEP_NS = 100_000_000


def _sleep(stream):
    from paper_2405_04437_b200._abi import check, lib

    check(lib().vattn_compute_proxy(SLEEP_NS, C.c_void_p(stream.cuda_stream)))


@pytest.mark.parametrize("mode,chunk", [("eager", 1), ("graph_unmarked", 1), ("graph_marked_other_stream", 1),
                                        ("eager", 4), ("graph_marked_other_stream", 4), ("eager_dead_stream", 1)])
def test_reclaim_waits_for_queued_decode(mode, chunk):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2405_04437_b200 import KVCacheManager, ManagerConfig, ModelGeometry
    from paper_2405_04437_b200.attention import decode_attention, kv_append

    dev = torch.device("cuda")
    g = ModelGeometry(1, 8, 128, 2, max_context=8192, max_batch=2, n_q_heads_total=32)
    mgr = KVCacheManager(g, ManagerConfig(page_group_size=MB2, pool_bytes=64 * MB2, reclaim_threshold=0.0),
                         phys_chunk_groups=chunk)
    try:
        r = mgr.alloc_reqid()
        lens = [0, 0]
        lens[r] = 4096
        assert mgr.step(lens).ok
        gen = torch.Generator(device=dev).manual_seed(3)
        kv = torch.randn(1, 4096, 8, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        idx = torch.tensor([r], dtype=torch.int32, device=dev)
        seq = torch.tensor([4096], dtype=torch.int32, device=dev)
        kv_append(mgr, 0, kv, kv, torch.zeros(1, dtype=torch.int32, device=dev), idx)
        q = torch.randn(1, 32, 128, device=dev, generator=gen, dtype=torch.bfloat16)
        ref = decode_attention(mgr, 0, q, seq, idx)
        torch.cuda.synchronize()
        out = torch.zeros_like(ref)
        if mode == "eager":
            s = torch.cuda.current_stream()
            _sleep(s)
            decode_attention(mgr, 0, q, seq, idx, out=out)
        elif mode == "eager_dead_stream":     # launched on a stream that is gone before the fence
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                _sleep(s)
                decode_attention(mgr, 0, q, seq, idx, out=out)
            del s                        # (no gc.collect(): in a long test process it can outlast the sleep)
        else:
            cap = torch.cuda.Stream()
            cap.wait_stream(torch.cuda.current_stream())
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=cap, capture_error_mode="thread_local"):
                decode_attention(mgr, 0, q, seq, idx, out=out)
                if mode == "graph_marked_other_stream":
                    mgr.mark_use()
            torch.cuda.synchronize()
            s = torch.cuda.Stream() if mode == "graph_marked_other_stream" else torch.cuda.current_stream()
            with torch.cuda.stream(s):
                _sleep(s)
                graph.replay()
        t0 = time.perf_counter()
        mgr.free_reqid(r)
        freed, _ = mgr._reclaim_until(1 << 60)
        waited = time.perf_counter() - t0
        torch.cuda.synchronize()
        assert freed > 0
        assert waited >= 0.05, waited            # the unmap waited for the queued decode
        assert torch.equal(out, ref)
    finally:
        mgr.close()
