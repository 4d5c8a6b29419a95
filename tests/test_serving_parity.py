"""The Algorithm-1 serving loop (paper_2405_04437_b200.serving, model clock, C++ allocator core)
reproduces the reference simulator (kvsim.simulator.run) iteration for iteration: every
IterationRecord field and the summary, in sync and overlapped modes — including the overlapped
protocol that executes the plan on the background thread *before* the next admission (plan
credits keep slot reuse identical)."""

import random

import pytest

from conftest import REF_SRC

MB2, KB64, GIB, MIB = 2 * 1024 * 1024, 65536, 1024 ** 3, 1024 ** 2


def _ref_rows(kvsim, metrics):
    from paper_2405_04437_b200.serving import IterationRecord
    return [[getattr(r, f) for f in IterationRecord.REF_FIELDS] for r in metrics.iterations]


def _ours_rows(metrics):
    from paper_2405_04437_b200.serving import IterationRecord
    return [r.row(IterationRecord.REF_FIELDS) for r in metrics.iterations]


def _compare(kvsim, geo_kw, rows, **kw):
    from kvsim.geometry import ModelGeometry as RefGeometry
    from kvsim.simulator import run as ref_run
    from kvsim.trace import SimTrace

    from paper_2405_04437_b200.geometry import ModelGeometry
    from paper_2405_04437_b200.serving import run

    from kvsim.simulator import SimulationAborted as RefAborted

    from paper_2405_04437_b200.serving import SimulationAborted

    try:
        ref = ref_run(SimTrace.from_rows(rows), RefGeometry(**geo_kw), allocator="vattention", **kw)
    except RefAborted:
        with pytest.raises(SimulationAborted):
            run(rows, ModelGeometry(**geo_kw), clock="model", backend="shadow", **kw)
        return
    ours = run(rows, ModelGeometry(**geo_kw), clock="model", backend="shadow", **kw)
    assert _ours_rows(ours) == _ref_rows(kvsim, ref)
    a, b = ours.summary(), ref.summary()
    for k in b:
        assert a[k] == b[k], k


@pytest.mark.reference
@pytest.mark.parametrize("mode", ["sync", "overlapped"])
def test_spike_trace(ref_kvsim, mode):
    geo = dict(n_layers=60, kv_heads_total=8, head_dim=128, bytes_per_elem=2, max_context=200_000,
               max_batch=8, tp_degree=2)
    rows = [(0, p, 8) for p in (2047, 2047, 6142, 2045, 2047)]
    _compare(ref_kvsim, geo, rows, page_group_size=MB2, mode=mode, pool_bytes=8 * GIB)


@pytest.mark.reference
@pytest.mark.parametrize("seed", range(24))
def test_random_small_traces(ref_kvsim, seed):
    rng = random.Random(seed)
    geo = dict(n_layers=3, kv_heads_total=4, head_dim=128, bytes_per_elem=2, max_context=4096, max_batch=6)
    rows, clock = [], 0
    for _ in range(rng.randint(3, 12)):
        clock += rng.randint(0, 40)
        rows.append((clock, rng.randint(1, 3000), rng.randint(1, 300)))
    pg = KB64 if seed % 2 else MB2
    pool = 48 * MIB if pg == KB64 else 640 * MIB
    if seed % 5 == 0:
        pool //= 4                      # memory pressure: preemption + reclaim paths
    _compare(ref_kvsim, geo, rows, page_group_size=pg, pool_bytes=pool,
             mode="overlapped" if seed % 3 else "sync", eager_groups=(seed % 4),
             reclaim_threshold=[0.1, 0.5, 0.9][seed % 3], preemption_cap=100_000)


@pytest.mark.reference
@pytest.mark.parametrize("mode", ["sync", "overlapped"])
def test_config5_trace_prefix(ref_kvsim, mode):
    """BASELINE config 5 (L8 shape, 2 MiB, eager = median prompt groups, reclaim 0.10)."""
    from pathlib import Path

    from paper_2405_04437_b200.geometry import ModelGeometry
    from paper_2405_04437_b200.serving import load_trace_csv, median_prompt_groups

    rows = load_trace_csv(Path(__file__).parent / "golden" / "trace_config5.csv")[:48]
    geo = dict(n_layers=32, kv_heads_total=8, head_dim=128, bytes_per_elem=2, max_context=4096, max_batch=64)
    eager = median_prompt_groups(rows, ModelGeometry(**geo), MB2)
    _compare(ref_kvsim, geo, rows, page_group_size=MB2, pool_bytes=6 * GIB, mode=mode,
             eager_groups=eager, reclaim_threshold=0.10, preemption_cap=100_000)


@pytest.mark.parametrize("mode", ["sync", "overlapped"])
def test_serving_call_log_replays_through_oracle(mode):
    """The serving loop's call recorder (serving.run(record=...)) replayed through the oracle on
    the shadow backend: the harness tests/test_gpu_serving_replay.py applies to the GPU run."""
    import random

    from allocator_replay import replay_serving_log
    from paper_2405_04437_b200.geometry import ModelGeometry
    from paper_2405_04437_b200.serving import run

    rnd = random.Random(3)
    t, rows = 0, []
    for _ in range(60):
        t += rnd.randint(0, 20)
        rows.append((t, rnd.randint(64, 3000), rnd.randint(2, 40)))
    geo = ModelGeometry(2, 8, 128, 2, max_context=4096, max_batch=8, n_q_heads_total=32)
    record = []
    m = run(rows, geo, clock="model", backend="shadow", mode=mode, page_group_size=MB2, pool_bytes=80 * MB2,
            eager_groups=2 if mode == "overlapped" else 0, reclaim_threshold=0.10, preemption_cap=100_000,
            record=record)
    stats = replay_serving_log(record, geo, MB2, 80 * MB2, 2 if mode == "overlapped" else 0, 0.10)
    assert stats["iterations"] == len(m.iterations) > 0
    s = m.summary()
    assert s["requests_with_first_token"] == 60
