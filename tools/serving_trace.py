"""BASELINE config 5 on the GPU: Algorithm-1 serving loop with real kernels (wall clock).

python tools/serving_trace.py --mode sync|overlapped --requests 128 [--out gpurun_out/serving]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2405_04437_b200.geometry import llama3_8b  # noqa: E402
from paper_2405_04437_b200.serving import (GemmDense, IterationModel, load_trace_csv, median_prompt_groups,  # noqa: E402
                                           run, run_paged)

MB2 = 2 * 1024 * 1024
ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="overlapped")
ap.add_argument("--requests", type=int, default=128)
ap.add_argument("--pool-gib", type=int, default=40)
ap.add_argument("--no-defer", action="store_true")
ap.add_argument("--prefetch", type=int, default=0, help="physical prefetch lookahead in tokens")
ap.add_argument("--spec-slots", type=int, default=0, help="speculative eager: slots to pre-map physically")
ap.add_argument("--spec-tokens", type=int, default=0, help="speculative eager: prompt tokens per slot")
ap.add_argument("--out", default=None)
ap.add_argument("--lazy-unmap", action="store_true", help="keep trimmed/reclaimed pages mapped until needed")
ap.add_argument("--hold", action="store_true", help="prefetch worker pauses during the launch burst")
ap.add_argument("--stage", type=int, default=0, help="staged admission: max iterations a prompt waits for its pages")
ap.add_argument("--dense-proxy", action="store_true", help="add IterationModel dense-layer time on the GPU")
ap.add_argument("--dense", choices=["sleep", "gemm"], default="gemm",
                help="dense-layer proxy with --dense-proxy: bf16 GEMMs (default) or the sleep kernel")
ap.add_argument("--sliced", action="store_true", help="layer-sliced cache layout (manager.py:93-96)")
ap.add_argument("--chunk", type=int, default=1, help="page-groups per physical handle (phys_chunk_groups)")
a = ap.parse_args()
rows = load_trace_csv(Path("tests/golden/trace_config5.csv"))[: a.requests]
g = llama3_8b(max_context=4096, max_batch=64)
eager = median_prompt_groups(rows, g, MB2, sliced=a.sliced)
dense = (GemmDense() if a.dense == "gemm" else IterationModel()) if a.dense_proxy else None
if a.mode == "paged":
    m = run_paged(rows, g, block_size=16, pool_bytes=a.pool_gib * 1024 ** 3,
                  dense_proxy=dense)
else:
    m = run(rows, g, mode=a.mode, clock="wall", page_group_size=MB2, pool_bytes=a.pool_gib * 1024 ** 3,
            eager_groups=eager if a.mode == "overlapped" else 0, reclaim_threshold=0.10,
            preemption_cap=100_000, defer=not a.no_defer,
            dense_proxy=dense, prefetch_tokens=a.prefetch, sliced=a.sliced,
            prefetch_slots=a.spec_slots, prefetch_slot_tokens=a.spec_tokens, lazy_unmap=a.lazy_unmap,
            stage_admission=a.stage > 0, stage_max_iters=a.stage, hold_worker=a.hold,
            phys_chunk_groups=a.chunk)
s = m.summary()
s.update({"mode": a.mode, "requests": a.requests, "eager_groups": eager, "defer": not a.no_defer,
          "dense_proxy": (a.dense if a.dense_proxy else None), "sliced": a.sliced, "prefetch": a.prefetch, "lazy_unmap": a.lazy_unmap, "stage": a.stage,
          "phys_chunk_groups": a.chunk})
if a.mode != "paged":
    its = m.iterations
    s["exposed_map_ms_median"] = sorted(r.exposed_ms for r in its)[len(its) // 2] if its else 0.0
    s["exposed_breakdown_ms"] = {k: sum(getattr(r, k) for r in its) for k in
                                 ("t_admit_ms", "t_bgwait_ms", "t_step_ms", "t_retire_ms")}
    s["driver_set_access_ms_total"] = sum(r.drv_set_access_ms for r in its)
    s["driver_maps_total"] = sum(r.drv_maps for r in its)
print(json.dumps(s))
if a.out:
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    tag = (a.mode + (f"_{a.dense}" if a.dense_proxy else "") + ("_sliced" if a.sliced else "") + (f"_pf{a.prefetch}" if a.prefetch else "")
           + (f"_ss{a.spec_slots}x{a.spec_tokens}" if a.spec_slots else "") + ("_lazy" if a.lazy_unmap else "")
           + (f"_stage{a.stage}" if a.stage else "") + ("_hold" if a.hold else "") + (f"_chunk{a.chunk}" if a.chunk > 1 else ""))
    m.write_iterations_csv(a.out + f"_{tag}.csv")
    with open(a.out + f"_{tag}.json", "w") as fh:
        json.dump(s, fh, indent=1)
