"""The reference arm of bench.py keeps the driver's JSON contract (one line; cpu_baseline and e2e
objects; the oracle port timed on host cores) and runs on a CPU-only host."""

import json
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_prints_one_contract_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == "decode_attn_tokens_per_s" and d["value"] > 0
    assert d["steps"] == 1 and d["warmup"] == 3 and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_clock_sampler_reports_without_a_gpu():
    """The clocks object is always present: NVML when it works, else nvidia-smi, else an explicit
    'unavailable' reason (CPU host)."""
    import time

    sys.path.insert(0, str(ROOT))
    import bench

    c = bench.ClockSampler(0)
    c.start()
    time.sleep(0.02)
    d = c.stop()
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d)
    assert isinstance(d["reasons"], list)
