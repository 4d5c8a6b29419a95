"""Summarise the `ncu --set full` captures of tools/gpu_ncu_r02.sh (gpurun_out/ncu/*.raw.csv) into
profiles/: a markdown table and the per-shape DRAM traffic bench.py reports as roofline.traffic
(profiles/ncu_traffic.json, keys "<kernel label>|<workload-shape>").

    python tools/ncu_summarize.py [gpurun_out/ncu] [round tag]
"""
import csv
import json
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SRC = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "gpurun_out" / "ncu"
TAG = sys.argv[2] if len(sys.argv) > 2 else "r02"

FIELDS = {
    "dur_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "l2_hit": "lts__t_sector_hit_rate.pct",
    "occ": "sm__warps_active.avg.pct_of_peak_sustained_active",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ms": 1e3, "ns": 1e-3}


def read(path):
    rows = list(csv.reader(open(path)))
    h, u, v = rows[0], rows[1], rows[2]
    col = {name: i for i, name in enumerate(h)}
    out = {"kernel": v[col["Kernel Name"]], "grid": v[col["Grid Size"]], "block": v[col["Block Size"]]}
    for k, name in FIELDS.items():
        if name in col and v[col[name]].strip():
            x = float(v[col[name]].replace(",", ""))
            out[k] = x * SCALE.get(u[col[name]], 1)
    return out


def label(kernel):
    m = re.match(r"void (?:vattn::)?(?:pf::)?(\w+)<([^>]*)>", kernel)
    if not m:
        return kernel
    args = [a.strip() for a in m.group(2).split(",")]
    # ncu prints bool template arguments as 0/1: decode_kernel<D, STAGES, PAGED, CW>,
    # prefill_kernel<POLY, PAGED, D, VARLEN>
    bools = {"decode_kernel": (2,), "prefill_kernel": (1, 3)}.get(m.group(1), ())
    args = [("true" if a in ("1", "true") else "false") if i in bools else a for i, a in enumerate(args)]
    return f"{m.group(1)}<{','.join(args)}>"


# algorithmic bytes / flops per launch of each capture (tools/ncu_targets.py shapes)
def algorithmic(name):
    m = re.match(r"decode_(l8|y34)_G(\d)", name)
    if m:
        G = int(m.group(2))
        B, ctx, hkv, hq = (64, 4097, 8 // G, 32 // G) if m.group(1) == "l8" else (128, 8193, 8 // G, 56 // G)
        return {"bytes": 2 * B * ctx * hkv * 128 * 2 + 2 * B * hq * 128 * 2,
                "shape": f"{'l8_decode' if m.group(1) == 'l8' else 'y34_decode'}-G{G}"}
    if name == "prefill_y6":
        return {"flops": 2.0 * 16384 ** 2 * 128 * 32, "shape": "y6-16k"}
    if name == "append_4x16k":
        return {"bytes": 2 * 2 * 4 * 16384 * 4 * 128 * 2, "shape": "append-4x16k"}
    return {"shape": name}


def main():
    caps = {}
    for f in sorted(SRC.glob("*.raw.csv")):
        name = f.name[: -len(".raw.csv")]
        try:
            caps[name] = read(f)
        except Exception as e:  # noqa: BLE001
            print("skip", f, e)
    traffic_path = ROOT / "profiles" / "ncu_traffic.json"
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    traffic = {k: v for k, v in traffic.items() if "|" in k or k == "note"}
    traffic["note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch from one ncu --set full capture "
                       "(tools/gpu_ncu_r02.sh, tools/ncu_targets.py); key = kernel variant | workload shape; "
                       "bench.py scales it by its run's algorithmic bytes / the capture's")
    lines = [f"# ncu captures, round {TAG[1:]} (`ncu --set full --clock-control none`, one launch each)", "",
             "Cold-cache, serialised launches under ncu: durations are not bench values; the bench's CUDA-event "
             "times are. `alg` = algorithmic bytes (decode/append) per launch; `traffic/alg` > 1 = re-reads.", "",
             "| capture | kernel | grid x block | regs | ncu µs | DRAM read | DRAM write | traffic/alg | DRAM TB/s (ncu) | SM % | tensor pipe % (active) |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for name, c in caps.items():
        a = algorithmic(name)
        tr = c.get("dram_read", 0) + c.get("dram_write", 0)
        ratio = f"{tr / a['bytes']:.3f}" if "bytes" in a else "—"
        lines.append(f"| {name} | `{label(c['kernel'])}` | {c['grid']} x {c['block']} | {c.get('regs', 0):.0f} | "
                     f"{c.get('dur_us', 0):.1f} | {c.get('dram_read', 0) / 1e6:.1f} MB | {c.get('dram_write', 0) / 1e6:.1f} MB | "
                     f"{ratio} | {tr / (c.get('dur_us', 1) * 1e-6) / 1e12:.2f} | {c.get('sm_pct', 0):.1f} | {c.get('tensor_pct', 0):.1f} |")
        ent = {"workload": a["shape"], "dram_read_bytes": c.get("dram_read"), "dram_write_bytes": c.get("dram_write"),
               "traffic_bytes": tr, "duration_us_ncu": c.get("dur_us"),
               "capture": f"profiles/{TAG}_ncu_summary.md ({name}, tools/gpu_ncu_r02.sh)"}
        if "bytes" in a:
            ent["algorithmic_bytes"] = a["bytes"]
        key_label = label(c["kernel"])
        if key_label.startswith("decode_kernel"):
            keys = [f"{key_label} (fused append)|{a['shape']}"]
        elif key_label.startswith("prefill_kernel"):
            keys = [f"{key_label}|{a['shape']}"]
        else:
            keys = [f"{key_label}|{a['shape']}"]
        for k in keys:
            traffic[k] = ent
    (ROOT / "profiles" / f"{TAG}_ncu_summary.md").write_text("\n".join(lines) + "\n")
    traffic_path.write_text(json.dumps(traffic, indent=1) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
