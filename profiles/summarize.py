#!/usr/bin/env python
"""Summarise a profiles/capture.sh run into committed, diff-able files:

    python profiles/summarize.py <tag> [gpurun_out]

* <tag>_launches.md   -- the ncu launch list (gpu__time_duration.sum,
  --clock-control none) of `bench.py --steps 2 --warmup 3`, aggregated per
  kernel: launches per step, time per step, share of the step. Per-launch times
  there are cold-cache and serialised; the SHARE is what bench.py's live CUDA
  event timing must agree with.
* <tag>_kernels.json  -- per kernel of one `--set full` step: duration, DRAM
  bytes read+written per launch (the roofline `traffic`), FP64 pipe and issue
  utilisation, occupancy. bench.py reads `traffic` from here.
* <tag>_launches.csv  -- the raw launch list (copied).
"""
from __future__ import annotations

import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import OrderedDict

HERE = os.path.dirname(os.path.abspath(__file__))

FULL_METRICS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read_mb": "dram__bytes_read.sum",
    "dram_write_mb": "dram__bytes_write.sum",
    "fp64_pipe_pct_active": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct_elapsed": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "fp64_tensor_pct_elapsed": "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "regs": "launch__registers_per_thread",
    "smem_per_block": "launch__shared_mem_per_block",
}


def short(name: str) -> str:
    n = name.replace("(anonymous namespace)::", "").replace("rk::", "").replace("void ", "")
    return n.split("(")[0]


def launches(tag, src):
    path = os.path.join(src, f"{tag}_launches.csv")
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        if "rk::" not in r["Kernel Name"]:  # torch fill/RNG kernels, the cuBLAS DGEMM of the peak probe
            continue
        k = short(r["Kernel Name"])
        ns = float(r["Metric Value"]) * (1e3 if r["Metric Unit"] == "us" else 1e6 if r["Metric Unit"] == "ms" else 1)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += ns
    shutil.copy(path, os.path.join(HERE, f"{tag}_launches.csv"))
    return agg


def full(tag, src):
    raw = os.path.join(src, f"{tag}_full_raw.csv")  # capture.sh exports it on the box (the .ncu-rep stays there)
    if os.path.exists(raw):
        out = open(raw).read()
    else:
        rep = os.path.join(src, f"{tag}_full.ncu-rep")
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = OrderedDict()
    for r in rows[2:]:
        k = short(r[head.index("Kernel Name")])
        d = OrderedDict()
        for key, m in FULL_METRICS.items():
            if m in head:
                i = head.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if key.endswith("_mb"):
                    v *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
                if key == "duration_ms":
                    v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0}.get(u, 1.0)
                d[key] = v
        if "dram_read_mb" in d and "dram_write_mb" in d:
            d["traffic_bytes"] = (d["dram_read_mb"] + d["dram_write_mb"]) * 1e6
        res.setdefault(k, []).append(d)
    return res


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(os.path.dirname(HERE), "gpurun_out")
    agg = launches(tag, src)
    mine = {k: v for k, v in agg.items() if k.startswith("<unnamed>::") or k.startswith("rk::")}
    steps = 5  # capture.sh: --steps 2 --warmup 3, every step launches the same kernels
    total = sum(v[1] for v in mine.values()) / steps
    cfg = os.environ.get("RK_CAPTURE_CONFIG", "c3")
    md = [f"# {tag}: ncu launch list of `bench.py --config {cfg} --steps 2 --warmup 3`, per step",
          "", "Cold-cache, serialised per-launch times (`--clock-control none`); library kernels only.", "",
          "| kernel | launches/step | µs/step | share |", "|---|---:|---:|---:|"]
    for k, (n, ns) in sorted(mine.items(), key=lambda kv: -kv[1][1]):
        md.append(f"| `{k}` | {n / steps:g} | {ns / steps / 1e3:.1f} | {ns / steps / total:.1%} |")
    md.append(f"| **total** | {sum(v[0] for v in mine.values()) / steps:g} | {total / 1e3:.1f} | 100% |")
    open(os.path.join(HERE, f"{tag}_launches.md"), "w").write("\n".join(md) + "\n")
    kern = full(tag, src)
    json.dump(kern, open(os.path.join(HERE, f"{tag}_kernels.json"), "w"), indent=1)
    km = [f"# {tag}: `ncu --set full` of one bench step (first launch of each kernel)", "",
          "| kernel | ms | DRAM MB (r+w) | FP64 pipe % active | FP64 tensor % | issue active % | warps active % | "
          "grid x block | regs |", "|---|---:|---:|---:|---:|---:|---:|---|---:|"]
    for k, ds in kern.items():
        d = ds[0]
        km.append(f"| `{k}` | {d.get('duration_ms', 0):.3f} | {d.get('traffic_bytes', 0) / 1e6:.1f} | "
                  f"{d.get('fp64_pipe_pct_active', 0):.1f} | {d.get('fp64_tensor_pct_elapsed', 0):.1f} | "
                  f"{d.get('issue_active_pct', 0):.1f} | {d.get('warps_active_pct', 0):.1f} | "
                  f"{d.get('grid', 0):.0f} x {d.get('block', 0):.0f} | {d.get('regs', 0):.0f} |")
    open(os.path.join(HERE, f"{tag}_kernels.md"), "w").write("\n".join(km) + "\n")
    bj = os.path.join(src, f"{tag}_bench.jsonl")
    if os.path.exists(bj):
        shutil.copy(bj, os.path.join(HERE, f"{tag}_bench.jsonl"))
    print("\n".join(md))
    for k, ds in kern.items():
        d = ds[0]
        print(k, {kk: round(v, 3) for kk, v in d.items() if isinstance(v, float)})


if __name__ == "__main__":
    main()
