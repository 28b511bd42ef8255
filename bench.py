#!/usr/bin/env python
"""Benchmark of the full Ranky SVD hot path (repair -> block SVDs -> UΣ merge -> V).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

One step = one full pass of the hot path over the BASELINE workload (configs[1],
c2: M=256, N=262144, 64 blocks, RandomChecker, full Σ, U, V) with the input
matrix already resident in HBM. For N>1 (torchrun, one process per GPU) the
blocks are sharded by merge-tree leaves, each rank factors its leaves, the
subtree R factors are all-gathered over NCCL and every rank finishes the same
tree top and recovers V for its own columns; time is the max over ranks.

`e2e` is the same metric through the reference-facing C-ABI call
(rk_run_pipeline with RK_WANT_V) on host buffers: entries H2D and sigma/U/V
D2H inside the timed region. `--impl reference` times the reference's own CPU
implementation (oracle/_ref: run_pipeline + recover_right_vectors, all host
threads) on the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "full Ranky SVD nnz/s"
UNIT = "nnz/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    # functional dry run of the N>1 path on a one-GPU box: every rank on device 0, the
    # collectives through gloo on host copies (not a performance configuration)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def weak_matrix(base, ws, R):
    """The weak-scaling workload for ws GPUs: the config's matrix tiled ws times
    along the columns ([A A ... A], ws x the blocks), so every GPU's share of
    column blocks is exactly the single-GPU workload."""
    import numpy as np
    a = base.generate()
    e = a.entries()
    t = np.concatenate([e] * ws)
    n = len(e)
    for k in range(1, ws):
        t["col"][k * n:(k + 1) * n] += k * base.cols
    t = t[np.lexsort((t["col"], t["row"]))]
    return R.SparseMatrix._trusted(base.rows, base.cols * ws, t)


def config_dict(cfg, n_gpus, extra=None):
    d = {"workload": cfg.name if n_gpus == 1 else f"{cfg.name} tiled x{n_gpus} along the columns (one {cfg.name} "
                                                   f"per GPU: {cfg.blocks // n_gpus} blocks, {cfg.cols // n_gpus} "
                                                   f"columns)",
         "rows": cfg.rows, "cols": cfg.cols, "blocks": cfg.blocks, "method": cfg.method,
         "keep": cfg.keep, "top_k": cfg.top_k, "seed": cfg.seed, "description": cfg.description,
         "parallelism": f"block-shard x{n_gpus}" if n_gpus > 1 else "single GPU",
         "l2": "flushed between steps (256 MiB write)"}
    if extra:
        d.update(extra)
    return d


# --------------------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = os.path.join("/tmp", f"rk_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows)}


class NvmlClockSampler:
    """The same samples through NVML from a thread of this process (no nvidia-smi
    process contending for the driver while the steps run)."""

    def __init__(self, device, period=0.1):
        self.device, self.period = device, period
        self.rows, self.stop_flag, self.thread = [], False, None

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
        except Exception:
            self.thread = None
            return
        bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

        def loop():
            smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self.stop_flag:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((sm, smax, sorted(k for k, b in bits.items() if r & b)))
                time.sleep(self.period)
        self.thread = threading.Thread(target=loop, daemon=True)
        self.thread.start()

    def stop(self):
        if not self.thread:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self.stop_flag = True
        self.thread.join(timeout=5)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted({x for r in self.rows for x in r[2]}), "samples": len(self.rows), "source": "nvml"}


# --------------------------------------------------------------------------- peaks

def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "MEASURED_PEAKS.json"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


def fp64_peak_tflops(torch):
    """FP64 peak is not in MEASURED_PEAKS.json: measured here as a cuBLAS DGEMM
    burst (torch.matmul float64, 8192^3, best of 5)."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def profiled_traffic(dominant):
    """DRAM bytes (read + write) per launch of the dominant kernel, from the newest
    committed `ncu --set full` summary (profiles/*_kernels.json, written by
    profiles/summarize.py); None when there is none."""
    import glob
    names = {"block_jacobi": "jacobi_cluster_kernel<16, 16, 1", "block_qr": "qr_kernel"}
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_kernels.json")))
    for f in reversed(files):
        try:
            kern = json.load(open(f))
        except Exception:
            continue
        for k, launches in kern.items():
            if names.get(dominant, "?") in k and launches and "traffic_bytes" in launches[0]:
                return launches[0]["traffic_bytes"], os.path.relpath(f, ROOT) + " :: " + k
    return None, None


# --------------------------------------------------------------------------- reference arm

def reference_arm(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle, available
    kind = "reference" if available("reference") else "port"
    orc = Oracle(kind)
    a = cfg.generate()
    r, c, v = a.coo()
    coo = (a.rows(), a.cols(), r, c, v)
    cores = os.cpu_count() or 1
    run = (lambda: orc.full_svd(coo, cfg.blocks, cfg.method, cfg.keep, cfg.seed, cores, cfg.top_k)) \
        if kind == "reference" else (lambda: orc.run_pipeline(coo, cfg.blocks, cfg.method, cfg.keep, cfg.seed))
    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = a.nnz() / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak" if ws > 1 else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_dict(dataclasses.replace(cfg, cols=cfg.cols * ws, blocks=cfg.blocks * ws) if ws > 1
                                  else cfg, ws, {"nnz": a.nnz()}),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": f"full {cfg.name} per step (run_pipeline workers={cores} + "
                                       f"recover_right_vectors), {args.steps} steps" +
                                       (f"; for {ws} GPUs (weak scaling) one GPU's {cfg.name}-sized share is the "
                                        f"sample" if ws > 1 else "")},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(cfg, a):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle, available
    kind = "reference" if available("reference") else "port"
    orc = Oracle(kind)
    r, c, v = a.coo()
    coo = (a.rows(), a.cols(), r, c, v)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    if kind == "reference":
        orc.full_svd(coo, cfg.blocks, cfg.method, cfg.keep, cfg.seed, cores, cfg.top_k)
    else:
        orc.run_pipeline(coo, cfg.blocks, cfg.method, cfg.keep, cfg.seed)
        cores = 1
    dt = time.perf_counter() - t0
    return {"value": a.nnz() / dt, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"one full {cfg.name} run (run_pipeline workers={cores} + recover_right_vectors), {dt:.2f} s"}


# --------------------------------------------------------------------------- our arm

def main():
    args = parse()
    from paper_2009_09767_b200 import configs
    cfg = configs.CONFIGS[args.config]
    if args.impl == "reference":
        return reference_arm(args, cfg)

    import ctypes as C

    import numpy as np
    import torch
    import paper_2009_09767_b200 as rk
    from paper_2009_09767_b200 import ranky as R

    ws, rank, local = dist_env()
    if ws > 1:
        # weak scaling: every GPU gets the single-GPU workload as its share -- the
        # matrix is [A A ... A] with ws x the columns and blocks (weak_matrix), the
        # paper's one-level distribution of column blocks over machines
        cfg = dataclasses.replace(cfg, cols=cfg.cols * ws, blocks=cfg.blocks * ws)
    if args.backend == "gloo":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    ctx = rk.Context(local)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)

    # FP64 peak first, before the library's stream-ordered pool holds the big buffers
    fp64 = fp64_peak_tflops(torch) if rank == 0 else 0.0
    a = weak_matrix(configs.CONFIGS[args.config], ws, R) if ws > 1 else cfg.generate()
    dm = rk.DeviceMatrix(a, ctx)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    L = R.lib()
    M = cfg.rows

    def allreduce_max(t):
        if args.backend == "gloo":
            t = t.cpu()
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    if ws == 1:
        def step():
            out, t = R.dev_full_svd(dm, cfg.blocks, cfg.method, cfg.keep, cfg.seed, True, cfg.top_k)
            R.dev_outputs_free(out)
            return t
    else:
        from paper_2009_09767_b200 import shard as SH
        sp = SH.plan(M, cfg.cols, cfg.blocks, cfg.keep, ws, rank)
        lo, hi, c_lo, c_hi = sp.leaf_lo, sp.leaf_hi, sp.col_lo, sp.col_hi
        roots = torch.empty((ws, M, M), dtype=torch.float64, device="cuda")
        mine = torch.empty((M, M), dtype=torch.float64, device="cuda")

        def gather():
            if args.backend == "nccl":
                torch.distributed.all_gather_into_tensor(roots, mine)
            else:
                parts = [torch.empty((M, M), dtype=torch.float64) for _ in range(ws)]
                torch.distributed.all_gather(parts, mine.cpu())
                roots.copy_(torch.stack(parts))

        def sharded(dmx, sink=None):
            """this rank's share: factor its leaves, all-gather the subtree's Gram
            partial (NCCL), finish the merge, V for its columns; the TSQR factors
            instead when the Gram route is rejected (identically on every rank);
            `sink(out)` sees the outputs"""
            shard = C.c_void_p()
            t = R.Timing()
            fargs = (ctx.handle, dmx.handle, cfg.blocks, R._method(cfg.method), cfg.keep, cfg.seed, lo, hi,
                     C.c_void_p(mine.data_ptr()), C.byref(shard), C.byref(t))
            st = L.rk_dev_shard_factor_gram(*fargs)
            gram = st == 0
            if st == R.GRAM_REJECTED:
                R._check(L.rk_dev_shard_factor(*fargs))
            else:
                R._check(st)
            gather()
            out = C.POINTER(R.DevOutputs)()
            t2 = R.Timing()
            gargs = (ctx.handle, shard, C.c_void_p(roots.data_ptr()), ws, R.WANT_V, cfg.top_k, c_lo, c_hi,
                     C.byref(out), C.byref(t2))
            st = L.rk_dev_shard_finish_gram(*gargs) if gram else L.rk_dev_shard_finish(*gargs)
            if gram and st == R.GRAM_REJECTED:
                R._check(L.rk_dev_shard_tsqr(ctx.handle, shard, C.c_void_p(mine.data_ptr())))
                gather()
                st = L.rk_dev_shard_finish(*gargs)
            R._check(st)
            if sink:
                sink(out)
            R.dev_outputs_free(out)
            L.rk_dev_shard_destroy(shard)
            t.merge_ms += t2.merge_ms
            t.merge_flops += t2.merge_flops
            t.merge_sweeps = t2.merge_sweeps
            t.recover_ms = t2.recover_ms
            t.kernel_launches += t2.kernel_launches
            return t

        def step():
            return sharded(dm)

    for _ in range(args.warmup):
        step()
        flush.zero_()
    barrier()
    clocks = ClockSampler(local) if os.environ.get("RK_CLOCKS", "nvml") == "smi" else NvmlClockSampler(local)
    clocks.start()
    ms_steps, launches, timings = [], 0, []
    barrier()
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t = step()
        e1.record(stream)
        flush.zero_()  # outside the step's events
        torch.cuda.synchronize()
        ms_steps.append(e0.elapsed_time(e1))
        launches += int(t.kernel_launches)
        timings.append(t.as_dict())
    barrier()
    wall = time.perf_counter() - wall0
    clk = clocks.stop()
    ms = sum(ms_steps) / len(ms_steps)
    if ws > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        ms = allreduce_max(tt)
    value = a.nnz() / (ms / 1e3)

    # ---- roofline of the dominant kernel (by device time) --------------------------
    med = {k: statistics.median([t[k] for t in timings]) for k in timings[0]}
    peaks, peak_src = measured_peaks()
    cand = {"block_jacobi": (med["jacobi_ms"], med["jacobi_flops"]), "block_qr": (med["qr_ms"], med["qr_flops"])}
    dom = max(cand, key=lambda k: cand[k][0])
    d_ms, d_flops = cand[dom]
    achieved = d_flops / (d_ms * 1e-3) / 1e12 if d_ms > 0 else 0.0
    traffic, traffic_src = profiled_traffic(dom)
    roofline = {"bound": "tensor", "pipe": "fp64 (DFMA rounds + DMMA)", "kernel": dom, "achieved": achieved,
                "peak": fp64, "unit": "TFLOP/s", "frac": achieved / fp64 if fp64 else None, "traffic": traffic,
                "traffic_source": traffic_src,
                "peak_source": "measured in bench.py: cuBLAS DGEMM burst (torch.matmul f64 8192^3, best of 5); "
                               "FP64 is not in MEASURED_PEAKS.json",
                "flops_per_launch": d_flops, "ms_per_launch": d_ms,
                "flops_model": "QR: sum_d 2 n_d M^2 - 2/3 M^3; Jacobi: per block sweeps*(c(c-1)/2*2M + 2Mc) "
                               "+ rotations*6M"}
    stages = {k: med[k] for k in ("repair_ms", "blocks_ms", "qr_ms", "jacobi_ms", "merge_ms", "recover_ms",
                                  "total_ms")}
    stages["jacobi_sweeps_max"] = med["jacobi_sweeps_max"]
    stages["merge_sweeps"] = med["merge_sweeps"]
    v_bytes = 8.0 * (cfg.cols // ws) * M  # this rank's V rows
    stages["recover_hbm_frac"] = (v_bytes / (med["recover_ms"] * 1e-3) / 1e9) / peaks["hbm_gbs"] \
        if med["recover_ms"] > 0 else None
    # every stage against its own roof: HBM for the rank check +
    # repair and the V SpMM (algorithmic bytes), FP64 for the factorizations
    nnz = a.nnz()
    repair_bytes = 12.0 * nnz + 8.0 * (M + 1) + 4.0 * M * cfg.blocks  # CSR col+val, row_ptr, presence flags
    spmm_bytes = v_bytes + 12.0 * nnz / ws + 8.0 * (cfg.cols // ws + 1) + 8.0 * M * M
    hbm = peaks["hbm_gbs"]

    def frac(x, ms, peak, scale):
        return {"achieved": x / (ms * 1e-3) / scale, "peak": peak, "frac": x / (ms * 1e-3) / scale / peak} \
            if ms > 0 and peak else None
    stage_roofs = {
        "repair (HBM, GB/s)": frac(repair_bytes, med["repair_ms"], hbm, 1e9),
        "block factor: Gram + Cholesky / QR (FP64, TF/s)": frac(med["qr_flops"], med["qr_ms"], fp64, 1e12),
        "block Jacobi (FP64, TF/s)": frac(med["jacobi_flops"], med["jacobi_ms"], fp64, 1e12),
        "merge: SYRK + Cholesky + Jacobi (FP64, TF/s)": frac(med["merge_flops"], med["merge_ms"], fp64, 1e12),
        "V recovery SpMM (HBM, GB/s)": frac(spmm_bytes, med["recover_ms"], hbm, 1e9),
    }

    # ---- e2e through the C ABI with host buffers -----------------------------------
    e2e = None
    if not args.no_e2e and ws > 1:
        # every rank: H2D of the entries (rk_dev_matrix_create from pinned memory), its
        # share of the pipeline with the NCCL all-gather, D2H of sigma, U and its V rows;
        # the step's time is the max over ranks
        pinned = torch.empty(a.nnz() * R.ENTRY_DTYPE.itemsize, dtype=torch.uint8, pin_memory=True)
        host_e = pinned.numpy().view(R.ENTRY_DTYPE)
        host_e[:] = a.entries()
        ha = R.SparseMatrix._trusted(a.rows(), a.cols(), host_e)
        k_out = cfg.top_k or M
        v_host = torch.empty((c_hi - c_lo) * k_out, dtype=torch.float64, pin_memory=True)
        u_host = torch.empty(M * M + M, dtype=torch.float64, pin_memory=True)
        moved = {}

        def to_host(out):
            sig_d, u_d, v_d = R.dev_outputs_tensors(out)
            nv = v_d.numel()
            v_host[:nv].copy_(v_d.reshape(-1), non_blocking=True)
            u_host[:u_d.numel()].copy_(u_d.reshape(-1), non_blocking=True)
            u_host[u_d.numel():u_d.numel() + sig_d.numel()].copy_(sig_d, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            moved["d2h"] = 8 * (nv + u_d.numel() + sig_d.numel())

        def e2e_step():
            dmx = rk.DeviceMatrix(ha, ctx)
            sharded(dmx, to_host)
            dmx.close()

        for _ in range(max(3, args.warmup)):
            e2e_step()
        e2e_ms = []
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            t0 = time.perf_counter()
            e2e_step()
            torch.cuda.synchronize()
            dt = torch.tensor([1e3 * (time.perf_counter() - t0)], dtype=torch.float64, device="cuda")
            e2e_ms.append(allreduce_max(dt))
        e_ms = sum(e2e_ms) / len(e2e_ms)
        e2e = {"value": a.nnz() / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": a.nnz() * R.ENTRY_DTYPE.itemsize, "d2h_bytes_per_step": moved.get("d2h", 0),
               "ms_median": statistics.median(e2e_ms),
               "path": "per rank: rk_dev_matrix_create(pinned host entries) + rk_dev_shard_factor + NCCL "
                       "all_gather + rk_dev_shard_finish + D2H of sigma, U and the rank's V rows; max over ranks",
               "bytes_note": "per rank"}
    if not args.no_e2e and ws == 1:
        pinned = torch.empty(a.nnz() * R.ENTRY_DTYPE.itemsize, dtype=torch.uint8, pin_memory=True)
        host_e = pinned.numpy().view(R.ENTRY_DTYPE)
        host_e[:] = a.entries()
        ha = R.SparseMatrix._trusted(a.rows(), a.cols(), host_e)
        ctx_e = rk.Context(local)  # what a user gets: the library's own stream
        res = None
        for _ in range(max(3, args.warmup)):  # as the timed loop: two result buffers alternate
            res = rk.run_pipeline(ha, cfg.blocks, cfg.method, cfg.keep, cfg.seed, 1, want_v=True, top_k=cfg.top_k,
                                  want_repaired=False, want_records=False, ctx=ctx_e)
        e2e_ms = []
        h2d = d2h = 0
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = rk.run_pipeline(ha, cfg.blocks, cfg.method, cfg.keep, cfg.seed, 1, want_v=True, top_k=cfg.top_k,
                                  want_repaired=False, want_records=False, ctx=ctx_e)
            e2e_ms.append(1e3 * (time.perf_counter() - t0))
            h2d = a.nnz() * R.ENTRY_DTYPE.itemsize
            d2h = 8 * (res.svd.u.size + res.svd.sigma.size + res.svd.v.size) + \
                28 * len(res.report.added_edges) + 8 * cfg.blocks
        e_ms = sum(e2e_ms) / len(e2e_ms)
        e2e = {"value": a.nnz() / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_median": statistics.median(e2e_ms),
               "ms_steps": [round(x, 3) for x in e2e_ms],
               "path": "rk_run_pipeline(host entries, RK_WANT_V) via ctypes; wall clock per call"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, a)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "weak" if ws > 1 else "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, csrc/gen.c)",
                "config": config_dict(cfg, ws, {"nnz": a.nnz()}), "roofline": roofline, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": launches, "clocks": clk, "stages_ms_median": stages,
                "stage_rooflines": stage_roofs,
                "wall_s_timed_region": wall, "peaks_source": peak_src}
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
