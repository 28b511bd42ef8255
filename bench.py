#!/usr/bin/env python
"""Benchmark of the full Ranky SVD hot path (repair -> block SVDs -> UΣ merge -> V).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]

One step = one full pass of the hot path over a BASELINE workload with the input
matrix already resident in HBM. The default is c3 (BASELINE.json configs[2]:
M=512, N=4,194,304, 512 blocks, Zipf column degrees, NeighborChecker, full Σ, U,
V), the largest config whose full step and host-side e2e (16 GiB of V) the
driver's run fits; c1/c2/c4/c5 are available with --config. For N>1 (torchrun,
one process per GPU) the same matrix's blocks are sharded by merge-tree leaves
(strong scaling): each rank factors its leaves, the subtree factors are
all-gathered over NCCL, every rank finishes the same tree top and recovers V for
its own columns; time is the max over ranks.

`e2e` is the same metric through the reference-facing C-ABI call
(rk_run_pipeline with RK_WANT_V | RK_WANT_REPAIRED | RK_WANT_RECORDS, i.e. the
reference run_pipeline's whole result plus V) on host buffers: entries H2D and
every output D2H inside the timed region. `--impl reference` times the
reference's own CPU implementation (oracle/_ref, all host threads) on the same
workload, rank 0 only: c1/c2 in full, c3-c5 by the stage-sampled estimator
(ReferenceEstimator, labelled extrapolated).
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
    ap.add_argument("--config", default="c3")
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


def config_dict(cfg, n_gpus, extra=None):
    d = {"workload": cfg.name if n_gpus == 1 else f"{cfg.name} with its {cfg.blocks} column blocks sharded over "
                                                   f"{n_gpus} GPUs (strong scaling: one matrix)",
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
    profiles/summarize.py): the longest captured launch whose name matches the stage;
    None when there is none."""
    import glob
    names = {"block_jacobi": ("jacobi_smem_kernel", "jacobi_wide_step_kernel", "jacobi_cluster_kernel", "jacobi_warp_kernel"),
             "block_qr": ("qr_kernel",),
             "merge": ("tridiag_cluster_kernel", "jacobi_cluster_kernel<32")}
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_kernels.json")))  # tags sort by round
    for f in reversed(files):
        try:
            kern = json.load(open(f))
        except Exception:
            continue
        best = None
        for k, launches in kern.items():
            if any(n in k for n in names.get(dominant, ())) and launches and "traffic_bytes" in launches[0]:
                d = max(launches, key=lambda x: x.get("duration_ms", 0.0))
                if best is None or d.get("duration_ms", 0.0) > best[0].get("duration_ms", 0.0):
                    best = (d, k)
        if best:
            return best[0]["traffic_bytes"], os.path.relpath(f, ROOT) + " :: " + best[1]
    return None, None


# --------------------------------------------------------------------------- reference arm

def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# configs whose full reference run (run_pipeline + recover_right_vectors) takes seconds:
# timed whole; the others by the stage-sampled estimator below
FULL_REFERENCE = ("c1", "c2")


class ReferenceEstimator:
    """The reference's run_pipeline + recover_right_vectors time, for configs whose
    full CPU run does not fit a bench step.

    The reference pipeline (proj/src/pipeline.cpp:61-121) is serial except the
    block-task pool, so its time is the sum of its stages. Every stage is the
    reference's own code, timed with std::chrono inside oracle/ref_capi.cpp
    (ref_sampled_pipeline) around the reference calls only:
      * repair — in full, every step (single-threaded, as in run_pipeline);
      * block_view + run_block_task — a seeded sample of `n` blocks, the tasks
        on min(workers, n) threads pulling from an atomic as pipeline.cpp:79-101
        does; scaled to D blocks by waves (ceil(D/pool) / ceil(n/pool));
      * proxy_from_records + proxy_svd — measured once on the first n/2 and on
        all n sampled records, fitted as a + b·Σk (Householder QR and apply_q are
        linear in Σk, the Jacobi on R is not) and evaluated at the full Σk;
      * recover_right_vectors — measured once on the first `slice` columns and
        scaled by N/slice.
    The estimate is labelled extrapolated."""

    def __init__(self, cfg, a, workers):
        import numpy as np
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from oracle import Oracle
        self.orc = Oracle("reference")
        self.cfg, self.workers = cfg, workers
        r, c, v = a.coo()
        self.coo = (a.rows(), a.cols(), r, c, v)
        self.nnz = a.nnz()
        self.n = int(os.environ.get("RK_REF_SAMPLE", str(2 * workers if cfg.rows <= 512 else workers)))
        # >= 16 blocks: the proxy fit's smaller sample (n/2 records) must already have full rank M,
        # or the reference's complete_columns dominates it (c3 blocks have rank ~127 of 512)
        self.n = max(min(16, cfg.blocks), min(self.n, cfg.blocks))
        rng = np.random.default_rng(1000 + cfg.seed)
        self.sample = np.sort(rng.choice(cfg.blocks, size=self.n, replace=False)).astype(np.uint64)
        self.slice = max(1, min(cfg.cols, cfg.cols // 64))
        self.calib = None

    def _call(self, phase):
        cfg = self.cfg
        return self.orc.sampled_pipeline(self.coo, cfg.blocks, cfg.method, cfg.keep, cfg.seed, self.workers,
                                         self.sample, self.slice, phase)

    def calibrate(self):
        t = self._call(7)
        cfg = self.cfg
        sk_all, sk_half, t_all, t_half = t[6], t[7], t[3], t[4]
        b = (t_all - t_half) / (sk_all - sk_half) if sk_all > sk_half else t_all / max(sk_all, 1)
        a0 = max(0.0, t_all - b * sk_all)
        sk_full = sk_all / self.n * cfg.blocks
        self.calib = {"proxy_s": a0 + b * sk_full, "recover_s": t[5] * cfg.cols / self.slice,
                      "proxy_fit": {"intercept_s": a0, "s_per_column": b, "sigma_k_full": sk_full,
                                    "measured": [[sk_half, t_half], [sk_all, t_all]]},
                      "recover_slice": [self.slice, t[5]]}
        return self.step(t)

    def step(self, t=None):
        if t is None:
            t = self._call(3)
        cfg = self.cfg
        pool = min(self.workers, self.n)
        waves = -(-cfg.blocks // self.workers) / -(-self.n // pool)  # full run's waves / the sample's
        parts = {"repair_s": t[0], "block_view_s": t[1] / self.n * cfg.blocks, "blocks_s": t[2] * waves,
                 "proxy_s": self.calib["proxy_s"], "recover_s": self.calib["recover_s"]}
        return sum(parts.values()), parts

    def describe(self):
        return (f"extrapolated from the reference's own stages timed in C++ (std::chrono in ref_capi.cpp): repair "
                f"in full; block_view + run_block_task on {self.n} seeded blocks of {self.cfg.blocks} on "
                f"{min(self.workers, self.n)} threads, scaled by waves; proxy_from_records + proxy_svd fitted "
                f"a + b*sum_k from {self.n // 2} and {self.n} records; recover_right_vectors on {self.slice} of "
                f"{self.cfg.cols} columns, scaled")


def reference_full_once(orc, cfg, coo, cores):
    """c1/c2: one full run_pipeline(workers=cores) + recover_right_vectors, timed in C++
    (ref_full_svd's t_blocks + t_proxy: input construction and result copies excluded)."""
    res = orc.full_svd(coo, cfg.blocks, cfg.method, cfg.keep, cfg.seed, cores, cfg.top_k)
    return res.times[1] + res.times[2]


def reference_arm(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle, available
    if not available("reference"):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libranky_ref.so not built"}))
        return 0
    a = cfg.generate()
    cores = os.cpu_count() or 1
    if cfg.name in FULL_REFERENCE:
        orc = Oracle("reference")
        r, c, v = a.coo()
        coo = (a.rows(), a.cols(), r, c, v)
        run = lambda: (reference_full_once(orc, cfg, coo, cores), None)  # noqa: E731
        sample = (f"one full {cfg.name} per step: run_pipeline(workers={cores}) + recover_right_vectors, timed in "
                  f"C++ around the reference calls")
        extra = {}
    else:
        est = ReferenceEstimator(cfg, a, cores)
        first = est.calibrate()
        run = est.step
        sample = est.describe()
        extra = {"calibration": est.calib, "first_estimate_s": first[0]}
    for _ in range(args.warmup):
        run()
    times, parts = [], []
    for _ in range(args.steps):
        t, p = run()
        times.append(t)
        parts.append(p)
    ms = 1e3 * sum(times) / len(times)
    value = a.nnz() / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_dict(cfg, ws, {"nnz": a.nnz()}),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "cpu_model": cpu_model(), "sample": sample,
                             "extrapolated": cfg.name not in FULL_REFERENCE},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if parts[0] is not None:
        line["stages_s_mean"] = {k: sum(p[k] for p in parts) / len(parts) for k in parts[0]}
    line.update(extra)
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(cfg, a):
    """One bounded sample of the reference on this host (rank 0, N=1)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle, available
    cores = os.cpu_count() or 1
    if not available("reference"):
        orc = Oracle("port")
        r, c, v = a.coo()
        t0 = time.perf_counter()
        orc.run_pipeline((a.rows(), a.cols(), r, c, v), cfg.blocks, cfg.method, cfg.keep, cfg.seed)
        dt = time.perf_counter() - t0
        return {"value": a.nnz() / dt, "unit": UNIT, "cores": 1, "kind": "port", "cpu_model": cpu_model(),
                "sample": f"one full {cfg.name} run_pipeline of the C restatement, {dt:.2f} s"}
    if cfg.name in FULL_REFERENCE:
        orc = Oracle("reference")
        r, c, v = a.coo()
        dt = reference_full_once(orc, cfg, (a.rows(), a.cols(), r, c, v), cores)
        return {"value": a.nnz() / dt, "unit": UNIT, "cores": cores, "kind": "reference", "cpu_model": cpu_model(),
                "sample": f"one full {cfg.name} run (run_pipeline workers={cores} + recover_right_vectors), "
                          f"{dt:.2f} s timed in C++", "extrapolated": False}
    est = ReferenceEstimator(cfg, a, cores)
    dt, parts = est.calibrate()
    return {"value": a.nnz() / dt, "unit": UNIT, "cores": cores, "kind": "reference", "cpu_model": cpu_model(),
            "sample": est.describe(), "extrapolated": True, "estimate_s": dt, "stages_s": parts}


# --------------------------------------------------------------------------- our arm

def main():
    args = parse()
    if os.environ.get("RK_BENCH_WATCHDOG"):  # debugging aid: every thread's stack, then exit
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["RK_BENCH_WATCHDOG"]), exit=True)
    from paper_2009_09767_b200 import configs
    cfg = configs.CONFIGS[args.config]
    if args.impl == "reference":
        return reference_arm(args, cfg)


    import numpy as np
    import torch
    import paper_2009_09767_b200 as rk
    from paper_2009_09767_b200 import ranky as R

    ws, rank, local = dist_env()
    # N > 1 is strong scaling: the config's one matrix, its column blocks sharded over
    # the ranks by merge-tree leaves (the paper's one-level distribution, BASELINE configs[3])
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
    a = cfg.generate()
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
        n_gather = [0]

        def allgather(mine, alls):
            """the library's one collective, on the caller's communicator (NCCL)"""
            n_gather[0] += 1
            if os.environ.get("RK_BENCH_WATCHDOG"):
                print(f"[rank {rank}] all-gather #{n_gather[0]}: sum {float(mine.sum()):.17g}", flush=True)
            if args.backend == "nccl":
                torch.distributed.all_gather_into_tensor(alls, mine)
            else:
                parts = [torch.empty(mine.numel(), dtype=torch.float64) for _ in range(ws)]
                torch.distributed.all_gather(parts, mine.cpu())
                alls.copy_(torch.cat(parts).to(alls.device))

        def sharded(dmx, sink=None):
            """this rank's share, orchestrated by the library (rk_dev_sharded_full_svd):
            factor its leaves, all-gather the subtree factors, finish the tree top
            (the TSQR factors when the kappa guard rejects the Gram route), V for its
            columns; `sink(out)` sees the outputs"""
            out, t, _, _ = R.dev_sharded_full_svd(dmx, cfg.blocks, cfg.method, cfg.keep, cfg.seed, ws, rank,
                                                  allgather, True, cfg.top_k)
            if sink:
                sink(out)
            R.dev_outputs_free(out)
            return t

        def step():
            return sharded(dm)

    for i in range(args.warmup):
        step()
        flush.zero_()
        if os.environ.get("RK_BENCH_WATCHDOG"):
            print(f"[rank {rank}] warm-up step {i} done", flush=True)
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
    cand = {"block_jacobi": (med["jacobi_ms"], med["jacobi_flops"]), "block_qr": (med["qr_ms"], med["qr_flops"]),
            "merge": (med["merge_ms"], med["merge_flops"])}
    # the dominant KERNEL, not stage: the block Jacobi and the block QR are one kernel each (plus a short
    # certifying launch); the merge is several (c3: SYRK 2.2, tridiagonalisation 4.0, bisection 0.5, vectors
    # 1.1, back-transformation 0.6 ms of 9.1 -- profiles/r02w_launches.md), so it competes with the share of
    # its largest kernel: 0.45 on the eigensolver route, 0.75 where its root is one Jacobi launch
    share = {"block_jacobi": 1.0, "block_qr": 1.0, "merge": 0.75 if med["merge_sweeps"] > 0 else 0.45}
    dom = max(cand, key=lambda k: cand[k][0] * share[k])
    d_ms, d_flops = cand[dom]
    achieved = d_flops / (d_ms * 1e-3) / 1e12 if d_ms > 0 else 0.0
    traffic, traffic_src = profiled_traffic(dom)
    roofline = {"bound": "tensor", "pipe": "fp64 (DFMA rounds + DMMA)", "kernel": dom, "achieved": achieved,
                "peak": fp64, "unit": "TFLOP/s", "frac": achieved / fp64 if fp64 else None, "traffic": traffic,
                "traffic_source": traffic_src,
                "peak_source": "measured in bench.py: cuBLAS DGEMM burst (torch.matmul f64 8192^3, best of 5); "
                               "FP64 is not in MEASURED_PEAKS.json",
                "flops_per_launch": d_flops, "ms_per_launch": d_ms,
                "flops_model": "QR: sum_d 2 n_d M^2 - 2/3 M^3 (wide blocks: 2 M n_d^2 - 2/3 n_d^3); Jacobi: per "
                               "block sweeps*(c(c-1)/2*2r + 2rc) + rotations*6r (r = the rows it runs on); merge: "
                               "Gram route M(M+1) sum k + M^3/3 + its Jacobi, TSQR route 2 sum k M^2 + its Jacobi"}
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
               "path": "per rank: rk_dev_matrix_create(pinned host entries) + rk_dev_sharded_full_svd (the "
                       "library's factor / NCCL all-gather / finish) + D2H of sigma, U and the rank's V rows; max "
                       "over ranks",
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
                                  ctx=ctx_e)
        e2e_ms = []
        h2d = d2h = 0
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = rk.run_pipeline(ha, cfg.blocks, cfg.method, cfg.keep, cfg.seed, 1, want_v=True, top_k=cfg.top_k,
                                  ctx=ctx_e)
            e2e_ms.append(1e3 * (time.perf_counter() - t0))
            h2d = a.nnz() * R.ENTRY_DTYPE.itemsize
            # the reference's run_pipeline result (sigma, U, report, repaired matrix, records) + V
            d2h = 8 * (res.svd.u.size + res.svd.sigma.size + res.svd.v.size) + \
                28 * len(res.report.added_edges) + 8 * cfg.blocks + \
                R.ENTRY_DTYPE.itemsize * res.repaired.nnz() + sum(8 * r.payload.size + 16 for r in res.records)
            del res
        e_ms = sum(e2e_ms) / len(e2e_ms)
        e2e = {"value": a.nnz() / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_median": statistics.median(e2e_ms),
               "ms_steps": [round(x, 3) for x in e2e_ms],
               "path": "rk_run_pipeline(host entries, RK_WANT_V | RK_WANT_REPAIRED | RK_WANT_RECORDS) via ctypes: "
                       "the reference run_pipeline's whole result (sigma, U, report, repaired matrix, records) plus V "
                       "on the host; wall clock per call"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, a)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong",
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
