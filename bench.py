#!/usr/bin/env python
"""Benchmark of the BILU numeric phase (BASELINE.json metric) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl reference]

A step is one bilu_factor (the whole hot path: scatter, Schur updates, pivot
inverses, scaling/dropping, progressive aggregation) of the configs[1] matrix
(3D 7-pt convection-diffusion 64^3, ND ordering, tau = 1e-3), inputs resident in
HBM.  At N > 1 the same factorization is split over the ranks (strong scaling):
phase A factors each rank's top-level ND subtrees, the interface panels are
all-gathered over NCCL, phase B factors the separators.  value = factorizations
per second; ms_per_step = device time of one factorization (CUDA events, max over
ranks).  `e2e` repeats the step through
the C-ABI with the matrix values copied from pinned HOST memory every step.
Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BILU numeric factor time & FP64 GFLOP/s (fraction of FP64 peak), 1-8 B200"
FP64_PEAK_TFLOPS = 37.2     # measured: DMMA m8n8k4 microbenchmark (profiles/r01_fp64_peak.md)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(config):
    """DRAM bytes per factor_kernel launch from the committed ncu --set full capture (or None)."""
    p = os.path.join(ROOT, "profiles", "r02_factor_traffic.json")
    try:
        d = json.load(open(p))
        if not d["workload"].startswith(config):
            return None
        return float(d["dram_bytes_read"] + d["dram_bytes_write"])
    except Exception:
        return None


def make_problem(name, world=1):
    """The bench workload; at world > 1 the same matrix and ordering with the top log2(world)
    ND levels labelled as subtrees (the ordering does not depend on the labels)."""
    from inputs.configs import make_config
    if world > 1:
        lv = int(round(np.log2(world)))
        if 2 ** lv != world:
            raise SystemExit("bench.py: --gpus must be a power of two for the subtree partition")
        return make_config(name, top_levels=lv)
    return make_config(name)


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""
    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.samples)}


def dist_init(n_gpus, force=False):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or force:
        if force and "MASTER_ADDR" not in os.environ:
            os.environ["MASTER_ADDR"] = "127.0.0.1"
            os.environ.setdefault("MASTER_PORT", "29531")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        import torch.distributed as dist
        dist.init_process_group("nccl" if n_gpus > 0 else "gloo")
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(x, world):
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x, world):
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def run_reference(args, rank, world):
    """Reference arm: the CPU oracle as it stands, on the box's host cores."""
    import oracle
    if rank != 0:
        return
    P = make_problem(args.config)
    ip, ix, dv = oracle.permute_csr(P.indptr, P.indices, P.data, P.perm)
    times = []
    for i in range(args.warmup + args.steps):
        f = oracle.factor(ip, ix, dv, P.block_sizes, P.tau, aggregate=True)
        if i >= args.warmup:
            times.append(f.t_factor_s)
    t = float(np.mean(times))
    val = 1.0 / t
    out = {"metric": METRIC, "value": val, "unit": "factorizations/s", "impl": "reference",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic",
           "config": {"workload": args.config + " (BASELINE.json configs[1])", "n": P.n, "nnz": P.nnz,
                      "tau": P.tau, "blocks_init": int(len(P.block_sizes)), "aggregate": True},
           "gflops": f.flops / t / 1e9, "flops_per_factorization": f.flops,
           "cpu_baseline": {"value": val, "unit": "factorizations/s", "cores": 1, "kind": "oracle",
                            "sample": "full %s factorization per step (plain C scalar oracle, 1 thread)" % args.config},
           "e2e": {"value": val, "unit": "factorizations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def cpu_baseline(P, budget_s=30.0):
    import oracle
    ip, ix, dv = oracle.permute_csr(P.indptr, P.indices, P.data, P.perm)
    times = []
    t_start = time.time()
    flops = 0.0
    while not times or (time.time() - t_start < budget_s * 0.4 and len(times) < 3):
        f = oracle.factor(ip, ix, dv, P.block_sizes, P.tau, aggregate=True)
        times.append(f.t_factor_s)
        flops = f.flops
    t = float(np.mean(times))
    return {"value": 1.0 / t, "unit": "factorizations/s", "cores": 1, "kind": "oracle",
            "sample": "%d full %s factorization(s), plain C scalar oracle, 1 thread; %.2f s each, %.3g flops"
                      % (len(times), P.name, t, flops)}


# Dense-zone budgets (bilu_options.zone_bytes, DESIGN 5b) of the extra configs where the
# library default (min(64 GiB, 45% of the free HBM)) is not the fastest measured one
# (profiles/r02_zone_sweep.log: c3 52.5 ms at 64 GiB, 49.3 at 96, 46.3 at 128; c5 flat beyond 64).
ZONE_GIB = {"c3": 120}


def time_config(name, steps, warmup, flush):
    """Device time of the other BASELINE configs' factorizations at N = 1 (extra keys of the
    bench line; c2 stays the headline): same protocol as the headline (warm-up, L2 flush,
    CUDA events around bilu_factor), inputs resident in HBM."""
    import torch
    from inputs.configs import make_config
    from paper_1908_10169_b200 import BILU
    t0 = time.time()
    P = make_config(name)
    opts = {}
    free = torch.cuda.mem_get_info()[0]
    if name in ZONE_GIB and free >= (ZONE_GIB[name] + 40) << 30:   # leave 40 GiB for the factors
        opts["zone_bytes"] = ZONE_GIB[name] << 30
    g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm, **opts)
    prep_s = time.time() - t0
    for _ in range(warmup):
        g.factor(P.tau)
    ms, kms = [], []
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = g.factor(P.tau)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        kms.append(st["t_factor_ms"] - st["t_merge_ms"])
    g.close()
    t, tk = float(np.mean(ms)), float(np.mean(kms))
    tf = st["flops"] / (tk * 1e-3) / 1e12
    return {"ms_per_step": t, "factorizations_per_s": 1e3 / t, "steps": steps, "warmup": warmup,
            "gflops": st["flops"] / (t * 1e-3) / 1e9, "flops_per_factorization": st["flops"],
            "n": P.n, "nnz": P.nnz, "blocks_init": int(len(P.block_sizes)), "blocks_final": int(st["n_blocks_final"]),
            "zone_blocks": int(st["zone_blocks"]),
            "zone_bytes": opts.get("zone_bytes", "library default"),
            "roofline": {"bound": "tensor", "kernel": "factor_kernel", "achieved": tf, "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": tf / FP64_PEAK_TFLOPS, "kernel_ms": tk},
            "generate_and_analyze_s": prep_s}


def time_config_dist(name, world, steps, warmup, flush):
    """N > 1: the distributed factorization (phase A, NCCL exchange, phase B) of another
    BASELINE config -- c5 is the 1/2/4/8-GPU config -- timed like the headline (device events,
    L2 flush, max over ranks).  Every rank takes part; rank 0 reports (extra key)."""
    import torch
    from paper_1908_10169_b200 import BILU
    from paper_1908_10169_b200.dist import factor_distributed, partition_owner
    rank = int(os.environ.get("RANK", "0"))
    t0 = time.time()
    P = make_problem(name, max(world, 2))
    g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm, device=torch.cuda.current_device())
    g.dist_setup(partition_owner(P.block_part, world), rank)
    prep_s = time.time() - t0
    for _ in range(warmup):
        factor_distributed(g, P.tau)
    ms = []
    for _ in range(steps):
        flush.zero_()
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st, sent, recv = factor_distributed(g, P.tau)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    local = g.local_stats["flops"]
    flops = allreduce_sum(local, world) + (st["flops"] - local)
    t = allreduce_max(float(np.mean(ms)), world)
    g.close()
    return {"ms_per_step": t, "factorizations_per_s": 1e3 / t, "steps": steps, "warmup": warmup,
            "gflops": flops / (t * 1e-3) / 1e9, "flops_per_factorization": flops,
            "fp64_peak_fraction": flops / (t * 1e-3) / 1e12 / (FP64_PEAK_TFLOPS * world),
            "n": P.n, "nnz": P.nnz, "blocks_init": int(len(P.block_sizes)),
            "exchange_bytes_rank0": {"sent": sent, "received": recv},
            "parallelism": "ND subtrees over %d GPUs, interface panels over NCCL, separators replicated" % world,
            "generate_and_analyze_s": prep_s}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the c3/c4/c5 factor timings (extra keys)")
    ap.add_argument("--dist", action="store_true",
                    help="use the distributed (subtree) path even at N=1 (checks its mechanics on one GPU)")
    args = ap.parse_args()

    rank, world, local = dist_init(args.gpus, force=args.dist)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    from paper_1908_10169_b200 import BILU
    from paper_1908_10169_b200.build import build
    torch.cuda.set_device(local)
    if rank == 0:
        build()
    barrier(world)

    use_dist = world > 1 or args.dist
    P = make_problem(args.config, max(world, 2) if use_dist else 1)
    g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm, device=local)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > L2 (126 MB)
    xfer = [0, 0]
    local_flops = [0.0]
    if use_dist:
        # multi-GPU: phase A on this rank's ND subtrees, interface exchange (NCCL), phase B
        from paper_1908_10169_b200.dist import factor_distributed, partition_owner
        owner = partition_owner(P.block_part, world)
        g.dist_setup(owner, rank)

        def step():
            st_, sent, recv = factor_distributed(g, P.tau)
            xfer[0], xfer[1] = sent, recv
            local_flops[0] = g.local_stats["flops"]
            return st_
    else:
        def step():
            return g.factor(P.tau)

    for _ in range(args.warmup):
        st = step()
    torch.cuda.synchronize()

    # ---------------- device-timed steps (inputs resident in HBM)
    clk = ClockSampler(local)
    clk.start()
    barrier(world)
    torch.cuda.synchronize()
    step_ms, kern_ms, launches = [], [], 0
    flops = 0.0
    for _ in range(args.steps):
        flush.zero_()                                  # L2 flush between timed iterations
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        st = step()
        e1.record()
        torch.cuda.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        kern_ms.append(st["t_factor_ms"] - st["t_merge_ms"])   # factor kernel(s) (phases A + B at N > 1)
        launches += int(st["n_kernel_launches"])
        flops = st["flops"]
    torch.cuda.synchronize()
    barrier(world)
    clocks = clk.stop()
    if use_dist:   # the factorization's flops: every rank's subtrees + the separators once
        flops = allreduce_sum(local_flops[0], world) + (flops - local_flops[0])
    t_step = allreduce_max(float(np.sum(step_ms)), world) / args.steps
    t_kern = allreduce_max(float(np.mean(kern_ms)), world)
    value = (world if world == 1 else 1) / (t_step * 1e-3)   # N > 1: one factorization per step

    # ---------------- distributed preconditioner apply (all ranks; reported by rank 0)
    dist_apply = None
    if use_dist and not args.no_solve:
        from paper_1908_10169_b200.dist import apply_distributed
        xb = torch.ones(P.n, dtype=torch.float64, device="cuda")
        for _ in range(2):
            apply_distributed(g, xb)
        barrier(world)
        torch.cuda.synchronize()
        ea0, ea1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea0.record()
        for _ in range(5):
            yb = apply_distributed(g, xb)
        ea1.record()
        torch.cuda.synchronize()
        dist_apply = {"dist_apply_ms": allreduce_max(ea0.elapsed_time(ea1) / 5, world),
                      "y_sum": float(yb.sum().item()),
                      "note": "bilu_apply_dist_begin/_end + 2 all-reduces, device time, max over ranks"}

    # ---------------- e2e through the C-ABI with host buffers
    e2e = None
    if not args.no_e2e:
        vals_pinned = torch.from_numpy(np.ascontiguousarray(P.data)).pin_memory()
        host_ptr = vals_pinned.data_ptr()
        import ctypes
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            g.lib.bilu_set_values(g.h, ctypes.c_void_p(host_ptr), 0)
            step()                                   # ends with its device->host status read
        torch.cuda.synchronize()
        t_e2e = allreduce_max((time.perf_counter() - t0) / args.steps, world)
        e2e = {"value": (world if world == 1 else 1) / t_e2e, "unit": "factorizations/s",
               "h2d_bytes_per_step": int(P.nnz * 8),
               "d2h_bytes_per_step": int(16 * 8 + (16 * 8 + 4 + 8 + 4 if g.opt.aggregate else 0)),
               "ms_per_step": t_e2e * 1e3,
               "note": "bilu_set_values from pinned host values + bilu_factor + its device->host statistics "
                       "read; the factors stay in HBM (they are a preconditioner, applied by bilu_apply)"}

    extra_dist = None
    if use_dist and not args.no_extra:
        extra_dist = {"c5": time_config_dist("c5", world, args.steps, args.warmup, flush)}

    if rank == 0:
        hbm_peak, hbm_src = load_peaks()
        achieved_tf = st["flops"] / (t_kern * 1e-3) / 1e12
        out = {
            "metric": METRIC, "value": value, "unit": "factorizations/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.config + " (BASELINE.json configs[1]): 3D 7-pt conv-diff 64^3, "
                                   "geometric ND, tau=1e-3, initial blocks <=8, aggregation on, max_block 128",
                       "n": P.n, "nnz": P.nnz, "tau": P.tau, "blocks_init": int(len(P.block_sizes)),
                       "blocks_final": int(st["n_blocks_final"]), "merges": int(st["n_merges"]),
                       "parallelism": ("ND subtrees over %d GPUs (%d top levels), interface panels "
                                       "all-gathered over NCCL, separators replicated" % (world, int(np.log2(world))))
                                      if use_dist else "single GPU",
                       "exchange_bytes_per_rank": {"sent": xfer[0], "received": xfer[1]} if use_dist else None,
                       "l2": "flushed between timed steps (256 MB write)"},
            "gflops": flops / (t_step * 1e-3) / 1e9,
            "flops_per_factorization": flops,
            "fp64_peak_fraction": (flops / (t_step * 1e-3) / 1e12) / FP64_PEAK_TFLOPS,
            "nnz_factors": int(st["nnz_L"] + st["nnz_U"] + st["nnz_D"]),
            "roofline": {"bound": "tensor", "kernel": "factor_kernel (persistent, all of a-1..a-8)",
                         "achieved": achieved_tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved_tf / FP64_PEAK_TFLOPS, "traffic": load_traffic(args.config),
                         "traffic_source": "profiles/r02_factor_traffic.json (ncu --set full, DRAM read+write bytes "
                                           "per factor_kernel launch)",
                         "peak_source": "measured FP64 DMMA microbenchmark (profiles/r01_fp64_peak.md)",
                         "kernel_ms": t_kern,
                         "hbm": {"achieved_gbs": st["bytes_min"] / (t_kern * 1e-3) / 1e9,
                                 "peak_gbs": hbm_peak, "peak_source": hbm_src}},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if e2e:
            out["e2e"] = e2e
        if not use_dist and not args.no_solve:
            # context: one preconditioned GMRES(30) solve with these factors,
            # b = ones, tol 1e-8, device time; and one preconditioner apply
            b = torch.ones(P.n, dtype=torch.float64, device="cuda")
            g.gmres(b, restart=30, tol=1e-8)
            _, sst = g.gmres(b, restart=30, tol=1e-8)
            ya = g.apply_tensor(b)
            torch.cuda.synchronize()
            ea0, ea1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea0.record()
            for _ in range(5):
                ya = g.apply_tensor(b)
            ea1.record()
            torch.cuda.synchronize()
            out["solve"] = {"gmres_iterations": int(sst["iterations"]), "converged": bool(sst["converged"]),
                            "rel_residual": sst["rel_residual"], "gmres_ms": sst["t_solve_ms"],
                            "apply_ms": ea0.elapsed_time(ea1) / 5}
        if dist_apply is not None:
            out["solve"] = dist_apply
        if not use_dist and not args.no_extra:
            g.close()   # c2's zone panels (38 GB) go back before the other configs are set up
            out["extra_configs"] = {c: time_config(c, args.steps, args.warmup, flush) for c in ("c3", "c4", "c5")}
        if extra_dist is not None:
            out["extra_configs"] = extra_dist
        if not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(P)
        print(json.dumps(out), flush=True)
    g.close()
    if world > 1 or args.dist:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
