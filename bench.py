#!/usr/bin/env python
"""Benchmark: ms per MPC solve (and per IPM iteration) of the condensed-space IPM.

Workload (N=1 default): BASELINE.json config 3, the 2-D heat-equation MPC (50 x 50 copper
plate, n_x = 2500, n_u = 10, T = 50 -> n = 500 controls, m = 251,000 inequality rows).
A "step" is one complete ipm::solve (proj/src/ipm.cpp:160-268) of that QP, tol 1e-8.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config c3]

value: device time of K solves with the QP resident in HBM (CUDA events on the solve's
stream, max over ranks). e2e: the same metric through the public API
(paper_2209_13049_b200.ipm.solve on a fresh DenseQp whose arrays sit in pinned host
memory): H2D upload + structure analysis + solve + D2H of the iterate + trajectory recovery,
wall clock. N > 1 (torchrun): configs 3/4 shard the rows of J across the ranks (one solve per
step, NCCL allreduces inside the iteration graphs -> strong scaling; --mode replica instead
solves an independent instance per rank -> weak scaling); config 5 splits the 1024-instance
batch across the ranks (no collective in the loop).
--impl reference: the oracle (CPU restatement of the reference solver) on all the box's host
cores, one whole solve per timed step (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.1   # measured DMMA (mma.sync f64) peak, profiles/r01_fp64_peak_probe.txt
CONFIGS = {
    "c1": dict(desc="config 1: random LQ-MPC n_x=10, n_u=2, T=10 (instance_rng(42, 0))"),
    "c2": dict(desc="config 2: 1-D heat rod MPC n_x=200, n_u=4, T=50 (n=200, m=20,400)"),
    "c3": dict(desc="config 3: 2-D heat plate MPC 50x50, n_x=2500, n_u=10, T=50 (n=500, m=251,000)"),
    "c4": dict(desc="config 4: long-horizon 2-D heat 40x25, n_x=1000, n_u=10, T=200 (n=2000, m=404,000)"),
    "c5": dict(desc="config 5: batch of 1024 independent 2-D heat MPC instances 20x25, n_x=500, n_u=5, "
                    "T=30 (n=150, m=30,300), initial temperature 300 K + U[-20,20] per cell, split across GPUs"),
}


C4_T = 200  # config 4's horizon (--T: the sweep 50, 100, 150, 200)


def build_problem(cfg, rank=0):
    from paper_2209_13049_b200 import problem as P
    if cfg == "c1":
        from oracle import oracle as O  # only the C1 random generator lives in the oracle
        p = O.random_problem(O.instance_rng(42, rank), fixed=(10, 2, 0, 10))
        d = p.as_dict()
        T = d.pop("T")
        data = P.LqProblemData(T=T, **d)
    elif cfg == "c2":
        data = P.heat1d_problem(200, 50)
    elif cfg == "c3":
        data = P.heat2d_problem(50, 50, T=50)
    elif cfg == "c4":
        data = P.heat2d_problem(40, 25, T=C4_T)
    elif cfg == "c5":
        data = P.heat2d_problem(20, 25, T=30)
    else:
        raise SystemExit(f"unknown config {cfg}")
    if rank > 0 and cfg != "c1":
        data.x_bar = P.batch_initial_states(data.A.shape[0], 1, seed=1000 + rank)[0]
    return data


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the first line takes nvidia-smi's start-up: wait for it so that the sampling is live
            # when the timed region starts (a short region would otherwise see no sample at all)
            t0 = time.perf_counter()
            while not self.samples and time.perf_counter() - t0 < 3.0:
                time.sleep(0.01)
            self.n0 = len(self.samples)
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            # a region shorter than the 200 ms period: the next sample, right at its end
            t0 = time.perf_counter()
            while len(self.samples) <= self.n0 and time.perf_counter() - t0 < 1.0:
                time.sleep(0.005)
            self.samples = self.samples[self.n0:]  # (taken from the region's start on)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return None
        sm = [float(s[1]) for s in self.samples if len(s) > 8 and s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if len(s) > 8 and s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            if len(s) > 8:
                for nm, v in zip(names, s[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def pinned_like(a):
    """copy into page-locked host memory (torch is used only as the allocator)."""
    import torch
    t = torch.empty(a.shape[::-1] if a.flags.f_contiguous and a.ndim == 2 else a.shape,
                    dtype=torch.float64, pin_memory=True)
    out = t.numpy()
    if a.ndim == 2 and a.flags.f_contiguous:
        out = out.T  # Fortran-ordered view of the pinned buffer
    out[...] = a
    return out


def host_cpu():
    """CPU model and logical core count of the host the CPU arms run on."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count() or 1}


def bench_config(cfg, qp, world, mode):
    """The `config` dict both arms print (same workload -> same dict)."""
    if world == 1:
        par = "single instance"
    elif mode == "shard":
        par = (f"rows of J sharded across {world} GPU(s) by whole stages; partial J_g' Sigma_g J_g "
               f"+ row reductions allreduced (NCCL)")
    else:
        par = f"{world} independent instances (one per GPU)"
    return {"workload": CONFIGS[cfg]["desc"], "n": qp.n, "m": qp.m, "tol": 1e-8,
            "parallelism": par,
            "l2": "inputs larger than L2 (J %.2f GB dense)" % (8.0 * qp.m * qp.n / 1e9)
                  if 8.0 * qp.m * qp.n > 126e6 else "L2 flushed between steps (256 MB write)"}


def cpu_sample(qp, threads, iters_full, full_budget_s=25.0):
    """Oracle (reference restatement) on the host cores. A one-iteration warm-up (thread pool,
    page faults) is timed and discarded; then a whole solve when it fits the budget (config 1,
    2, 5 instances), else one more iteration scaled by the iteration count (bounded sample)."""
    from oracle import oracle as O
    O.set_threads(threads)
    oq = O.qp_from_arrays(qp.H, qp.h, qp.h0, qp.J, qp.d)
    O.solve(oq, max_iter=1, log=False)  # warm-up
    t = time.perf_counter()
    r0 = O.solve(oq, max_iter=1, log=False)
    dt = time.perf_counter() - t
    if dt * iters_full <= full_budget_s:
        t = time.perf_counter()
        r = O.solve(oq, log=False)
        full = time.perf_counter() - t
        return dict(ms_per_iter=full * 1e3 / max(r.iter, 1), ms_per_solve=full * 1e3, status=r.status,
                    sample=f"one whole solve ({r.iter} iterations)")
    return dict(ms_per_iter=dt * 1e3, ms_per_solve=dt * 1e3 * iters_full, status=r0.status,
                sample=f"one IPM iteration x{iters_full} iterations")


def run_reference(args, rank, world):
    """The reference CPU path: the oracle (C++ restatement of proj/src/ipm.cpp +
    dense_linalg.cpp; the reference itself needs Eigen3, absent here and on the box) on
    all host cores. Each timed step is one WHOLE solve of the config's QP (dense J, as the
    reference multiplies it); warm-up steps are one IPM iteration each (untimed, they only
    warm the thread pool and the page cache). Rank 0 alone runs it."""
    if rank != 0:
        return None
    from oracle import oracle as O
    from paper_2209_13049_b200 import problem as P
    cfg = args.config
    mode = args.mode if args.mode != "auto" else ("shard" if cfg in ("c3", "c4") and world > 1 else "replica")
    qp = P.build_dense_qp(build_problem(cfg))
    threads = os.cpu_count() or 1
    O.set_threads(threads)
    O.set_skip_zeros(False)
    oq = O.qp_from_arrays(qp.H, qp.h, qp.h0, qp.J, qp.d)
    for _ in range(args.warmup):
        O.solve(oq, max_iter=1, log=False)
    times, iters, status = [], [], None
    wall = time.perf_counter()
    for _ in range(args.steps):
        t = time.perf_counter()
        r = O.solve(oq, log=False)
        times.append((time.perf_counter() - t) * 1e3)
        iters.append(r.iter)
        status = r.status
    wall = time.perf_counter() - wall
    ms = float(np.mean(times))
    # the reference's own build is single-threaded Eigen (-O3, no -march: proj/CMakeLists.txt:8-9):
    # one iteration of the same QP on one thread, scaled by the solve's iteration count
    O.set_threads(1)
    t = time.perf_counter()
    O.solve(oq, max_iter=1, log=False)
    st_iter = (time.perf_counter() - t) * 1e3
    O.set_threads(threads)
    cpu = host_cpu()
    line = {"impl": "reference", "metric": "ms per MPC solve", "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": False,
            "scaling": "strong" if (world > 1 and mode == "shard") else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(cfg, qp, world, mode),
            "value": ms, "ms_per_step": ms, "ms_per_iter": ms / max(float(np.mean(iters)), 1.0),
            "iterations": iters[-1], "status": status, "samples_ms": [round(x, 1) for x in times],
            "wall_s": wall,
            "cpu_baseline": {"value": ms, "unit": "ms", "cores": threads, "kind": "port",
                             "cpu": cpu,
                             "sample": f"{args.steps} whole solves ({iters[-1]} IPM iterations each) of "
                                       f"the full {cfg} QP by the oracle (CPU restatement of "
                                       f"proj/src/ipm.cpp + dense_linalg.cpp, dense J, OpenMP over "
                                       f"independent output entries) on {threads} threads; warm-up "
                                       f"steps are one iteration each"},
            "single_thread": {"ms_per_iter": st_iter, "ms_per_solve_extrapolated": st_iter * iters[-1],
                              "sample": "one IPM iteration on 1 thread (the reference's own "
                                        "single-threaded build), x the solve's iteration count"},
            "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


def run_shard(args, rank, world, local, dist):
    """Configs 3/4 at N GPUs: the rows of J split across the ranks by whole stages
    (problem.shard_rows), one solve per step: every rank condenses its rows, the partial
    condensed matrices and the row reductions are allreduced over NVLink (NCCL, captured in
    the iteration's CUDA graphs), and the Cholesky + solve run redundantly. value = ms per
    solve (strong scaling: the whole QP is fixed), max over ranks."""
    import torch
    from paper_2209_13049_b200 import _lib, ipm, problem as P
    cfg = args.config
    qp = P.build_dense_qp(build_problem(cfg, 0))  # the same QP on every rank
    uid = ipm.nccl_unique_id() if rank == 0 else None
    if dist:
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    rows = P.shard_rows(qp, world)[rank]
    sh = ipm.ShardedQp(qp, rows, uid, world, rank)
    info = sh.dq.info()
    opts = ipm.IpmOptions()

    def barrier():
        torch.cuda.synchronize(local)
        if dist:
            dist.barrier()

    for _ in range(args.warmup):
        r = sh.solve(opts)
    barrier()
    l0 = _lib.launch_count()
    dev_s, syrk_s, syrk_n, chol_s, iters = 0.0, 0.0, 0, 0.0, []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            r = sh.solve(opts)
            dev_s += r.device_seconds
            syrk_s += r.syrk_seconds
            syrk_n += r.condensations
            chol_s += r.chol_seconds
            iters.append(r.iter)
    barrier()
    launches = _lib.launch_count() - l0

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms_total = max_over_ranks(dev_s) * 1e3
    e2e = None
    if not args.no_e2e:
        loc = sh.local
        pin = P.DenseQp(H=pinned_like(loc.H), h=pinned_like(loc.h), h0=loc.h0,
                        J=pinned_like(loc.J), d=pinned_like(loc.d))
        e2e_ms = []
        for k in range(args.warmup + args.steps):
            barrier()
            t0 = time.perf_counter()
            sh.reload(P.DenseQp(H=pin.H, h=pin.h, h0=pin.h0, J=pin.J, d=pin.d))
            re = sh.solve(opts)
            if rank == 0:
                P.recover_trajectory(qp, re.v)
            torch.cuda.synchronize(local)
            dt = time.perf_counter() - t0
            if k >= args.warmup:
                e2e_ms.append(dt * 1e3)
        e2e_tot = max_over_ranks(float(np.sum(e2e_ms)))
        n, m = loc.n, loc.m
        e2e = {"value": e2e_tot / args.steps, "unit": "ms",
               "h2d_bytes_per_step": int(8 * (n * n + n + m * n + m)),
               "d2h_bytes_per_step": int(8 * (n + 3 * m)),
               "median_ms": statistics.median(e2e_ms), "samples_ms": [round(x, 2) for x in e2e_ms],
               "status": re.status.name, "iterations": re.iter,
               "note": "per rank: its rows of J, d (pinned host) + H, h; max over ranks"}
    syrk_max = max_over_ranks(syrk_s)
    if rank != 0:
        sh.close()
        if dist:
            dist.destroy_process_group()
        return
    flops_rank0 = info["syrk_flops"]
    line = {
        "metric": "ms per MPC solve", "value": ms_total / args.steps, "unit": "ms", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": bench_config(cfg, qp, world, "shard"),
        "structure": {"rows_rank0": int(len(rows)), "prototype_rows_rank0": info["prototypes"]},
        "ms_per_iter": ms_total / max(sum(iters), 1), "iterations": iters[-1], "status": r.status.name,
        "roofline": {"bound": "tensor", "kernel": "k_syrk + k_syrk_reduce (rank 0's rows)",
                     "achieved": flops_rank0 / (syrk_s / max(syrk_n, 1)) / 1e12,
                     "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": flops_rank0 / (syrk_s / max(syrk_n, 1)) / 1e12 / FP64_PEAK_TFLOPS,
                     "peak_source": "measured FP64 DMMA peak, profiles/r01_fp64_peak_probe.txt",
                     "algorithmic_flops_per_launch": flops_rank0,
                     "avg_launch_ms": syrk_s / max(syrk_n, 1) * 1e3,
                     "share_of_step": syrk_max / max(dev_s, 1e-30), "traffic": None},
        "phase_ms_per_iter": {"condense": syrk_s * 1e3 / max(sum(iters), 1),
                              "cholesky": chol_s * 1e3 / max(sum(iters), 1)},
        "gpu_launches": launches, "clocks": clk.summary(), "e2e": e2e,
    }
    print(json.dumps(line), flush=True)
    sh.close()
    if dist:
        dist.destroy_process_group()


def run_batch(args, rank, world, local, dist):
    """config 5: 1024 instances split across the ranks; each rank solves its share as one
    lockstep batch (ipm.BatchSolver: one host loop, every kernel over all its instances; H and
    J shared, per-instance h, h0, d). A step = the whole batch. No collective in the loop."""
    import torch
    from paper_2209_13049_b200 import _lib, ipm, linalg, problem as P
    linalg.DEVICE = local
    from paper_2209_13049_b200 import batch
    total = 1024
    first, share = batch.shard_range(total, world, rank)
    data = P.heat2d_problem(20, 25, T=30)
    base = P.build_dense_qp(data)
    xbs = P.batch_initial_states(500, total, seed=42)[first:first + share]
    bs = ipm.BatchSolver(base, share)
    for i, xb in enumerate(xbs):
        bs.set_instance(i, *batch.instance_affine(base, xb))
    opts = ipm.IpmOptions()

    def barrier():
        torch.cuda.synchronize(local)
        if dist:
            dist.barrier()

    for _ in range(args.warmup):
        res = bs.solve(opts)
    barrier()
    l0 = _lib.launch_count()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters, biters, cstats = [], [], []
    with ClockSampler(local) as clk:
        st.record()
        for _ in range(args.steps):
            res = bs.solve(opts)
            iters.append(float(np.mean(res.iter)))
            ls = getattr(bs, "last_stats", {})
            biters.append(ls.get("batch_iterations", int(np.max(res.iter))))
            cstats.append(ls)
        torch.cuda.synchronize(local)
        en.record()
        en.synchronize()
    ms_local = st.elapsed_time(en)
    launches = _lib.launch_count() - l0
    ms = ms_local
    if dist:
        t = torch.tensor([ms_local], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # end to end: the instances' (h, h0, d) uploaded from host memory every step
    e2e = None
    if not args.no_e2e:
        e2e_ms = []
        for k in range(args.warmup + args.steps):
            barrier()
            t0 = time.perf_counter()
            bs._dirty = True  # re-upload h, h0, d (host -> device) inside the timed region
            re = bs.solve(opts)
            torch.cuda.synchronize(local)
            if k >= args.warmup:
                e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_local = float(np.sum(e2e_ms))
        if dist:
            t = torch.tensor([e2e_local], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_local = float(t.item())
        e2e = {"value": e2e_local / (args.steps * total), "unit": "ms",
               "h2d_bytes_per_step": int(8 * share * (base.n + 1 + base.m)),
               "d2h_bytes_per_step": int(8 * share * (base.n + 14)),
               "samples_ms": [round(x, 2) for x in e2e_ms],
               "note": "ms per solve: the batch's h, h0, d uploaded and v + scalars read back every step"}
    if rank != 0:
        bs.close()
        return
    conv = sum(1 for x in res.status if x == "converged")
    line = {
        "metric": "ms per MPC solve", "value": ms / (args.steps * total), "unit": "ms",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": CONFIGS["c5"]["desc"], "instances": total, "per_gpu": share,
                   "parallelism": f"batch split across {world} GPU(s); lockstep batch per GPU ({bs.mode})"},
        "mean_iterations": float(np.mean(iters)), "converged": conv, "instances_on_rank0": share,
        "batch_iterations": int(biters[-1]),
        "ms_per_batch_iteration": ms / args.steps / max(1, biters[-1]),
        "gpu_launches": launches, "clocks": clk.summary(), "e2e": e2e,
    }
    if cstats and "condense_seconds" in cstats[-1]:
        # the lockstep condensation kernel (csrc/bsyrk.cu): its algorithmic FLOPs (sum over the
        # SYRK rows of hi (hi + 1) per instance it covered) over its CUDA-event time in the solves
        sec = sum(c["condense_seconds"] for c in cstats)
        nl = sum(c["condense_launches"] for c in cstats)
        flops = sum(c["condense_instances"] * c["condense_flops_per_instance"] for c in cstats)
        achieved = flops / sec / 1e12 if sec > 0 else 0.0
        line["roofline"] = {
            "bound": "tensor", "kernel": "k_bsyrk (lockstep condensation, one CTA per instance)",
            "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
            "peak_source": "measured FP64 DMMA peak (profiles/r01_fp64_peak_probe.txt)",
            "algorithmic_flops_per_launch": flops / max(1, nl), "avg_launch_ms": sec * 1e3 / max(1, nl),
            "share_of_step": sec * 1e3 / ms if ms > 0 else None, "traffic": None}
    if not args.no_cpu_baseline and world == 1:
        one = P.build_dense_qp(data)
        s_ = cpu_sample(one, os.cpu_count() or 1, int(round(float(np.mean(iters)))))
        line["cpu_baseline"] = {
            "value": s_["ms_per_solve"], "unit": "ms", "cores": os.cpu_count() or 1, "kind": "port",
            "cpu": host_cpu(),
            "sample": f"the oracle on one config-5 instance (dense J): {s_['sample']}; ms per instance solve"}
    print(json.dumps(line), flush=True)
    bs.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--T", type=int, default=200, help="config 4's horizon (50, 100, 150, 200)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-markov", action="store_true",
                    help="skip the device-built (Markov table) leg")
    ap.add_argument("--mode", default="auto", choices=["auto", "shard", "replica"],
                    help="N > 1: shard = rows of J split across the GPUs, one solve (configs 3/4, "
                         "the default there); replica = an independent instance per GPU")
    args = ap.parse_args()
    global C4_T
    C4_T = args.T
    if args.config == "c4" and args.T != 200:
        CONFIGS["c4"] = dict(desc=f"config 4: long-horizon 2-D heat 40x25, n_x=1000, n_u=10, T={args.T} "
                                  f"(n={10 * args.T}, m={2020 * args.T:,})")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1 and args.impl != "reference":
        from paper_2209_13049_b200.ipm import NCCL_DETERMINISM
        for k, v in NCCL_DETERMINISM.items():  # before any communicator exists
            os.environ.setdefault(k, v)
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    if args.impl == "reference":
        line = run_reference(args, rank, world)
        if line:
            print(json.dumps(line), flush=True)
        if dist:
            dist.destroy_process_group()
        return

    import torch
    from paper_2209_13049_b200 import _lib, ipm, linalg, problem as P
    linalg.DEVICE = local
    cfg = args.config
    if cfg == "c5":
        return run_batch(args, rank, world, local, dist)
    mode = args.mode if args.mode != "auto" else ("shard" if cfg in ("c3", "c4") and world > 1 else "replica")
    if mode == "shard":
        return run_shard(args, rank, world, local, dist)
    data = build_problem(cfg, rank)
    qp = P.build_dense_qp(data)
    dq = ipm.DeviceQp(qp, device=local)
    qp._device, qp._device_key = dq, qp.device_key()
    info = dq.info()
    opts = ipm.IpmOptions()

    def barrier():
        torch.cuda.synchronize(local)
        if dist:
            dist.barrier()

    for _ in range(args.warmup):
        r = ipm.solve_loaded(dq, qp, opts)
    barrier()
    l0 = _lib.launch_count()
    dev_s, syrk_s, syrk_n, chol_s, iters, wall = 0.0, 0.0, 0, 0.0, [], time.perf_counter()
    syrk_k = 0.0
    # inputs smaller than L2 (configs 1, 2): a 256 MB write between the timed solves (the
    # solve's own CUDA events exclude it)
    flush = None
    if 8.0 * qp.m * qp.n <= 126e6:
        flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device=f"cuda:{local}")
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            if flush is not None:
                flush.fill_(float(k))
                torch.cuda.synchronize(local)  # the solve runs on its own non-blocking stream
            r = ipm.solve_loaded(dq, qp, opts)
            dev_s += r.device_seconds
            syrk_s += r.syrk_seconds
            syrk_k += r.syrk_kernel_seconds
            syrk_n += r.condensations
            chol_s += r.chol_seconds
            iters.append(r.iter)
    barrier()
    wall = time.perf_counter() - wall
    launches = _lib.launch_count() - l0
    status = r.status.name
    t_local = dev_s
    if dist:
        t = torch.tensor([dev_s], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s = float(t.item())
    ms_total = dev_s * 1e3
    ms_per_step = ms_total / args.steps
    value = ms_total / (args.steps * world)  # whole job: ms per solve over all ranks

    # end to end through the public API with host (pinned) buffers. The resident context of
    # the device-timed loop is released first: a second loaded 1.5 GB context in the process
    # made the pinned 1 GB H2D and the pool allocations of each fresh context erratic
    # (21-35 ms instead of 18 ms, occasional 0.6 s stalls; tools/e2e_probe2.py)
    dq.close()
    qp._device = None
    e2e = None
    if not args.no_e2e:
        pin = dict(H=pinned_like(qp.H), h=pinned_like(qp.h), J=pinned_like(qp.J), d=pinned_like(qp.d))
        e2e_ms = []
        for k in range(args.warmup + args.steps):
            fresh = P.DenseQp(H=pin["H"], h=pin["h"], h0=qp.h0, J=pin["J"], d=pin["d"],
                              source=qp.source, gk=qp.gk, x0=qp.x0)
            barrier()
            t0 = time.perf_counter()
            re = ipm.solve(fresh, opts)
            torch.cuda.synchronize(local)
            dt = time.perf_counter() - t0
            fresh.invalidate_device()
            if k >= args.warmup:
                e2e_ms.append(dt * 1e3)
        e2e_local = float(np.sum(e2e_ms))
        if dist:
            t = torch.tensor([e2e_local], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_local = float(t.item())
        n, m = qp.n, qp.m
        e2e = {"value": e2e_local / (args.steps * world), "unit": "ms",
               "h2d_bytes_per_step": int(8 * (n * n + n + m * n + m)),
               "d2h_bytes_per_step": int(8 * (n + 3 * m)),
               "median_ms": statistics.median(e2e_ms), "samples_ms": [round(x, 2) for x in e2e_ms],
               "status": re.status.name,
               "iterations": re.iter}
        # the same from ordinary (pageable) numpy arrays, as a drop-in caller hands Eigen
        # storage: the library stages them through its pinned slots (a few samples, reported
        # beside the contract's pinned figure)
        pg_ms = []
        for k in range(1 + min(args.steps, 3)):
            fresh = P.DenseQp(H=qp.H.copy(), h=qp.h.copy(), h0=qp.h0, J=qp.J.copy(), d=qp.d.copy(),
                              source=qp.source, gk=qp.gk, x0=qp.x0)
            barrier()
            t0 = time.perf_counter()
            ipm.solve(fresh, opts)
            torch.cuda.synchronize(local)
            dt = time.perf_counter() - t0
            fresh.invalidate_device()
            if k >= 1:
                pg_ms.append(dt * 1e3)
        e2e["pageable_median_ms"] = statistics.median(pg_ms)
        e2e["pageable_samples_ms"] = [round(x, 2) for x in pg_ms]

    # end to end from the structured problem: host LqProblemData ->
    # dense QP built and analysed on the device -> solve -> trajectory recovered on the device
    e2e_problem = None
    if not args.no_e2e:
        pb_ms = []
        for k in range(1 + min(args.steps, 5)):
            barrier()
            t0 = time.perf_counter()
            rp = ipm.solve_problem(data, opts)
            torch.cuda.synchronize(local)
            if k >= 1:
                pb_ms.append((time.perf_counter() - t0) * 1e3)
        nbytes = sum(int(np.asarray(getattr(data, f)).nbytes) for f in
                     ("A", "B", "Q", "Qf", "R", "S", "E", "F", "gl", "gu", "xl", "xu", "ul", "uu",
                      "w", "x_bar", "K"))
        e2e_problem = {"value": statistics.median(pb_ms), "unit": "ms", "h2d_bytes_per_step": nbytes,
                       "d2h_bytes_per_step": int(8 * (rp.solution.x.size + rp.solution.u.size + qp.n + 3 * qp.m)),
                       "samples_ms": [round(x, 2) for x in pb_ms], "iterations": rp.iter,
                       "status": rp.status.name,
                       "note": "build_dense_qp + solve + recover_trajectory on the device (median); "
                               "the reference cannot build this QP (bigAtilde alone is 127 GB at config 3)"}

    # the same QP built on the device with the Markov table as the prototype source (SURVEY
    # §8(f) row 2: P never stored), device-resident solves timed like the main leg
    markov = None
    if not args.no_markov and cfg in ("c2", "c3", "c4", "c5"):
        dqm = ipm.DeviceQp.from_problem(data, device=local, options={"markov": 2})
        mi = dqm.info()
        if mi["markov"]:
            for _ in range(min(args.warmup, 2)):
                ipm.solve_loaded(dqm, None, opts)
            md, mk_k, mk_n, mit = 0.0, 0.0, 0, 0
            for _ in range(args.steps):
                rm = ipm.solve_loaded(dqm, None, opts)
                md += rm.device_seconds
                mk_k += rm.syrk_kernel_seconds
                mk_n += rm.condensations
                mit = rm.iter
            kk = mk_k / max(mk_n, 1)
            markov = {"ms_per_solve": md * 1e3 / args.steps, "iterations": mit, "status": rm.status.name,
                      "syrk_avg_launch_ms": kk * 1e3,
                      "syrk_frac": mi["syrk_flops"] / kk / 1e12 / FP64_PEAK_TFLOPS,
                      "table_mb": mi["stored_bytes"] / 1e6, "table_rows": mi["markov_rows"],
                      "table_cols": mi["markov_cols"], "p_mb_not_stored": info["p_bytes"] / 1e6,
                      "note": "QP built on the device (cmpc_build_qp, option markov = 2); the SYRK and the "
                              "P products read the Markov table of B-responses, P is never stored "
                              "(csrc/markov.cu). The default (markov = 1) uses the table when P would "
                              "exceed 64 MB (configs 3, 4)"}
        dqm.close()

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    avg_syrk_s = syrk_s / max(syrk_n, 1)
    avg_syrk_k = syrk_k / max(syrk_n, 1)
    small = syrk_n == 0  # the one-CTA solver (csrc/small.cu): the whole solve is one kernel
    if small:
        # its condensation FLOPs per solve over the kernel's whole (latency-bound) duration
        avg_syrk_k = avg_syrk_s = ms_total * 1e-3 / max(args.steps, 1)
        flops_launch = info["syrk_flops"] * iters[-1]
    else:
        flops_launch = info["syrk_flops"]
    achieved = flops_launch / avg_syrk_k / 1e12
    line = {
        "metric": "ms per MPC solve", "value": value, "unit": "ms", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": bench_config(cfg, qp, world, mode),
        "structure": {"prototype_rows": info["prototypes"], "syrk_rows": info["syrk_prototypes"],
                      "p_mb": info["p_bytes"] / 1e6},
        "ms_per_iter": ms_total / max(sum(iters), 1) * (1 if world == 1 else 1),
        "iterations": iters[-1], "status": status,
        "roofline": {"bound": "tensor",
                     "kernel": ("k_small_ipm (the whole solve in one CTA: latency-bound; its condensation "
                                "FLOPs over its duration)") if small else
                               "k_syrk (the condensation's SYRK, right-hand side fused)",
                     "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP64_PEAK_TFLOPS,
                     "peak_source": "measured FP64 DMMA peak (mma.sync m16n8k16.f64, "
                                    "profiles/r01_fp64_peak_probe.txt); MEASURED_PEAKS.json has no FP64 entry",
                     "algorithmic_flops_per_launch": flops_launch,
                     "avg_launch_ms": avg_syrk_k * 1e3,
                     "condensation_ms": avg_syrk_s * 1e3,
                     "condensation_frac": flops_launch / avg_syrk_s / 1e12 / FP64_PEAK_TFLOPS,
                     "share_of_step": syrk_k / max(t_local, 1e-30),
                     "traffic": None},
        "phase_ms_per_iter": {"condense": syrk_s * 1e3 / max(sum(iters), 1),
                              "cholesky": chol_s * 1e3 / max(sum(iters), 1)},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "e2e": e2e,
        "e2e_from_problem": e2e_problem,
        "markov": markov,
        "wall_s": wall,
    }
    if not args.no_cpu_baseline and world == 1:
        s = cpu_sample(qp, os.cpu_count() or 1, r.iter)
        line["cpu_baseline"] = {
            "value": s["ms_per_solve"], "unit": "ms", "cores": os.cpu_count() or 1, "kind": "port",
            "cpu": host_cpu(),
            "sample": f"the oracle (CPU restatement of proj/src/ipm.cpp + dense_linalg.cpp, dense J) "
                      f"on the same QP: {s['sample']}"}
    traffic = os.path.join(ROOT, "profiles", f"syrk_traffic_{cfg}.json")
    if os.path.exists(traffic):
        line["roofline"]["traffic"] = json.load(open(traffic)).get("dram_bytes_per_launch")
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
