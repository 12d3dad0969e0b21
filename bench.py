#!/usr/bin/env python
"""Benchmark of the B200 space-time DG-SEM slab operator (BASELINE.json metric).

Workload (north star): c4 = 3-D + t linear advection, N = 3 in x, y, z, t,
32^3 elements x 1 time element per slab (8,388,608 DOF), dt = 0.002.
A "step" is one fused R(U) apply (st_residual, stdg.hpp:56-76) over the whole
slab with U ~ uniform[-1,1) (seed 3) and u_n = u0 at the LGL nodes.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  `value` = whole-job DOF-applications/s with
inputs resident in HBM (CUDA events on the launching stream, barrier + sync
on both sides, max over ranks).  `e2e` = the same metric through the C ABI's
host-buffer entry point (stg_st_residual_host: H2D of U and u_n from pinned
memory, apply, D2H of R, every step).  Multi-GPU runs are independent
replicas (the north star is one GPU).
`--impl reference` times the CPU oracle (the reference restated; the reference
itself cannot be built here) with all host threads on the same workload.
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
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fp64 space-time DG-SEM operator DOF/s & % HBM roofline; solve time/slab"
UNIT = "DOF/s"
WORKLOAD = "c4"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback (used only if MEASURED_PEAKS.json is absent)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                return
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def cpu_baseline(cfg, threads: int, budget_s: float):
    """Oracle R(U) on the host cores (bounded sample: whole applies until budget)."""
    import oracle as O
    O.set_threads(threads)
    pr = O.Problem(cfg.dim, cfg.degree, list(cfg.cells), list(cfg.lower), list(cfg.upper),
                   list(cfg.velocity), n_tau=cfg.n_tau)
    from paper_2201_05800_b200 import configs as C
    U = C.random_slab(cfg)
    un = C.initial_state(cfg)
    pr.st_residual(0.0, cfg.dt, un, U)  # warm-up
    n = 0
    t0 = time.perf_counter()
    while True:
        pr.st_residual(0.0, cfg.dt, un, U)
        n += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    el = time.perf_counter() - t0
    return n * cfg.n_dof / el, n, el


def run_reference(args):
    from paper_2201_05800_b200 import configs as C
    import oracle as O
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = C.CONFIGS[args.workload]
    threads = O.max_threads()
    O.set_threads(threads)
    pr = O.Problem(cfg.dim, cfg.degree, list(cfg.cells), list(cfg.lower), list(cfg.upper),
                   list(cfg.velocity), n_tau=cfg.n_tau)
    U = C.random_slab(cfg)
    un = C.initial_state(cfg)
    for _ in range(min(args.warmup, 2)):
        pr.st_residual(0.0, cfg.dt, un, U)
    budget = float(os.environ.get("STG_REF_BUDGET_S", "60"))
    n = 0
    t0 = time.perf_counter()
    while n < args.steps:
        pr.st_residual(0.0, cfg.dt, un, U)
        n += 1
        if time.perf_counter() - t0 >= budget:
            break
    el = time.perf_counter() - t0
    value = n * cfg.n_dof / el
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": n, "warmup": min(args.warmup, 2), "ms_per_step": 1e3 * el / n,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{cfg.name}: {cfg.note}", "n_dof": cfg.n_dof,
                   "cells": list(cfg.cells), "degree": cfg.degree, "n_tau": cfg.n_tau},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{n} full R(U) applies of {cfg.name} (capped at "
                                   f"{budget:.0f} s or --steps); reference unbuildable here "
                                   "(Eigen3 absent), oracle restatement timed instead"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    from paper_2201_05800_b200 import configs as C
    from paper_2201_05800_b200.api import NewtonConfig, SlabOperator

    ws, rank, local = dist_env()
    dist = None
    if ws > 1:
        import torch.distributed as dist  # noqa: F811
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    cfg = C.CONFIGS[args.workload]
    op = SlabOperator(**cfg.kwargs())
    stream = torch.cuda.current_stream()

    # inputs resident in HBM; rotate NSETS (U, u_n, R) sets so consecutive
    # applies never hit L2 (each set is 144 MiB > 126 MB L2)
    nsets = 3
    U0 = torch.as_tensor(C.random_slab(cfg), device=dev)
    un0 = torch.as_tensor(C.initial_state(cfg), device=dev)
    Us = [U0.clone() for _ in range(nsets)]
    uns = [un0.clone() for _ in range(nsets)]
    Rs = [torch.empty(cfg.n_dof, dtype=torch.float64, device=dev) for _ in range(nsets)]

    def step(i):
        k = i % nsets
        op.st_residual(0.0, cfg.dt, uns[k], Us[k], out=Rs[k])

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = op.kernel_launches()
    with ClockSampler(dev.index) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for i in range(args.steps):
            step(i)
        ev1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    launches = op.kernel_launches() - launches0
    ms = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = ws * cfg.n_dof * args.steps / (ms / 1e3)

    hbm, hbm_src = peaks()
    alg = C.residual_bytes(cfg)
    achieved = alg / (ms_step / 1e3) / 1e9
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get("slab3d_n4_tma")
        except Exception:
            traffic = None

    # ---- e2e through the reference-facing C-ABI host entry point -------------
    e2e_steps = max(3, min(args.steps, args.e2e_steps))
    pin_U = torch.empty(cfg.n_dof, dtype=torch.float64, pin_memory=True)
    pin_un = torch.empty(cfg.n_sdof, dtype=torch.float64, pin_memory=True)
    pin_R = torch.empty(cfg.n_dof, dtype=torch.float64, pin_memory=True)
    pin_U.copy_(U0.cpu())
    pin_un.copy_(un0.cpu())
    npU, npun, npR = pin_U.numpy(), pin_un.numpy(), pin_R.numpy()
    for _ in range(2):
        op.st_residual_host(0.0, cfg.dt, npun, npU, out=npR)
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        op.st_residual_host(0.0, cfg.dt, npun, npU, out=npR)
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_val = ws * cfg.n_dof * e2e_steps / e2e_s

    extra = {}
    if not args.no_extra and rank == 0:
        extra = extras(op, cfg, C, NewtonConfig, torch, dev, args)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        try:
            v, n, el = cpu_baseline(cfg, 1, args.cpu_budget)
            cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
                   "sample": f"{n} full R(U) applies of {cfg.name} ({el:.1f} s, 1 thread; the "
                             "reference is single-threaded, SPEC.md:426)"}
        except Exception as e:  # oracle missing on the box: report, do not fake
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "port",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.note}", "op": "st_residual R(U)",
                       "n_dof": cfg.n_dof, "cells": list(cfg.cells), "degree": cfg.degree,
                       "n_tau": cfg.n_tau, "parallelism": f"replicas{ws}",
                       "l2": f"{nsets} rotating (U,u_n,R) sets of "
                             f"{(2 * cfg.n_dof + cfg.n_sdof) * 8 / 2**20:.0f} MiB (> 126 MB L2)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "peak_source": hbm_src,
                         "algorithmic_bytes_per_launch": alg},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": UNIT, "steps": e2e_steps,
                    "h2d_bytes_per_step": 8 * (cfg.n_dof + cfg.n_sdof),
                    "d2h_bytes_per_step": 8 * cfg.n_dof,
                    "path": "stg_st_residual_host (pinned host buffers)"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "extra": extra,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def timed(fn, stream, torch, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def extras(op, cfg, C, NewtonConfig, torch, dev, args):
    """J.v and stage-apply throughput and the slab-solve time (not the headline)."""
    stream = torch.cuda.current_stream()
    out = {}
    U = torch.as_tensor(C.random_slab(cfg), device=dev)
    v = torch.as_tensor(C.random_slab(cfg, 99), device=dev)
    un = torch.as_tensor(C.initial_state(cfg), device=dev)
    R = torch.empty_like(U)
    hbm, _ = peaks()
    ms = timed(lambda: op.st_jvp(0.0, cfg.dt, None, v, out=R), stream, torch, 50)
    out["jvp"] = {"dof_per_s": cfg.n_dof / (ms / 1e3), "ms": ms,
                  "hbm_frac": C.jvp_bytes(cfg) / (ms / 1e3) / 1e9 / hbm}
    for form, name in ((1, "stage_residual_a_inv"), (0, "stage_residual_a")):
        ms = timed(lambda: op.stage_residual(form, 0.0, cfg.dt, un, U, out=R), stream, torch, 50)
        out[name] = {"dof_per_s": cfg.n_dof / (ms / 1e3), "ms": ms,
                     "hbm_frac": C.residual_bytes(cfg) / (ms / 1e3) / 1e9 / hbm}
    # one slab solve (GMRES(30), rel tol 1e-10), u_n resident, from guess 1 (x) u_n
    cfgn = NewtonConfig(abs_tol=0.0, rel_tol=1e-10, gmres_tol=1e-10, gmres_restart=30)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Us, un1, info = op.stdg_step(0.0, cfg.dt, un, cfgn)
    torch.cuda.synchronize()
    out["slab_solve"] = {"seconds": time.perf_counter() - t0, "gmres_tol": 1e-10,
                         "newton_iterations": info.newton_iterations,
                         "gmres_iterations": info.linear_iterations,
                         "final_residual_inf": info.final_residual}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default=WORKLOAD, choices=["c2", "c4"])
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
