"""Slab-solve timings for the BASELINE configs (device-resident; CUDA sync
around each solve).  Prints one JSON object."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200 import _lib as L  # noqa: E402
from paper_2201_05800_b200.api import NewtonConfig, SlabOperator  # noqa: E402


def t_solve(fn, reps=1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps, out


res = {}
names = sys.argv[1:] or ["c1", "c4", "c5", "c3", "c2"]
def run(name):
    cfg = C.CONFIGS[name]
    op = SlabOperator(**cfg.kwargs())
    un = torch.as_tensor(C.initial_state(cfg), device="cuda")
    if name == "c1":
        nc = NewtonConfig(abs_tol=0.0, rel_tol=1e-11, gmres_tol=1e-12)
        op.stdg_step(0.0, cfg.dt, un, nc)
        t, (U, u1, info) = t_solve(lambda: op.stdg_step(0.0, cfg.dt, un, nc), 5)
        # 1000 R(U) applies (latency-bound)
        Ur = torch.as_tensor(C.random_slab(cfg), device="cuda")
        R = torch.empty_like(Ur)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(1000):
            op.st_residual(0.0, cfg.dt, un, Ur, out=R)
        e1.record()
        torch.cuda.synchronize()
        res[name] = {"solve_s": t, "newton": info.newton_iterations,
                     "gmres": info.linear_iterations, "res_inf": info.final_residual,
                     "us_per_apply_1000": e0.elapsed_time(e1)}
    elif name in ("c2", "c4"):
        nc = NewtonConfig(abs_tol=0.0, rel_tol=1e-9, gmres_tol=1e-10)
        t, (U, u1, info) = t_solve(lambda: op.stdg_step(0.0, cfg.dt, un, nc))
        ms_op = None
        Ur = torch.as_tensor(C.random_slab(cfg), device="cuda")
        R = torch.empty_like(Ur)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(50):
            op.st_jvp(0.0, cfg.dt, None, Ur, out=R)
        e1.record()
        torch.cuda.synchronize()
        ms_op = e0.elapsed_time(e1) / 50
        res[name] = {"solve_s": t, "newton": info.newton_iterations,
                     "gmres": info.linear_iterations, "res_inf": info.final_residual,
                     "ms_per_gmres_it": 1e3 * t / max(info.linear_iterations, 1),
                     "ms_jvp": ms_op}
    elif name == "c5":
        nc = NewtonConfig(abs_tol=0.0, rel_tol=1e-9, gmres_tol=1e-10)
        t, (U, u1, info) = t_solve(lambda: op.rk_step(L.STG_FORM_A_INV, 0.0, cfg.dt, un, nc))
        res[name] = {"solve_s": t, "newton": info.newton_iterations,
                     "gmres": info.linear_iterations, "res_inf": info.final_residual}
    elif name == "c3":
        # inexact Newton: FD J.v (eps = 1e-7) limits the attainable linear
        # accuracy, so GMRES runs to a forcing tolerance of 1e-6
        nc = NewtonConfig(abs_tol=1e-12, rel_tol=1e-10, gmres_tol=1e-6, fd_eps=1e-7)
        u = un
        its = []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(10):
            U, u, info = op.stdg_step(k * cfg.dt, cfg.dt, u, nc)
            its.append((info.newton_iterations, info.linear_iterations))
        torch.cuda.synchronize()
        res[name] = {"ten_slabs_s": time.perf_counter() - t0, "per_slab_s":
                     (time.perf_counter() - t0) / 10, "newton_gmres_per_slab": its}
for name in names:
    try:
        run(name)
    except Exception as e:  # record and continue
        res[name] = {"error": str(e)}
    print(json.dumps({name: res[name]}), flush=True)
print(json.dumps(res))
