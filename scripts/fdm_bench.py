"""c4 element-block preconditioner apply (CUDA events, rotating buffers) and
warm slab-solve times.  Prints one JSON object."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200 import _lib as L  # noqa: E402
from paper_2201_05800_b200.api import NewtonConfig, SlabOperator  # noqa: E402

cfg = C.CONFIGS["c4"]
op = SlabOperator(**cfg.kwargs())
X = [torch.as_tensor(C.random_slab(cfg), device="cuda") for _ in range(3)]
Y = [torch.empty_like(x) for x in X]
out = {}
for name, pc in (("eblock", L.STG_PRECOND_EBLOCK), ("tblock", L.STG_PRECOND_TBLOCK)):
    for k in range(3):
        op.st_precond_apply(cfg.dt, X[k], precond=pc, out=Y[k])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    reps = 60
    e0.record()
    for k in range(reps):
        op.st_precond_apply(cfg.dt, X[k % 3], precond=pc, out=Y[k % 3])
    e1.record()
    torch.cuda.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / reps
    out[name + "_us"] = us
    out[name + "_gbs"] = 16 * cfg.n_dof / us / 1e3
un = torch.as_tensor(C.initial_state(cfg), device="cuda")
for name, pc in (("eblock", L.STG_PRECOND_EBLOCK), ("tblock", L.STG_PRECOND_TBLOCK)):
    nc = NewtonConfig(abs_tol=0.0, rel_tol=1e-9, gmres_tol=1e-10, precond=pc)
    op.stdg_step(0.0, cfg.dt, un, nc)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        U, u1, info = op.stdg_step(0.0, cfg.dt, un, nc)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    out["solve_" + name + "_ms"] = 1e3 * sorted(ts)[2]
    out["solve_" + name + "_its"] = info.linear_iterations
print(json.dumps(out))
