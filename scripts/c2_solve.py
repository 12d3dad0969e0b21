"""Warm c2 slab-solve timing per preconditioner.  Prints JSON."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200 import _lib as L  # noqa: E402
from paper_2201_05800_b200.api import NewtonConfig, SlabOperator  # noqa: E402

cfg = C.CONFIGS["c2"]
op = SlabOperator(**cfg.kwargs())
un = torch.as_tensor(C.initial_state(cfg), device="cuda")
out = {}
for name, pc in (("eblock", L.STG_PRECOND_EBLOCK), ("tblock", L.STG_PRECOND_TBLOCK)):
    nc = NewtonConfig(abs_tol=0.0, rel_tol=1e-9, gmres_tol=1e-10, precond=pc)
    op.stdg_step(0.0, cfg.dt, un, nc)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        U, u1, info = op.stdg_step(0.0, cfg.dt, un, nc)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    out[name] = {"ms": 1e3 * sorted(ts)[1], "gmres": info.linear_iterations}
x = torch.as_tensor(C.random_slab(cfg), device="cuda")
y = torch.empty_like(x)
for k in range(3):
    op.st_precond_apply(cfg.dt, x, precond=L.STG_PRECOND_EBLOCK, out=y)
print(json.dumps(out))
