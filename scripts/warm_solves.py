"""Warm slab-solve wall times (best of 5 after a warm call; CUDA sync around
each): c4, c5 (A^-1 form), c2, and c3 as 10 sequential slabs.  Prints one
JSON object.  For A/B builds: STG_CUDA_LIB=<variant> python scripts/warm_solves.py"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200 import _lib as L  # noqa: E402
from paper_2201_05800_b200.api import NewtonConfig, SlabOperator  # noqa: E402


def best(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    b = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        b = min(b, time.perf_counter() - t0)
    return b


out = {}
nc = NewtonConfig(abs_tol=0.0, rel_tol=1e-9, gmres_tol=1e-10)
for name in ("c4", "c2"):
    cfg = C.CONFIGS[name]
    op = SlabOperator(**cfg.kwargs())
    un = torch.as_tensor(C.initial_state(cfg), device="cuda")
    out[name + "_ms"] = 1e3 * best(lambda: op.stdg_step(0.0, cfg.dt, un, nc))
    if name == "c4":
        out["c5_ms"] = 1e3 * best(lambda: op.rk_step(L.STG_FORM_A_INV, 0.0, cfg.dt, un, nc))
    del op
c3 = C.CONFIGS["c3"]
op3 = SlabOperator(**c3.kwargs())
u3 = torch.as_tensor(C.initial_state(c3), device="cuda")
nc3 = NewtonConfig(abs_tol=1e-12, rel_tol=1e-10, gmres_tol=1e-6, fd_eps=1e-7)


def ten():
    u = u3
    for k in range(10):
        _, u, _ = op3.stdg_step(k * c3.dt, c3.dt, u, nc3)


out["c3_per_slab_ms"] = 1e3 * best(ten, 3) / 10
print(json.dumps(out))
