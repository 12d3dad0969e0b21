"""Slab solve per preconditioner (warm, best of 5, device-resident u_n):
c4 / c2 slab, c5 stage solve, c3 first slab.  STG_POLY_TERMS sets m for
STG_PRECOND_POLY.  Usage: python scripts/poly_bench.py [names] -- prints JSON."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200 import _lib as L  # noqa: E402
from paper_2201_05800_b200.api import NewtonConfig, SlabOperator  # noqa: E402

names = sys.argv[1:] or ["c4", "c2", "c5", "c3"]
pcs = {"auto": L.STG_PRECOND_AUTO, "poly": L.STG_PRECOND_POLY}
out = {"m": int(os.environ.get("STG_POLY_TERMS", "7"))}
for name in names:
    cfg = C.CONFIGS[name]
    op = SlabOperator(**cfg.kwargs())
    u = torch.as_tensor(C.initial_state(cfg), device="cuda")
    res = {}
    sols = {}
    for pn, pc in pcs.items():
        if name == "c3":
            nc = NewtonConfig(abs_tol=1e-12, rel_tol=1e-10, gmres_tol=1e-6, fd_eps=1e-7, precond=pc)
        else:
            nc = NewtonConfig(abs_tol=0.0, rel_tol=1e-9, gmres_tol=1e-10, precond=pc)
        if name == "c5":
            fn = lambda: op.rk_step(L.STG_FORM_A_INV, 0.0, cfg.dt, u, nc)  # noqa: E731
        else:
            fn = lambda: op.stdg_step(0.0, cfg.dt, u, nc)  # noqa: E731
        fn()
        best, info, U = 1e9, None, None
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = fn()
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
            if el < best:
                best, info = el, r[-1]
                U = r[0].clone()
        sols[pn] = U
        res[pn] = {"ms": best * 1e3, "newton": info.newton_iterations,
                   "gmres": info.linear_iterations}
    res["max_rel_gap"] = float((sols["poly"] - sols["auto"]).abs().max() / sols["auto"].abs().max())
    out[name] = res
print(json.dumps(out))
