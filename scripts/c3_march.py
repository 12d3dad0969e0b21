"""c3 (1-D Burgers, 65,536 cells) marched 10 slabs on the device, per
preconditioner: best-of-3 wall time per slab and the (Newton, GMRES) counts.
Prints one JSON object.  Usage: python scripts/c3_march.py [precond ...]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200 import _lib as L  # noqa: E402
from paper_2201_05800_b200.api import NewtonConfig, SlabOperator  # noqa: E402

names = {"eblock": L.STG_PRECOND_EBLOCK, "sweep": L.STG_PRECOND_SWEEP, "auto": L.STG_PRECOND_AUTO}
sel = sys.argv[1:] or ["eblock", "sweep"]
cfg = C.CONFIGS["c3"]
op = SlabOperator(**cfg.kwargs())
u0 = torch.as_tensor(C.initial_state(cfg), device="cuda")
out = {}
for name in sel:
    nc = NewtonConfig(abs_tol=1e-12, rel_tol=1e-10, gmres_tol=1e-6, fd_eps=1e-7, precond=names[name])
    best, its, uend = 1e9, None, None
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        u, it = u0, []
        for k in range(10):
            _, u, inf = op.stdg_step(k * cfg.dt, cfg.dt, u, nc)
            it.append([inf.newton_iterations, inf.linear_iterations])
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if el < best:
            best, its, uend = el, it, u.clone()
    out[name] = {"per_slab_ms": best * 100, "newton_gmres": its}
    out.setdefault("_u", []).append(uend)
us = out.pop("_u")
if len(us) > 1:
    out["max_rel_gap"] = float((us[1] - us[0]).abs().max() / us[0].abs().max())
print(json.dumps(out))
