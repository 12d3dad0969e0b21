"""Warm c4 slab solve (best of 10) with the AUTO (polynomial: coupled fdm3
applies) and EBLOCK (plain fdm3 applies) preconditioners, and the c5 stage
solve.  For A/B builds: STG_CUDA_LIB=<variant> python scripts/c4_precond_ab.py"""
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
u = torch.as_tensor(C.initial_state(cfg), device="cuda")
out = {}
for pn, pc in (("auto", L.STG_PRECOND_AUTO), ("eblock", L.STG_PRECOND_EBLOCK)):
    nc = NewtonConfig(abs_tol=0.0, rel_tol=1e-9, gmres_tol=1e-10, precond=pc)
    for kind, fn in (("c4", lambda: op.stdg_step(0.0, cfg.dt, u, nc)),
                     ("c5", lambda: op.rk_step(L.STG_FORM_A_INV, 0.0, cfg.dt, u, nc))):
        fn()
        best = 1e9
        for _ in range(10):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        out[f"{kind}_{pn}_ms"] = round(best * 1e3, 4)
print(json.dumps(out))
