"""Host-buffer call times at c4 (best of 5 after a warm call, wall clock
around the blocking call): R(U), the slab step and the stage step from
page-locked and from pageable numpy arrays; pageable with the library's
worker-thread staging (default) and with the driver's own staging
(STG_HOST_NO_STAGING=1 in a second process).  Prints one JSON object.
  python scripts/host_paths.py [threads ...]"""
import json
import os
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def measure():
    import numpy as np
    import torch
    from paper_2201_05800_b200 import configs as C
    from paper_2201_05800_b200 import _lib as L
    from paper_2201_05800_b200.api import NewtonConfig, SlabOperator
    cfg = C.CONFIGS["c4"]
    op = SlabOperator(**cfg.kwargs())
    U, un = C.random_slab(cfg), C.initial_state(cfg)
    pin = lambda n: torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    pU, pu, pR, pu1 = pin(cfg.n_dof), pin(cfg.n_sdof), pin(cfg.n_dof), pin(cfg.n_sdof)
    pU[:] = U
    pu[:] = un
    R, u1 = np.empty(cfg.n_dof), np.empty(cfg.n_sdof)
    nc = NewtonConfig(abs_tol=0.0, rel_tol=1e-9, gmres_tol=1e-10)

    def best(fn, reps=5):
        fn()
        b = 1e9
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            b = min(b, time.perf_counter() - t0)
        return 1e3 * b
    out = {
        "residual_pinned_ms": best(lambda: op.st_residual_host(0.0, cfg.dt, pu, pU, out=pR)),
        "residual_pageable_ms": best(lambda: op.st_residual_host(0.0, cfg.dt, un, U, out=R)),
        "stdg_step_pinned_ms": best(lambda: op.stdg_step_host(0.0, cfg.dt, pu, nc, U=pR, u_next=pu1)),
        "stdg_step_pageable_ms": best(lambda: op.stdg_step_host(0.0, cfg.dt, un, nc, U=R, u_next=u1)),
        "rk_step_pageable_ms": best(lambda: op.rk_step_host(L.STG_FORM_A_INV, 0.0, cfg.dt, un, nc,
                                                            U=R, u_next=u1)),
    }
    a = np.empty(cfg.n_dof)
    out["numpy_copy_64MiB_ms"] = best(lambda: np.copyto(a, U))
    print(json.dumps(out))


if __name__ == "__main__":
    if os.environ.get("_HOST_PATHS_CHILD"):
        measure()
        sys.exit(0)
    res = {}
    variants = [("driver_staging", {"STG_HOST_NO_STAGING": "1"})]
    for t in (sys.argv[1:] or ["2", "4", "8", "16"]):
        variants.append((f"threads_{t}", {"STG_HOST_THREADS": t}))
    for name, env in variants:
        r = subprocess.run([sys.executable, __file__], capture_output=True, text=True,
                           env={**os.environ, **env, "_HOST_PATHS_CHILD": "1"}, timeout=900)
        res[name] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-400:]
    print(json.dumps(res))
