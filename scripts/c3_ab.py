"""c3 (Burgers) 10-slab timing, fused vs host-driven FD Jacobian (same process)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200 import _lib as L  # noqa: E402
from paper_2201_05800_b200.api import NewtonConfig, SlabOperator  # noqa: E402

cfg = C.CONFIGS["c3"]
out = {}
for name, kern in (("fused", L.STG_KERNEL_AUTO), ("host", L.STG_KERNEL_GENERIC)):
    op = SlabOperator(**cfg.kwargs(), kernel=kern)
    u0 = torch.as_tensor(C.initial_state(cfg), device="cuda")
    nc = NewtonConfig(abs_tol=1e-12, rel_tol=1e-10, gmres_tol=1e-6, fd_eps=1e-7)
    op.stdg_step(0.0, cfg.dt, u0, nc)
    best = 1e9
    for _ in range(3):
        u = u0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(10):
            _, u, info = op.stdg_step(k * cfg.dt, cfg.dt, u, nc)
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) / 10)
    out[name] = {"ms_per_slab": 1e3 * best, "launches": op.kernel_launches()}
print(json.dumps(out))
