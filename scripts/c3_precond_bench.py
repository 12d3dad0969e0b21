"""c3 (Burgers): 10 slabs of Newton-GMRES, wall time per slab."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import NewtonConfig, SlabOperator  # noqa: E402

cfg = C.CONFIGS["c3"]
op = SlabOperator(**cfg.kwargs())
un = torch.as_tensor(C.initial_state(cfg), device="cuda")
nc = NewtonConfig(abs_tol=1e-12, rel_tol=1e-10, gmres_tol=1e-6, fd_eps=1e-7)
op.stdg_step(0.0, cfg.dt, un, nc)
torch.cuda.synchronize()
t0 = time.perf_counter()
u = un
for k in range(10):
    _, u, info = op.stdg_step(k * cfg.dt, cfg.dt, u, nc)
torch.cuda.synchronize()
print(json.dumps({"c3_per_slab_ms": (time.perf_counter() - t0) * 100}))
