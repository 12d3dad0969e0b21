"""Host-buffer R(U) (c4) wall time per call: best of 3 rounds of 20 calls."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import SlabOperator  # noqa: E402

cfg = C.CONFIGS["c4"]
op = SlabOperator(**cfg.kwargs())
pin_U = torch.empty(cfg.n_dof, dtype=torch.float64, pin_memory=True)
pin_un = torch.empty(cfg.n_sdof, dtype=torch.float64, pin_memory=True)
pin_R = torch.empty(cfg.n_dof, dtype=torch.float64, pin_memory=True)
pin_U.copy_(torch.as_tensor(C.random_slab(cfg)))
pin_un.copy_(torch.as_tensor(C.initial_state(cfg)))
a, b, c = pin_un.numpy(), pin_U.numpy(), pin_R.numpy()
for _ in range(3):
    op.st_residual_host(0.0, cfg.dt, a, b, out=c)
best = 1e9
for _ in range(3):
    t0 = time.perf_counter()
    for _ in range(20):
        op.st_residual_host(0.0, cfg.dt, a, b, out=c)
    best = min(best, (time.perf_counter() - t0) / 20)
print(json.dumps({"ms": 1e3 * best, "dof_per_s": cfg.n_dof / best}))
