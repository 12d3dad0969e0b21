"""Why the bench's e2e leg reads slower than scripts/e2e_ab.py: time the
host-buffer R(U) call (c4, pinned) both ways in one process — CUDA events
around 50 back-to-back calls (the bench's leg) and wall clock per call —
and print every call's wall time so outliers show."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import SlabOperator  # noqa: E402

cfg = C.CONFIGS["c4"]
op = SlabOperator(**cfg.kwargs())
stream = torch.cuda.current_stream()
pU = torch.empty(cfg.n_dof, dtype=torch.float64, pin_memory=True)
pun = torch.empty(cfg.n_sdof, dtype=torch.float64, pin_memory=True)
pR = torch.empty(cfg.n_dof, dtype=torch.float64, pin_memory=True)
pU.copy_(torch.as_tensor(C.random_slab(cfg)))
pun.copy_(torch.as_tensor(C.initial_state(cfg)))
a, b, c = pun.numpy(), pU.numpy(), pR.numpy()
for _ in range(3):
    op.st_residual_host(0.0, cfg.dt, a, b, out=c)
torch.cuda.synchronize()
out = {}
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(stream)
    walls = []
    for _ in range(50):
        t0 = time.perf_counter()
        op.st_residual_host(0.0, cfg.dt, a, b, out=c)
        walls.append(1e3 * (time.perf_counter() - t0))
    e1.record(stream)
    torch.cuda.synchronize()
    w = np.array(walls)
    out[f"rep{rep}"] = {"events_ms_per_call": e0.elapsed_time(e1) / 50, "wall_mean": w.mean(),
                        "wall_min": w.min(), "wall_p50": float(np.median(w)), "wall_max": w.max(),
                        "slow_calls": int((w > 1.2 * w.min()).sum())}
print(json.dumps(out))
