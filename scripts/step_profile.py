"""Per-step device time of the bench loop (c4 R(U), 3 rotating sets): an
event between every step, after the same sync + gate as bench.py.  Shows
whether the first steps of a short timed region cost more than the steady
state.  Prints one JSON object."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import SlabOperator  # noqa: E402

cfg = C.CONFIGS["c4"]
op = SlabOperator(**cfg.kwargs())
U = [torch.as_tensor(C.random_slab(cfg), device="cuda").clone() for _ in range(3)]
un = [torch.as_tensor(C.initial_state(cfg), device="cuda").clone() for _ in range(3)]
R = [torch.empty(cfg.n_dof, dtype=torch.float64, device="cuda") for _ in range(3)]


def step(i):
    op.st_residual(0.0, cfg.dt, un[i % 3], U[i % 3], out=R[i % 3])


for i in range(2000):
    step(i)
torch.cuda.synchronize()
out = {}
for K in (20, 200):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    torch.cuda.synchronize()
    torch.cuda._sleep(400_000)
    ev[0].record()
    for i in range(K):
        step(i)
        ev[i + 1].record()
    torch.cuda.synchronize()
    d = [1e3 * ev[i].elapsed_time(ev[i + 1]) for i in range(K)]
    out[f"K{K}_us_per_step"] = 1e3 * ev[0].elapsed_time(ev[K]) / K
    out[f"K{K}_first5_us"] = d[:5]
    out[f"K{K}_median_us"] = sorted(d)[K // 2]
# without per-step events
for K in (20, 200, 2000):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    torch.cuda._sleep(400_000)
    e0.record()
    for i in range(K):
        step(i)
    e1.record()
    torch.cuda.synchronize()
    out[f"plain_K{K}_us"] = 1e3 * e0.elapsed_time(e1) / K
print(json.dumps(out))
