"""Device timeline of the host-buffer R(U) call (stg_st_residual_host, pinned
buffers) under torch.profiler: the H2D / kernel / D2H intervals of one warm
call and the call's wall time, next to the box's one-way and duplex pinned
copy times for the same bytes.  Prints one JSON object."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import SlabOperator  # noqa: E402

cfg = C.CONFIGS["c4"]
op = SlabOperator(**cfg.kwargs())
pU = torch.empty(cfg.n_dof, dtype=torch.float64, pin_memory=True)
pun = torch.empty(cfg.n_sdof, dtype=torch.float64, pin_memory=True)
pR = torch.empty(cfg.n_dof, dtype=torch.float64, pin_memory=True)
pU.copy_(torch.as_tensor(C.random_slab(cfg)))
pun.copy_(torch.as_tensor(C.initial_state(cfg)))
a, b, c = pU.numpy(), pun.numpy(), pR.numpy()
for _ in range(3):
    op.st_residual_host(0.0, cfg.dt, b, a, out=c)
torch.cuda.synchronize()
walls = []
for _ in range(10):
    t0 = time.perf_counter()
    op.st_residual_host(0.0, cfg.dt, b, a, out=c)
    walls.append(time.perf_counter() - t0)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        op.st_residual_host(0.0, cfg.dt, b, a, out=c)
    torch.cuda.synchronize()
ev = sorted([(e.time_range.start, e.time_range.end, e.name) for e in prof.events()
             if e.device_type == torch.autograd.DeviceType.CUDA])
# the second call: events after the midpoint gap
gaps = [(ev[i + 1][0] - ev[i][1], i) for i in range(len(ev) - 1)]
cut = max(gaps)[1] + 1
call = ev[cut:]
t0 = call[0][0]
rows = [[round(s - t0, 1), round(e - t0, 1), n.split("(")[0][:40]] for s, e, n in call]
print(json.dumps({"wall_ms_min": min(walls) * 1e3, "device_span_us": call[-1][1] - t0,
                  "events": rows}))
# per-call wall distribution over 50 back-to-back calls (the bench's e2e leg)
ws = []
for _ in range(50):
    t0 = time.perf_counter()
    op.st_residual_host(0.0, cfg.dt, b, a, out=c)
    ws.append((time.perf_counter() - t0) * 1e3)
ws.sort()
print(json.dumps({"calls_ms_sorted": [round(w, 3) for w in ws]}))
