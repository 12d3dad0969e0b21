"""Device timeline of one warm solve under torch.profiler (CUPTI activity
records, no kernel replay): per-kernel totals, the device-busy time and the
idle gaps between kernels.  Usage: python scripts/kineto_timeline.py c3|c4|c2 [2: c3's second slab]
Prints one JSON object."""
import collections
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import NewtonConfig, SlabOperator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = C.CONFIGS[name]
op = SlabOperator(**cfg.kwargs())
u = torch.as_tensor(C.initial_state(cfg), device="cuda")
if name == "c3":
    nc = NewtonConfig(abs_tol=1e-12, rel_tol=1e-10, gmres_tol=1e-6, fd_eps=1e-7)
else:
    nc = NewtonConfig(abs_tol=0.0, rel_tol=1e-9, gmres_tol=1e-10)
if name == "c3" and len(sys.argv) > 2:  # a later slab (second slab: 3 Newton steps)
    _, u, _ = op.stdg_step(0.0, cfg.dt, u, nc)
for _ in range(2):
    op.stdg_step(0.0, cfg.dt, u, nc)
torch.cuda.synchronize()
walls = []
for _ in range(5):
    t0 = time.perf_counter()
    op.stdg_step(0.0, cfg.dt, u, nc)
    torch.cuda.synchronize()
    walls.append(time.perf_counter() - t0)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    U, u1, info = op.stdg_step(0.0, cfg.dt, u, nc)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev])
tot = collections.defaultdict(float)
cnt = collections.Counter()
for s, e, n in ks:
    key = n.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][-48:]
    tot[key] += e - s
    cnt[key] += 1
busy = sum(e - s for s, e, _ in ks)
span = ks[-1][1] - ks[0][0] if ks else 0
gaps = sorted(((ks[i + 1][0] - ks[i][1]), ks[i][2][:40], ks[i + 1][2][:40]) for i in range(len(ks) - 1))[::-1][:12]
print(json.dumps({"config": name, "wall_ms": wall * 1e3, "unprofiled_wall_ms": min(walls) * 1e3, "newton": info.newton_iterations,
                  "gmres": info.linear_iterations, "kernels": len(ks), "span_us": span,
                  "busy_us": busy,
                  "by_kernel_us": {k: [round(v, 1), cnt[k]] for k, v in sorted(tot.items(), key=lambda x: -x[1])},
                  "largest_gaps_us": [[round(g, 1), a, b] for g, a, b in gaps]}, indent=1))
