"""Kernel busy time vs wall time of one warm slab solve (torch profiler /
CUPTI timestamps): how much of the solve is GPU idle between launches."""
import json
import re
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import NewtonConfig, SlabOperator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = C.CONFIGS[name]
op = SlabOperator(**cfg.kwargs())
un = torch.as_tensor(C.initial_state(cfg), device="cuda")
tol = dict(c1=(1e-11, 1e-12)).get(name, (1e-9, 1e-10))
nc = NewtonConfig(abs_tol=0.0, rel_tol=tol[0], gmres_tol=tol[1])
op.stdg_step(0.0, cfg.dt, un, nc)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    op.stdg_step(0.0, cfg.dt, un, nc)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = [e for e in ev if "memcpy" not in e.name.lower() and "memset" not in e.name.lower()]
busy = sum(e.device_time_total for e in kern) / 1e3  # us -> ms
span = (max(e.time_range.end for e in kern) - min(e.time_range.start for e in kern)) / 1e3
by = {}
for e in kern:
    k = re.sub(r"^void |\(anonymous namespace\)::|stg::", "", e.name).split("(")[0][:48]
    by[k] = by.get(k, 0.0) + e.device_time_total / 1e3
print(json.dumps({"config": name, "wall_ms": 1e3 * wall, "kernel_busy_ms": busy,
                  "first_to_last_kernel_ms": span, "launches": len(kern),
                  "top": dict(sorted(by.items(), key=lambda x: -x[1])[:12]),
                  "counts": {k: sum(1 for e in kern if re.sub(r"^void |\(anonymous namespace\)::|stg::", "", e.name).split("(")[0][:48] == k)
                             for k in by}}))
if "--seq" in sys.argv:  # per-launch sequence: gap before each kernel, duration
    ks = sorted(kern, key=lambda e: e.time_range.start)
    prev = None
    for e in ks:
        gap = (e.time_range.start - prev) if prev is not None else 0.0
        nm = re.sub(r"^void |\(anonymous namespace\)::|stg::", "", e.name).split("(")[0][:40]
        print(f"  gap {gap:7.1f} us  dur {e.device_time_total:7.1f} us  {nm}")
        prev = e.time_range.end
