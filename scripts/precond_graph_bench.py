"""Device time per kernel of repeated preconditioner applies (torch.profiler
CUPTI records; run with STG_NO_PDL=1 so kernel spans do not overlap).
Burgers configs linearise at a fixed state; every call rebuilds the blocks
(stg_st_precond_apply), listed separately.
Usage: python scripts/precond_graph_bench.py c3 [precond] [reps]"""
import collections
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200 import _lib as L  # noqa: E402
from paper_2201_05800_b200.api import SlabOperator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
pc = int(sys.argv[2]) if len(sys.argv) > 2 else L.STG_PRECOND_AUTO
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
cfg = C.CONFIGS[name]
op = SlabOperator(**cfg.kwargs())
U = torch.as_tensor(np.tile(C.initial_state(cfg), cfg.n_tau), device="cuda")
X = [torch.as_tensor(C.random_slab(cfg, k), device="cuda") for k in range(3)]
Y = [torch.empty_like(x) for x in X]
for k in range(3):
    op.st_precond_apply(cfg.dt, X[k], U, precond=pc, out=Y[k])
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for k in range(reps):
        op.st_precond_apply(cfg.dt, X[k % 3], U, precond=pc, out=Y[k % 3])
    torch.cuda.synchronize()
tot = collections.defaultdict(float)
cnt = collections.Counter()
for e in prof.events():
    if e.device_type != torch.autograd.DeviceType.CUDA:
        continue
    key = e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][-48:]
    tot[key] += e.time_range.end - e.time_range.start
    cnt[key] += 1
print(json.dumps({"config": name, "precond": pc,
                  "us_per_launch": {k: round(v / cnt[k], 2) for k, v in tot.items()}}))
