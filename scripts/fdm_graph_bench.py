"""Device time of the c4 element-block preconditioner apply (FDM): 30 applies
over 3 rotating buffer pairs captured in a CUDA graph, replayed; no host
launch overhead in the measurement.  Prints one JSON object."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200 import _lib as L  # noqa: E402
from paper_2201_05800_b200.api import SlabOperator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
pc = int(sys.argv[2]) if len(sys.argv) > 2 else L.STG_PRECOND_EBLOCK
cfg = C.CONFIGS[name]
if len(sys.argv) > 3:  # another mesh with the config's physics, e.g. 32x24x37
    cfg = cfg.scaled(tuple(int(c) for c in sys.argv[3].split("x")))
op = SlabOperator(**cfg.kwargs())
X = [torch.as_tensor(C.random_slab(cfg, k), device="cuda") for k in range(3)]
Y = [torch.empty_like(x) for x in X]
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
reps = 30
with torch.cuda.stream(side):
    for k in range(3):  # builds and uploads the factors (host syncs) before capture
        op.st_precond_apply(cfg.dt, X[k], precond=pc, out=Y[k])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for k in range(reps):
            op.st_precond_apply(cfg.dt, X[k % 3], precond=pc, out=Y[k % 3])
torch.cuda.current_stream().wait_stream(side)
g.replay()
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda._sleep(400_000)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / reps)
print(json.dumps({"config": cfg.name, "precond": pc, "us_per_apply": 1e3 * best,
                  "ns_per_cell": 1e6 * best / cfg.n_cells,
                  "gbs": 16 * cfg.n_dof / (best * 1e-3) / 1e9}))
