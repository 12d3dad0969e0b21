"""Steady-state DRAM traffic per R(U) launch (the bench's rotating c4 loop).

Run under `ncu --cache-control none --metrics dram__bytes_read.sum,
dram__bytes_write.sum,gpu__time_duration.sum -k regex:slab3d`: caches are not
flushed between launches, so each launch's counters include the write-back of
the previous launch's R still dirty in L2 and lose its own tail -- averaged
over consecutive launches that is the true per-launch DRAM traffic (a single
cold launch under-counts the writes).  K launches over 3 rotating sets."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import SlabOperator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg = C.CONFIGS[name]
op = SlabOperator(**cfg.kwargs())
U = [torch.as_tensor(C.random_slab(cfg), device="cuda").clone() for _ in range(3)]
un = [torch.as_tensor(C.initial_state(cfg), device="cuda").clone() for _ in range(3)]
R = [torch.empty(cfg.n_dof, dtype=torch.float64, device="cuda") for _ in range(3)]
for i in range(K):
    op.st_residual(0.0, cfg.dt, un[i % 3], U[i % 3], out=R[i % 3])
torch.cuda.synchronize()
