"""Small driver for ncu: a few c4 applies of each operator family."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import SlabOperator  # noqa: E402
from paper_2201_05800_b200 import _lib as L  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = C.CONFIGS[name]
op = SlabOperator(**cfg.kwargs())
U = torch.as_tensor(C.random_slab(cfg), device="cuda")
un = torch.as_tensor(C.initial_state(cfg), device="cuda")
R = torch.empty_like(U)
for _ in range(reps):
    op.st_residual(0.0, cfg.dt, un, U, out=R)
for _ in range(reps):
    op.st_jvp(0.0, cfg.dt, None, U, out=R)
if name == "c4":
    gen = SlabOperator(**cfg.kwargs(), kernel=L.STG_KERNEL_GENERIC)
    for _ in range(reps):
        gen.st_residual(0.0, cfg.dt, un, U, out=R)
torch.cuda.synchronize()
print("ok")
