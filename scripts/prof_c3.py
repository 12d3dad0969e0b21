"""ncu driver: one warm c3 (Burgers) slab solve inside cudaProfilerStart/Stop."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import NewtonConfig, SlabOperator  # noqa: E402

cfg = C.CONFIGS["c3"]
op = SlabOperator(**cfg.kwargs())
u = torch.as_tensor(C.initial_state(cfg), device="cuda")
nc = NewtonConfig(abs_tol=1e-12, rel_tol=1e-10, gmres_tol=1e-6, fd_eps=1e-7)
op.stdg_step(0.0, cfg.dt, u, nc)
torch.cuda.synchronize()
torch.cuda.profiler.start()
t0 = time.perf_counter()
U, u1, info = op.stdg_step(0.0, cfg.dt, u, nc)
torch.cuda.synchronize()
t = time.perf_counter() - t0
torch.cuda.profiler.stop()
print(f"solve {t*1e3:.2f} ms, newton {info.newton_iterations}, gmres {info.linear_iterations}")
