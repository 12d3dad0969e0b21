"""ncu driver: one warm slab solve inside cudaProfilerStart/Stop (run ncu with
--profile-from-start off).  c3 uses its inexact Newton-GMRES config."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import NewtonConfig, SlabOperator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
rk = name == "c5"  # the Lobatto IIIC stage solve (A^-1 form) on the c4 mesh
cfg = C.CONFIGS[name]
op = SlabOperator(**cfg.kwargs())
un = torch.as_tensor(C.initial_state(cfg), device="cuda")
nc = (NewtonConfig(abs_tol=1e-12, rel_tol=1e-10, gmres_tol=1e-6, fd_eps=1e-7) if name == "c3"
      else NewtonConfig(abs_tol=0.0, rel_tol=1e-9, gmres_tol=1e-10))
from paper_2201_05800_b200 import _lib as L  # noqa: E402
step = ((lambda: op.rk_step(L.STG_FORM_A_INV, 0.0, cfg.dt, un, nc)) if rk
        else (lambda: op.stdg_step(0.0, cfg.dt, un, nc)))
step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
t0 = time.perf_counter()
U, u1, info = step()
torch.cuda.synchronize()
t = time.perf_counter() - t0
torch.cuda.profiler.stop()
print(f"solve {t*1e3:.2f} ms, {info.linear_iterations} GMRES its")
