import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2201_05800_b200 import configs as C
from paper_2201_05800_b200.api import SlabOperator
cfg = C.CONFIGS["c4"]
op = SlabOperator(**cfg.kwargs())
pU = torch.empty(cfg.n_dof, dtype=torch.float64, pin_memory=True)
pun = torch.empty(cfg.n_sdof, dtype=torch.float64, pin_memory=True)
pR = torch.empty(cfg.n_dof, dtype=torch.float64, pin_memory=True)
pU.copy_(torch.as_tensor(C.random_slab(cfg))); pun.copy_(torch.as_tensor(C.initial_state(cfg)))
a, b, c = pun.numpy(), pU.numpy(), pR.numpy()
for rep in range(6):
    for _ in range(40):
        t0 = time.perf_counter()
        op.st_residual_host(0.0, cfg.dt, a, b, out=c)
        print(f"wall {1e3*(time.perf_counter()-t0):.3f}", file=sys.stderr)
    time.sleep(0.2)
