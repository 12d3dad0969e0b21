"""c2 R(U) / J.v timing (CUDA events, 3 rotating buffer sets).  Prints JSON."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import SlabOperator  # noqa: E402

cfg = C.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
op = SlabOperator(**cfg.kwargs())
Us = [torch.as_tensor(C.random_slab(cfg, s), device="cuda") for s in range(3)]
un = [torch.as_tensor(C.initial_state(cfg), device="cuda") for _ in range(3)]
Rs = [torch.empty_like(U) for U in Us]
out = {}
for name, fn in (("residual", lambda k: op.st_residual(0.0, cfg.dt, un[k], Us[k], out=Rs[k])),
                 ("jvp", lambda k: op.st_jvp(0.0, cfg.dt, None, Us[k], out=Rs[k]))):
    for k in range(6):
        fn(k % 3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    reps = 300
    e0.record()
    for k in range(reps):
        fn(k % 3)
    e1.record()
    torch.cuda.synchronize()
    us = 1e3 * e0.elapsed_time(e1) / reps
    by = C.residual_bytes(cfg) if name == "residual" else C.jvp_bytes(cfg)
    out[name] = {"us": us, "gbs": by / us / 1e3, "frac": by / us / 1e3 / 6545.6}
print(json.dumps(out))
