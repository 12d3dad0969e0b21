"""Device time per apply (CUDA graph of 30 applies over 3 rotating buffer
sets, > L2): R(U), J.v, both stage residuals of a config.  One JSON object.
  python scripts/apply_graph_bench.py c2"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import SlabOperator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = C.CONFIGS[name]
op = SlabOperator(**cfg.kwargs())
S = [(torch.as_tensor(C.random_slab(cfg, 10 + k), device="cuda"),
      torch.as_tensor(C.initial_state(cfg), device="cuda").clone(),
      torch.empty(cfg.n_dof, dtype=torch.float64, device="cuda")) for k in range(3)]
hbm = 6548.5
ops = {
    "residual": (lambda k: op.st_residual(0.0, cfg.dt, S[k][1], S[k][0], out=S[k][2]),
                 C.residual_bytes(cfg)),
    "jvp": (lambda k: op.st_jvp(0.0, cfg.dt, None, S[k][0], out=S[k][2]), C.jvp_bytes(cfg)),
    "stage_a_inv": (lambda k: op.stage_residual(1, 0.0, cfg.dt, S[k][1], S[k][0], out=S[k][2]),
                    C.residual_bytes(cfg)),
    "stage_a": (lambda k: op.stage_residual(0, 0.0, cfg.dt, S[k][1], S[k][0], out=S[k][2]),
                C.residual_bytes(cfg)),
}
out = {"config": name}
side = torch.cuda.Stream()
for key, (fn, nbytes) in ops.items():
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for k in range(3):
            fn(k)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for i in range(30):
                fn(i % 3)
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
        best = min(best, e0.elapsed_time(e1) / 30)
    out[key] = {"us": 1e3 * best, "hbm_frac": nbytes / (best * 1e-3) / 1e9 / hbm}
print(json.dumps(out))
