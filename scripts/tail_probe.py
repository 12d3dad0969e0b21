"""Fast 3-D kernel: DOF/s at 32^3 (4096 segments = 9.22 rounds of 444 CTAs)
against meshes whose segment count is a whole number of rounds."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import SlabOperator  # noqa: E402

for cells in [(32, 32, 32), (24, 37, 36), (24, 37, 40), (32, 37, 24), (16, 37, 48), (40, 40, 40)]:
    cfg = C.CONFIGS["c4"].scaled(cells)
    op = SlabOperator(**cfg.kwargs())
    sets = [(torch.rand(cfg.n_dof, dtype=torch.float64, device="cuda"),
             torch.rand(cfg.n_sdof, dtype=torch.float64, device="cuda"),
             torch.empty(cfg.n_dof, dtype=torch.float64, device="cuda")) for _ in range(3)]
    for i in range(30):
        U, un, R = sets[i % 3]
        op.st_residual(0.0, cfg.dt, un, U, out=R)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 3000
    e0.record()
    for i in range(n):
        U, un, R = sets[i % 3]
        op.st_residual(0.0, cfg.dt, un, U, out=R)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / n
    nseg = cfg.n_dof // 4 // 512
    gbs = 8 * (2 * cfg.n_dof + cfg.n_sdof) / us / 1e3
    print(f"cells {cells} segs {nseg} rounds {nseg/444:.2f}: {us:.2f} us, {cfg.n_dof/us/1e3:.1f} GDOF/s, {gbs:.0f} GB/s")
