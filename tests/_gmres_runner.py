"""Subprocess helper for tests/test_gpu_gmres.py: runs a fixed set of device
solves and writes the solutions and iteration counts to an .npz file, so the
test can compare runs under different STG_* environment knobs (read once per
process by the library)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2201_05800_b200 import _lib as L  # noqa: E402
from paper_2201_05800_b200 import configs as C  # noqa: E402
from paper_2201_05800_b200.api import NewtonConfig, SlabOperator  # noqa: E402


def main(out: str) -> None:
    res = {}
    # c4 physics on 8^3 cells: FDM (AUTO), temporal blocks, restarted cycles
    cfg = C.CONFIGS["c4"].scaled((8, 8, 8))
    op = SlabOperator(**cfg.kwargs())
    un = torch.as_tensor(C.initial_state(cfg), device="cuda")
    for name, pc, m in [("fdm30", L.STG_PRECOND_AUTO, 30), ("fdm3", L.STG_PRECOND_AUTO, 3),
                        ("tblock4", L.STG_PRECOND_TBLOCK, 4), ("none30", L.STG_PRECOND_NONE, 30)]:
        nc = NewtonConfig(abs_tol=0.0, rel_tol=1e-11, gmres_tol=1e-12, precond=pc,
                          gmres_restart=m, gmres_max_it=4000)
        U, _, info = op.stdg_step(0.0, cfg.dt, un, nc)
        res[name] = U.cpu().numpy()
        res[name + "_its"] = np.array([info.newton_iterations, info.linear_iterations])
    # c2 physics on 32 x 8 cells: the d = 2 element block (FDM; dense with STG_NO_FDM2=1)
    c2 = C.CONFIGS["c2"].scaled((32, 8))
    op2 = SlabOperator(**c2.kwargs())
    u2 = torch.as_tensor(C.initial_state(c2), device="cuda")
    U2, _, info2 = op2.stdg_step(0.0, c2.dt, u2, NewtonConfig(abs_tol=0.0, rel_tol=1e-11,
                                                             gmres_tol=1e-12))
    res["c2"] = U2.cpu().numpy()
    res["c2_its"] = np.array([info2.newton_iterations, info2.linear_iterations])
    U2s, _, _ = op2.rk_step(L.STG_FORM_A_INV, 0.0, c2.dt, u2,
                            NewtonConfig(abs_tol=0.0, rel_tol=1e-11, gmres_tol=1e-12))
    res["c2rk"] = U2s.cpu().numpy()
    res["c2rk_its"] = np.array([0, 0])
    # plain linear solve through the ABI entry (non-zero initial guess)
    rng = np.random.default_rng(5)
    b = torch.as_tensor(rng.uniform(-1, 1, cfg.n_dof), device="cuda")
    x0 = torch.as_tensor(rng.uniform(-1e-3, 1e-3, cfg.n_dof), device="cuda")
    x, it, rr = op.gmres_st(0.0, cfg.dt, None, b, x=x0.clone(), restart=5, tol=1e-11)
    res["gmres_st"] = x.cpu().numpy()
    res["gmres_st_its"] = np.array([it])
    # c3 physics (Burgers, FD J.v, fp32 element blocks): 256 cells take the
    # host-steered FD action (no speculation), 4096 cells the fused lane-kernel
    # FD action (speculative steps)
    for key, cells in [("c3", 256), ("c3f", 4096)]:
        c3 = C.CONFIGS["c3"].scaled((cells,))
        op3 = SlabOperator(**c3.kwargs())
        u3 = torch.as_tensor(C.initial_state(c3), device="cuda")
        U3, _, info3 = op3.stdg_step(0.0, c3.dt, u3, NewtonConfig(abs_tol=1e-12, rel_tol=1e-10,
                                                                 gmres_tol=1e-8, fd_eps=1e-7))
        res[key] = U3.cpu().numpy()
        res[key + "_its"] = np.array([info3.newton_iterations, info3.linear_iterations])
    torch.cuda.synchronize()
    np.savez(out, **res)


if __name__ == "__main__":
    main(sys.argv[1])
