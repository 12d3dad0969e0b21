"""Generate tests/golden/ fixtures.

* reference_kats.json -- the reference test suite's inline known answers
  (closed forms and scalar KATs, with the file:line they come from).  These are
  the reference's own golden values; the reference ships no vector files.
* c1_seed0.npz -- CPU-oracle outputs for the exact c1 configuration (1-D,
  N = 3, K = 64, dt = 0.005): R(U), J.v and both stage residuals on U ~
  U[-1,1) (PCG64 seed 0).  Regression fixture for the oracle and a direct GPU
  parity target.

Run:  python tests/golden/make_golden.py
"""
import json
import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

import oracle as O  # noqa: E402
from paper_2201_05800_b200 import configs as C  # noqa: E402

S5 = math.sqrt(5.0)


def kats():
    return {
        "lgl_n4_nodes": {"value": [-1.0, -1 / S5, 1 / S5, 1.0], "tol": 1e-13,
                         "src": "test_quadrature.cpp:26-34"},
        "lgl_n4_weights": {"value": [1 / 6, 5 / 6, 5 / 6, 1 / 6], "tol": 1e-13,
                           "src": "test_quadrature.cpp:26-34"},
        "lgl_n3_weights": {"value": [1 / 3, 4 / 3, 1 / 3], "tol": 1e-13,
                           "src": "test_quadrature.cpp:19-24"},
        "D2": {"value": [[-0.5, 0.5], [-0.5, 0.5]], "tol": 1e-13,
               "src": "test_operators.cpp:17-18"},
        "D3": {"value": [[-1.5, 2.0, -0.5], [-0.5, 0.0, 0.5], [0.5, -2.0, 1.5]], "tol": 1e-13,
               "src": "test_operators.cpp:24-26"},
        "D4": {"value": [[-3.0, (5 + 5 * S5) / 4, (5 - 5 * S5) / 4, 0.5],
                         [-(1 + S5) / 4, 0.0, S5 / 2, (1 - S5) / 4],
                         [(S5 - 1) / 4, -S5 / 2, 0.0, (1 + S5) / 4],
                         [-0.5, (5 * S5 - 5) / 4, -(5 + 5 * S5) / 4, 3.0]], "tol": 1e-13,
               "src": "test_operators.cpp:32-37"},
        "A4": {"value": [[1 / 12, -S5 / 12, S5 / 12, -1 / 12],
                         [1 / 12, 0.25, (10 - 7 * S5) / 60, S5 / 60],
                         [1 / 12, (10 + 7 * S5) / 60, 0.25, -S5 / 60],
                         [1 / 12, 5 / 12, 5 / 12, 1 / 12]], "tol": 1e-13,
               "src": "acceptance.cpp:110-113"},
        "b4": {"value": [1 / 12, 5 / 12, 5 / 12, 1 / 12], "tol": 1e-15,
               "src": "test_operators.cpp:78-80"},
        "c4": {"value": [0.0, 0.5 - S5 / 10, 0.5 + S5 / 10, 1.0], "tol": 1e-15,
               "src": "test_operators.cpp:81-82"},
        "single_cell_operator": {"value": [[-1.0, 1.0], [1.0, -1.0]], "tol": 1e-14,
                                 "src": "test_spatial.cpp:56-65"},
        "testeq_u_next_dt01": {"value": 3.6199095, "tol": 1e-7,
                               "src": "test_stdg.cpp:114, test_lodg.cpp:49"},
        "testeq_stage2_dt01": {"value": 4.0 / 1.105, "tol": 1e-12, "src": "test_lodg.cpp:44"},
        "st_jacobian_n2_dt0": {"value": [[0.5, 0.5], [-0.5, 0.5]], "tol": 1e-14,
                               "src": "test_stdg.cpp:75-86"},
        "stage_jacobian_aform_n2": {"value": [[1.5, -0.5], [0.5, 1.5]], "tol": 1e-14,
                                    "src": "test_lodg.cpp:101-108"},
    }


def c1_fixture():
    cfg = C.CONFIGS["c1"]
    pr = O.Problem(cfg.dim, cfg.degree, list(cfg.cells), list(cfg.lower), list(cfg.upper),
                   list(cfg.velocity), n_tau=cfg.n_tau)
    U = C.random_slab(cfg)
    un = C.initial_state(cfg)
    v = np.random.default_rng(100).uniform(-1, 1, cfg.n_dof)
    return dict(
        U=U, u_n=un, v=v,
        R=pr.st_residual(0.0, cfg.dt, un, U),
        Jv=pr.st_jvp(0.0, cfg.dt, U, v),
        stage_a=pr.stage_residual(4, O.A_FORM, 0.0, cfg.dt, un, U),
        stage_ainv=pr.stage_residual(4, O.A_INV_FORM, 0.0, cfg.dt, un, U),
    )


def small_fixtures():
    """Oracle outputs for small cases of the other model families (kept small
    so the npz stays a few hundred KB):
      c4p  -- c4 physics (d = 3, N = 3, n_tau = 4, b = (1,1,1)) on 2 x 2 x 2 cells
      c2p  -- c2 physics (d = 2, N = 4, n_tau = 5, b = (1, 0.5)) on 4 x 4 cells
      pulse -- rotating pulse (advdiff, rotating field, eps 1e-3) 4 x 4, p = 2
      euler -- 2-D Euler (gamma 1.4) 4 x 4 on [-10,10]^2, p = 1, vortex data
    For each: the inputs (seeded PCG64) and R(U), J.v (linear models),
    F(u)."""
    out = {}
    rng = np.random.default_rng(20261019)
    for name, cfg in (("c4p", C.CONFIGS["c4"].scaled((2, 2, 2))),
                      ("c2p", C.CONFIGS["c2"].scaled((4, 4)))):
        pr = O.Problem(cfg.dim, cfg.degree, list(cfg.cells), list(cfg.lower), list(cfg.upper),
                       list(cfg.velocity), n_tau=cfg.n_tau)
        U = rng.uniform(-1, 1, cfg.n_dof)
        un = rng.uniform(-1, 1, cfg.n_sdof)
        v = rng.uniform(-1, 1, cfg.n_dof)
        out.update({f"{name}_U": U, f"{name}_un": un, f"{name}_v": v,
                    f"{name}_R": pr.st_residual(0.0, cfg.dt, un, U),
                    f"{name}_Jv": pr.st_jvp(0.0, cfg.dt, U, v)})
    pu = O.Problem(2, 2, [4, 4], [0.0, 0.0], [1.0, 1.0], model=O.ADVDIFF,
                   field=O.FIELD_ROTATING, eps=0.001, n_tau=3)
    X = pu.coords()
    u = C.rotating_pulse_exact(0.0, X[:, 0], X[:, 1]) + 0.05 * rng.uniform(-1, 1, pu.dof)
    U = np.concatenate([u, 0.9 * u, 1.1 * u])
    out.update({"pulse_u": u, "pulse_F": pu.rhs(u), "pulse_U": U,
                "pulse_R": pu.st_residual(0.0, 0.02, u, U)})
    eu = O.Problem(2, 1, [4, 4], [-10.0, -10.0], [10.0, 10.0], model=O.EULER, n_tau=2)
    X = eu.coords()
    u = C.vortex_initial(X[:, 0], X[:, 1]).reshape(-1) * (1 + 0.01 * rng.uniform(-1, 1, eu.dof))
    U = np.concatenate([u, 1.001 * u])
    out.update({"euler_u": u, "euler_F": eu.rhs(u), "euler_U": U,
                "euler_R": eu.st_residual(0.0, 0.05, u, U)})
    return out


if __name__ == "__main__":
    (HERE / "reference_kats.json").write_text(json.dumps(kats(), indent=1))
    np.savez_compressed(HERE / "c1_seed0.npz", **c1_fixture())
    np.savez_compressed(HERE / "small_cases.npz", **small_fixtures())
    print("wrote", HERE / "reference_kats.json", HERE / "c1_seed0.npz",
          HERE / "small_cases.npz")
