"""Golden fixtures (tests/golden/, made by make_golden.py): the reference's
inline known answers, and c1 oracle outputs.  CPU: the oracle and the
product's host constants reproduce them.  GPU: the CUDA path matches the c1
fixture at 1e-12."""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from paper_2201_05800_b200 import configs as C

G = Path(__file__).resolve().parent / "golden"
KATS = json.loads((G / "reference_kats.json").read_text())


def close(a, k):
    return np.abs(np.asarray(a) - np.asarray(KATS[k]["value"])).max() <= KATS[k]["tol"]


def test_oracle_reproduces_reference_kats():
    x4, w4 = O.lgl(4)
    assert close(x4, "lgl_n4_nodes") and close(w4, "lgl_n4_weights")
    assert close(O.lgl(3)[1], "lgl_n3_weights")
    for n in (2, 3, 4):
        assert close(O.diff_matrix(n), f"D{n}")
    A, b, c = O.lobatto(4)
    assert close(A, "A4") and close(b, "b4") and close(c, "c4")
    A, b, c = O.to_butcher(4)
    assert close(A, "A4")
    pr = O.Problem(1, 1, [1], [0.0], [1.0], [1.0])
    M = np.stack([pr.rhs(e) for e in np.eye(2)], axis=1)
    assert close(M, "single_cell_operator")
    te = O.Problem(1, 1, [1], [0.0], [1.0], [0.0], O.TEST_EQUATION, n_tau=2)
    _, un1, _, _ = te.stdg_step(0.0, 0.1, [4.0])
    assert close(un1[0], "testeq_u_next_dt01")
    U, _, _, _ = te.rk_step(2, O.A_FORM, 0.0, 0.1, [4.0])
    assert close(U[1], "testeq_stage2_dt01")
    J = np.stack([te.st_jvp(0.0, 0.0, np.full(2, 4.0), e) for e in np.eye(2)], axis=1)
    assert close(J, "st_jacobian_n2_dt0")
    J = np.stack([te.stage_jvp(2, O.A_FORM, 0.0, 1.0, np.full(2, 4.0), e) for e in np.eye(2)],
                 axis=1)
    assert close(J, "stage_jacobian_aform_n2")


def test_product_constants_reproduce_reference_kats():
    from paper_2201_05800_b200 import _lib as L
    lib = L.load()
    for n in (2, 3, 4):
        D = np.zeros((n, n))
        assert lib.stg_diff_matrix(n, D.ctypes.data) == 0
        assert close(D, f"D{n}")
    A, b, c = np.zeros((4, 4)), np.zeros(4), np.zeros(4)
    assert lib.stg_lobatto_tableau(4, A.ctypes.data, b.ctypes.data, c.ctypes.data) == 0
    assert close(A, "A4") and close(b, "b4") and close(c, "c4")


def test_oracle_reproduces_c1_fixture():
    f = np.load(G / "c1_seed0.npz")
    cfg = C.CONFIGS["c1"]
    assert np.array_equal(f["U"], C.random_slab(cfg))          # generator pinned
    assert np.array_equal(f["u_n"], C.initial_state(cfg))
    pr = O.Problem(1, 3, [64], [0.0], [1.0], [1.0], n_tau=4)
    R = pr.st_residual(0.0, cfg.dt, f["u_n"], f["U"])
    assert np.abs(R - f["R"]).max() <= 1e-14 * np.abs(f["R"]).max()
    Jv = pr.st_jvp(0.0, cfg.dt, f["U"], f["v"])
    assert np.abs(Jv - f["Jv"]).max() <= 1e-14 * np.abs(f["Jv"]).max()


@pytest.mark.gpu
def test_cuda_matches_c1_fixture():
    import torch
    from paper_2201_05800_b200.api import SlabOperator
    f = np.load(G / "c1_seed0.npz")
    cfg = C.CONFIGS["c1"]
    op = SlabOperator(**cfg.kwargs())
    d = lambda a: torch.as_tensor(a, device="cuda")
    rel = lambda a, b: np.abs(a.cpu().numpy() - b).max() / np.abs(b).max()
    assert rel(op.st_residual(0.0, cfg.dt, d(f["u_n"]), d(f["U"])), f["R"]) <= 1e-12
    assert rel(op.st_jvp(0.0, cfg.dt, d(f["U"]), d(f["v"])), f["Jv"]) <= 1e-12
    assert rel(op.stage_residual(0, 0.0, cfg.dt, d(f["u_n"]), d(f["U"])), f["stage_a"]) <= 1e-12
    assert rel(op.stage_residual(1, 0.0, cfg.dt, d(f["u_n"]), d(f["U"])), f["stage_ainv"]) <= 1e-12


SMALL = G / "small_cases.npz"


def _small_problems():
    c4p, c2p = C.CONFIGS["c4"].scaled((2, 2, 2)), C.CONFIGS["c2"].scaled((4, 4))
    return c4p, c2p


def test_oracle_reproduces_small_fixtures():
    """Regression pin of the oracle on the small 3-D / 2-D / pulse / Euler cases."""
    f = np.load(SMALL)
    c4p, c2p = _small_problems()
    for name, cfg in (("c4p", c4p), ("c2p", c2p)):
        pr = O.Problem(cfg.dim, cfg.degree, list(cfg.cells), list(cfg.lower), list(cfg.upper),
                       list(cfg.velocity), n_tau=cfg.n_tau)
        R = pr.st_residual(0.0, cfg.dt, f[f"{name}_un"], f[f"{name}_U"])
        assert np.abs(R - f[f"{name}_R"]).max() <= 1e-14 * np.abs(f[f"{name}_R"]).max()
    pu = O.Problem(2, 2, [4, 4], [0.0, 0.0], [1.0, 1.0], model=O.ADVDIFF,
                   field=O.FIELD_ROTATING, eps=0.001, n_tau=3)
    assert np.abs(pu.rhs(f["pulse_u"]) - f["pulse_F"]).max() <= 1e-13 * np.abs(f["pulse_F"]).max()
    eu = O.Problem(2, 1, [4, 4], [-10.0, -10.0], [10.0, 10.0], model=O.EULER, n_tau=2)
    assert np.abs(eu.rhs(f["euler_u"]) - f["euler_F"]).max() <= 1e-13 * np.abs(f["euler_F"]).max()


@pytest.mark.gpu
def test_cuda_matches_small_fixtures():
    import torch
    from paper_2201_05800_b200 import _lib as L
    from paper_2201_05800_b200.api import SlabOperator
    f = np.load(SMALL)
    d = lambda a: torch.as_tensor(a, device="cuda")
    rel = lambda a, b: np.abs(a.cpu().numpy() - b).max() / np.abs(b).max()
    c4p, c2p = _small_problems()
    for name, cfg in (("c4p", c4p), ("c2p", c2p)):
        op = SlabOperator(**cfg.kwargs())
        assert rel(op.st_residual(0.0, cfg.dt, d(f[f"{name}_un"]), d(f[f"{name}_U"])),
                   f[f"{name}_R"]) <= 1e-12
        assert rel(op.st_jvp(0.0, cfg.dt, None, d(f[f"{name}_v"])), f[f"{name}_Jv"]) <= 1e-12
    pu = SlabOperator(2, 2, 3, (4, 4), (0.0, 0.0), (1.0, 1.0), model=L.STG_MODEL_ADVDIFF,
                      velocity_field=L.STG_FIELD_ROTATING, eps=0.001)
    assert rel(pu.spatial_rhs(d(f["pulse_u"])), f["pulse_F"]) <= 1e-12
    assert rel(pu.st_residual(0.0, 0.02, d(f["pulse_u"]), d(f["pulse_U"])), f["pulse_R"]) <= 1e-12
    eu = SlabOperator(2, 1, 2, (4, 4), (-10.0, -10.0), (10.0, 10.0), model=L.STG_MODEL_EULER)
    assert rel(eu.spatial_rhs(d(f["euler_u"])), f["euler_F"]) <= 1e-12
    assert rel(eu.st_residual(0.0, 0.05, d(f["euler_u"]), d(f["euler_U"])), f["euler_R"]) <= 1e-12
