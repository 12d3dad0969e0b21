"""Host-side helpers of the product against the oracle, bit for bit (no GPU).

node_coord (mesh.hpp:82-90), interpolate_scalar (mesh.hpp:145-165) and
global_mass (mesh.hpp:125-141) feed every parity test and the bench: u_n of
each config is interpolated on the host.  The GPU and oracle sides of the
parity tests consume the same generated u_n, so a wrong coordinate would pass
them -- these tests pin the generator itself against the oracle's own
restatement of the reference (oracle/stdg_oracle.hpp interpolate / global_mass).
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_2201_05800_b200 import api as A
from paper_2201_05800_b200 import configs as C


def oracle_problem(cfg):
    return O.Problem(cfg.dim, cfg.degree, list(cfg.cells), list(cfg.lower), list(cfg.upper),
                     list(cfg.velocity), model=cfg.model, n_tau=cfg.n_tau)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_config_node_coords_bitwise_equal_oracle(name):
    cfg = C.CONFIGS[name]
    X = C.node_coords(cfg)
    Xo = oracle_problem(cfg).coords()
    assert X.shape == Xo.shape
    assert np.array_equal(X[:, :cfg.dim], Xo[:, :cfg.dim])


@pytest.mark.parametrize("name", ["c1", "c2", "c4"])
def test_config_initial_state_bitwise_equal_oracle_interpolation(name):
    """u_n of the bench / parity inputs = the oracle's interpolate_scalar of u0."""
    cfg = C.CONFIGS[name]
    f = {"sin2pi_x": lambda x, y, z: np.sin(C.TWO_PI * x),
         "sin2pix_sin2piy": lambda x, y, z: np.sin(C.TWO_PI * x) * np.sin(C.TWO_PI * y),
         "sin2pi_xyz": lambda x, y, z: np.sin(C.TWO_PI * (x + y + z))}[cfg.u0]
    assert np.array_equal(C.initial_state(cfg), oracle_problem(cfg).interpolate(f))


def test_c3_initial_state_matches_oracle_coordinates():
    cfg = C.CONFIGS["c3"]
    x = oracle_problem(cfg).coords()[:, 0]
    noise = np.random.default_rng(cfg.seed).standard_normal(cfg.n_sdof)
    assert np.array_equal(C.initial_state(cfg), 1.0 + 0.5 * np.sin(x) + 0.01 * noise)


@pytest.mark.parametrize("d,p,cells,lo,hi", [
    (1, 3, (7,), (0.0,), (1.0,)),
    (2, 4, (5, 3), (0.0, -1.0), (1.0, 2.0)),
    (3, 3, (4, 3, 2), (0.0, 0.0, 0.0), (1.0, 2.0, 0.5)),
    (3, 2, (2, 2, 5), (-1.0, 0.0, 0.25), (1.0, 1.0, 1.0)),
])
def test_api_field_helpers_bitwise_equal_oracle(d, p, cells, lo, hi):
    sp = A.dg_space(A.uniform_mesh(d, lo, hi, cells), p)
    pr = O.Problem(d, p, list(cells), list(lo), list(hi), [0.0] * d, n_tau=2)
    assert np.array_equal(A.node_coords(sp)[:, :d], pr.coords()[:, :d])
    assert np.array_equal(A.global_mass(sp), pr.mass())
    f = lambda X: np.cos(X[:, 0] + 2 * X[:, 1] - X[:, 2])
    got = A.interpolate_scalar(sp, f).coeffs
    assert np.array_equal(got, pr.interpolate(lambda x, y, z: np.cos(x + 2 * y - z)))


def test_api_mass_and_l2_kats():
    """test_mesh.cpp:98-190: mass sums to the measure (times r), hand entry,
    l2 norm of constants, l2_error basics."""
    for p in (1, 2, 3):
        m1 = A.global_mass(A.dg_space(A.uniform_mesh(1, [0.0], [1.0], [8]), p))
        assert (m1 > 0).all() and math.isclose(m1.sum(), 1.0, rel_tol=1e-12)
        m2 = A.global_mass(A.dg_space(A.uniform_mesh(2, [0, 0], [1, 1], [5, 5]), p, 4))
        assert math.isclose(m2.sum(), 4.0, rel_tol=1e-12)
    s = A.dg_space(A.uniform_mesh(2, [0, 0], [1, 1], [2, 2]), 2)
    assert math.isclose(A.global_mass(s)[1 * 3 + 1], 0.0625 * 16.0 / 9.0, rel_tol=1e-14)
    one = A.interpolate_scalar(A.dg_space(A.uniform_mesh(1, [0.0], [1.0], [4]), 2),
                               lambda X: np.ones(len(X)))
    assert math.isclose(A.l2_norm(one), 1.0, rel_tol=1e-13)
    s6 = A.dg_space(A.uniform_mesh(1, [0.0], [1.0], [6]), 2)
    exact = lambda X, t: np.cos(X[:, 0] + t)
    field = A.interpolate(s6, lambda X: exact(X, 0.75), 0.75)
    assert A.l2_error(field, exact, 0.75) <= 1e-14
    flat = A.interpolate_scalar(s6, lambda X: np.ones(len(X)))
    assert math.isclose(A.l2_error(flat, lambda X, t: np.full(len(X), 1.125), 0.0), 0.125,
                        rel_tol=1e-13)
    # r = 4, component innermost (test_mesh.cpp:88-96)
    s4 = A.dg_space(A.uniform_mesh(2, [0, 0], [1, 1], [2, 2]), 1, 4)
    f4 = A.interpolate(s4, lambda X: np.stack([np.ones(len(X)), X[:, 0], X[:, 1],
                                               np.full(len(X), 2.0)], axis=1))
    assert f4.coeffs.size == 64 and f4.coeffs[4 * 1 + 1] == A.node_coords(s4)[1, 0]
