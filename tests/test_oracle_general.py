"""Oracle pins for the general flux models: the rotating
pulse (advdiff_model with rotating_field and interior-penalty diffusion) and
the 2-D Euler equations, checked against the reference's own known-answer
tests (test_spatial.cpp, acceptance.cpp criteria 5, 6, 9).  CPU only."""
import math

import numpy as np
import pytest

import oracle as O
from paper_2201_05800_b200 import configs as C


def pulse(cells, p, eps=0.001, n_tau=None):
    return O.Problem(2, p, [cells, cells], [0.0, 0.0], [1.0, 1.0], model=O.ADVDIFF,
                     field=O.FIELD_ROTATING, eps=eps, n_tau=n_tau or p + 1)


def euler(cells, p, n_tau=2):
    return O.Problem(2, p, [cells, cells], [-10.0, -10.0], [10.0, 10.0], model=O.EULER,
                     n_tau=n_tau)


def pulse_u(pr, t=0.0):
    X = pr.coords()
    return C.rotating_pulse_exact(t, X[:, 0], X[:, 1])


def vortex_u(pr):
    X = pr.coords()
    return C.vortex_initial(X[:, 0], X[:, 1]).reshape(-1)


def l2(pr, u):  # l2_norm, mesh.hpp:168-172
    return math.sqrt(float(np.dot(u * u, pr.mass())))


def test_free_stream():  # test_spatial.cpp:67-89
    pr = pulse(5, 3)
    assert pr.eta == 90.0  # 10 p^2 (spatial.hpp:366)
    assert np.abs(pr.rhs(np.full(pr.dof, -0.6))).max() <= 1e-12
    eu = euler(4, 1)
    c3 = np.tile([1.0, 0.3, -0.2, 2.5], eu.dof // 4)
    assert np.abs(eu.rhs(c3)).max() <= 1e-12


def test_conservation():  # test_spatial.cpp:91-118
    for pr, u in ((pulse(6, 2), None), (euler(4, 2), "vortex")):
        u = vortex_u(pr) if u else pulse_u(pr)
        mr = pr.mass() * pr.rhs(u)
        for comp in range(pr.r):
            assert abs(mr[comp::pr.r].sum()) <= 1e-11


def test_interior_penalty_dissipates_energy():  # test_spatial.cpp:254-266
    pr = O.Problem(1, 2, [4], [0.0], [1.0], velocity=(0.0,), model=O.ADVDIFF, eps=0.01)
    rng = np.random.default_rng(7)
    m = pr.mass()
    for _ in range(5):
        u = rng.uniform(-1.0, 1.0, pr.dof)
        assert float(np.dot(u, m * pr.rhs(u))) <= 1e-12


def test_linear_jacobian_exact():  # test_spatial.cpp:281-291
    pr = pulse(4, 2)
    u = pulse_u(pr)
    ref = pr.rhs(u)
    lin = pr.spatial_jvp(u, u)
    assert np.abs(lin - ref).max() < 1e-12 * (1 + np.abs(ref).max())


def test_pulse_rhs_consistency():  # test_spatial.cpp:169-191
    def err_at(cells):
        pr = pulse(cells, 3)
        X = pr.coords()
        dt = 1e-6
        dudt = (C.rotating_pulse_exact(dt, X[:, 0], X[:, 1])
                - C.rotating_pulse_exact(-dt, X[:, 0], X[:, 1])) / (2 * dt)
        return l2(pr, pr.rhs(pulse_u(pr)) - dudt)
    e32, e64 = err_at(32), err_at(64)
    assert e32 / e64 > 6.0
    assert e64 < 2e-3


def test_euler_jvp_against_directional_fd():  # test_spatial.cpp:308-326
    pr = euler(4, 1)
    u0 = vortex_u(pr)
    v = np.random.default_rng(42).uniform(-1.0, 1.0, pr.dof)
    h = 1e-6
    fd = (pr.rhs(u0 + h * v) - pr.rhs(u0 - h * v)) / (2 * h)
    Jv = pr.spatial_jvp(u0, v)
    assert np.abs(fd - Jv).max() <= 1e-5 * np.abs(Jv).max()


def test_rejects_inconsistent_inputs():  # test_spatial.cpp:328-337, models.hpp:69, 121
    with pytest.raises(O.OracleError):
        O.Problem(1, 1, [4], [0.0], [1.0], model=O.EULER)
    with pytest.raises(O.OracleError):
        O.Problem(2, 1, [4, 4], [0.0] * 2, [1.0] * 2, model=O.ADVDIFF, eps=-1e-3)
    with pytest.raises(O.OracleError):
        O.Problem(2, 1, [4, 4], [0.0] * 2, [1.0] * 2, model=O.EULER, gamma=1.0)


def test_euler_admissibility_error():  # models.hpp:108-113, test_models.cpp:98-103
    pr = euler(2, 1)
    bad = np.tile([1.0, 4.0, 0.0, 1.0], pr.dof // 4)  # kinetic 8 > e -> P < 0
    with pytest.raises(O.OracleError) as e:
        pr.rhs(bad)
    assert "code 5" in str(e.value) and "nonphysical" in str(e.value)


def test_criterion5_pulse_step_equivalence():  # acceptance.cpp:221-261 (pulse rows)
    for n_tau in (2, 3):
        pr = pulse(8, n_tau - 1, n_tau=n_tau)
        u = pulse_u(pr)
        t, dt = 0.0, 0.125
        for _ in range(4):
            kw = dict(abs_tol=1e-13, rel_tol=1e-13, linear=O.GMRES, gmres_tol=1e-14,
                      gmres_max_it=5000)
            _, lo, _, _ = pr.rk_step(n_tau, 0, t, dt, u, **kw)
            _, st, _, _ = pr.stdg_step(t, dt, u, **kw)
            rel = np.abs(lo - st).max() / (1.0 + np.abs(st).max())
            assert rel <= 1e-9
            u, t = st, t + dt


# acceptance.cpp:265-269: (n_tau, N, lodg_ref, stdg_ref), tolerance 25 %
PULSE_TABLE = [(2, 8, 4.66e-2, 4.46e-2), (2, 16, 3.49e-2, 3.39e-2),
               (3, 8, 2.42e-2, 2.41e-2), (3, 16, 5.36e-3, 5.38e-3)]


@pytest.mark.parametrize("n_tau,N,lodg_ref,stdg_ref", PULSE_TABLE)
def test_criterion6_pulse_error_table(n_tau, N, lodg_ref, stdg_ref):  # experiments.hpp:133-175
    pr = pulse(N, n_tau - 1, n_tau=n_tau)
    kw = dict(linear=O.GMRES, gmres_tol=1e-12, gmres_max_it=5000)
    for method, ref in (("lodg", lodg_ref), ("stdg", stdg_ref)):
        u, dt = pulse_u(pr), 1.0 / N
        for k in range(N):
            if method == "lodg":
                _, u, _, _ = pr.rk_step(n_tau, 0, k * dt, dt, u, **kw)
            else:
                _, u, _, _ = pr.stdg_step(k * dt, dt, u, **kw)
        err = l2(pr, u - pulse_u(pr, 1.0))
        assert abs(err / ref - 1.0) <= 0.25, (method, err, ref)


def euler_vortex(n_steps, dt, n_tau=2, cells=16, p=1):
    """run_euler_vortex (experiments.hpp:188-262), lodg A-form."""
    pr = euler(cells, p, n_tau=n_tau)
    u = vortex_u(pr)
    min_rho = u[0::4].min()
    max_newton = 0
    t = 0.0
    for _ in range(n_steps):
        _, u, nit, _ = pr.rk_step(n_tau, 0, t, dt, u, linear=O.GMRES, gmres_tol=1e-8,
                                  gmres_max_it=5000)
        t += dt
        max_newton = max(max_newton, nit)
        min_rho = min(min_rho, u[0::4].min())
    X = pr.coords()
    xb = X[:, 0] - t
    xb -= 20.0 * np.floor((xb + 10.0) / 20.0)
    rho_exact = C.vortex_initial(xb, X[:, 1])[:, 0]
    m = pr.mass()[0::4]
    err = math.sqrt(float(np.dot(m, (u[0::4] - rho_exact) ** 2)))
    return err, min_rho, max_newton


def test_criterion9_euler_vortex_smoke():  # acceptance.cpp:451-466
    e_full, rho_full, nit_full = euler_vortex(10, 0.05)
    assert rho_full > 0.0
    assert nit_full <= 10
    e_half, rho_half, _ = euler_vortex(20, 0.025)
    assert rho_half > 0.0
    assert e_half / e_full <= 1.005
