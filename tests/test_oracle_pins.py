"""Pin the CPU oracle against the reference's own known-answer tests.

Every assertion below restates an inline known answer from the reference test
suite (file:line cited per test) -- the reference has no golden-vector files
(SURVEY.md §4), so these KATs *are* the golden vectors.  The same values are
also committed as tests/golden/reference_kats.json (see test_golden.py).
CPU only.
"""
import math

import numpy as np
import pytest

import oracle as O

S5 = math.sqrt(5.0)


# ---- quadrature (test_quadrature.cpp) ---------------------------------------
def test_lgl_closed_forms():  # test_quadrature.cpp:9-35
    x, w = O.lgl(2)
    assert x[0] == -1.0 and x[1] == 1.0
    assert abs(w[0] - 1) < 1e-13 and abs(w[1] - 1) < 1e-13
    x, w = O.lgl(3)
    assert x[1] == 0.0
    assert np.allclose(w, [1 / 3, 4 / 3, 1 / 3], rtol=1e-13, atol=0)
    x, w = O.lgl(4)
    assert abs(x[1] + 1 / S5) < 1e-13 and abs(x[2] - 1 / S5) < 1e-13
    assert np.allclose(w, [1 / 6, 5 / 6, 5 / 6, 1 / 6], rtol=1e-13, atol=0)


def test_lgl_order_symmetry_sum():  # test_quadrature.cpp:37-51
    for n in range(2, 10):
        x, w = O.lgl(n)
        assert x[0] == -1.0 and x[-1] == 1.0
        assert np.all(np.diff(x) > 0)
        assert np.all(x == -x[::-1])
        assert np.all(w > 0)
        assert abs(w.sum() - 2.0) < 1e-14


def test_lgl_exactness():  # test_quadrature.cpp:53-64
    for n in range(2, 10):
        x, w = O.lgl(n)
        for k in range(0, 2 * n - 2):
            q = float(np.sum(w * x ** k))
            exact = 2.0 / (k + 1) if k % 2 == 0 else 0.0
            assert abs(q - exact) < 1e-13


def test_lgl_rejects_small_n():  # test_quadrature.cpp:66-69
    for n in (0, 1):
        with pytest.raises(O.OracleError):
            O.lgl(n)


def test_diff_matrix_closed_forms():  # test_quadrature.cpp:71-84
    assert np.abs(O.diff_matrix(2) - np.array([[-0.5, 0.5], [-0.5, 0.5]])).max() < 1e-13
    D3 = np.array([[-1.5, 2.0, -0.5], [-0.5, 0.0, 0.5], [0.5, -2.0, 1.5]])
    assert np.abs(O.diff_matrix(3) - D3).max() < 1e-13


def test_diff_matrix_monomials():  # test_quadrature.cpp:86-98
    for n in range(2, 10):
        x, _ = O.lgl(n)
        D = O.diff_matrix(n)
        assert np.abs(D @ np.ones(n)).max() < 1e-13
        for k in range(1, n):
            assert np.abs(D @ x ** k - k * x ** (k - 1)).max() < 1e-12


def test_eval_interpolant():  # test_quadrature.cpp:100-147
    x5, _ = O.lgl(5)
    for i in range(5):
        e = np.zeros(5)
        e[i] = 1
        for j in range(5):
            assert abs(O.eval_interpolant(5, e, x5[j]) - (1.0 if i == j else 0.0)) < 1e-13
    for tau in (-1.0, -0.731, -0.25, 0.0, 0.111, 0.5, 0.999, 1.0):
        assert abs(O.eval_interpolant(5, np.ones(5), tau) - 1) < 1e-12
    x4, _ = O.lgl(4)
    p = lambda t: 2 * t ** 3 - t + 0.25
    for tau in (-0.9, -0.3, 0.2, 0.7):
        assert abs(O.eval_interpolant(4, p(x4), tau) - p(tau)) < 1e-13
    x3, _ = O.lgl(3)
    assert abs(O.eval_interpolant(3, x3, 0.5) - 0.5) < 1e-13
    assert abs(O.eval_interpolant(2, [0.0, 1.0], 0.0) - 0.5) < 1e-13
    with pytest.raises(O.OracleError):
        O.eval_interpolant(3, np.ones(3), 1.5)


# ---- temporal operators (test_operators.cpp, acceptance.cpp:64-97) ---------
D4_REF = np.array([
    [-3.0, (5 + 5 * S5) / 4, (5 - 5 * S5) / 4, 0.5],
    [-(1 + S5) / 4, 0.0, S5 / 2, (1 - S5) / 4],
    [(S5 - 1) / 4, -S5 / 2, 0.0, (1 + S5) / 4],
    [-0.5, (5 * S5 - 5) / 4, -(5 + 5 * S5) / 4, 3.0],
])


def test_sbp_closed_forms():  # test_operators.cpp:9-38
    assert np.abs(O.diff_matrix(4) - D4_REF).max() < 1e-13
    _, w = O.lgl(4)
    assert np.abs(w - np.array([1 / 6, 5 / 6, 5 / 6, 1 / 6])).max() < 1e-13
    # The paper's printed D4 has a sign typo in row 2, col 3;
    # the D 1 = 0 row-sum identity rules it out.
    assert np.abs(D4_REF.sum(axis=1)).max() < 1e-14


def test_sbp_defect():  # test_operators.cpp:40-50
    assert O.sbp_defect(2) <= 1e-15
    assert O.sbp_defect(3) <= 1e-15
    for n in range(2, 9):
        assert O.sbp_defect(n) <= 1e-13


def test_to_butcher_matches_lobatto():  # test_operators.cpp:52-60
    for n in (2, 3, 4):
        A, b, c = O.to_butcher(n)
        Ar, br, cr = O.lobatto(n)
        assert np.abs(A - Ar).max() < 1e-13
        assert np.abs(b - br).max() < 1e-13
        assert np.abs(c - cr).max() < 1e-13


def test_lobatto_closed_forms():  # test_operators.cpp:62-86
    A2, _, _ = O.lobatto(2)
    assert np.abs(A2 - np.array([[0.5, -0.5], [0.5, 0.5]])).max() == 0.0
    A3, _, c3 = O.lobatto(3)
    assert np.abs(A3[1] - [1 / 6, 5 / 12, -1 / 12]).max() < 1e-15
    assert c3[1] == 0.5
    A4, b4, c4 = O.lobatto(4)
    assert np.abs(A4[0] - [1 / 12, -S5 / 12, S5 / 12, -1 / 12]).max() < 1e-15
    assert np.abs(b4 - [1 / 12, 5 / 12, 5 / 12, 1 / 12]).max() < 1e-15
    assert abs(c4[1] - (0.5 - S5 / 10)) < 1e-15 and abs(c4[2] - (0.5 + S5 / 10)) < 1e-15
    for s in (1, 5):
        with pytest.raises(O.OracleError):
            O.lobatto(s)


def test_tableau_invariants():  # test_operators.cpp:88-96
    for s in (2, 3, 4):
        A, b, c = O.lobatto(s)
        assert abs(b.sum() - 1) < 1e-14
        assert np.abs(A @ np.ones(s) - c).max() < 1e-13
        assert c[0] == 0.0 and c[-1] == 1.0


# ---- spatial operator (test_spatial.cpp) ------------------------------------
def adv1d(cells, p, b=1.0, n_tau=None, lo=0.0, hi=1.0):
    return O.Problem(1, p, [cells], [lo], [hi], [b], O.ADVECTION, n_tau=n_tau)


def test_spatial_single_cell_kat():  # test_spatial.cpp:56-65
    pr = adv1d(1, 1)
    Aref = np.array([[-1.0, 1.0], [1.0, -1.0]])
    for u in (np.array([1.0, 0.0]), np.array([0.3, -0.7])):
        assert np.abs(pr.rhs(u) - Aref @ u).max() < 1e-14


def test_llf_consistency_upwinding():  # test_spatial.cpp:40-42
    # llf(2,2) = 2 and llf(2,0) = 2 for b = 1: the face flux between cells 0
    # and 1 only sees the upwind trace, so rhs at cell 0's right node is
    # unchanged (exactly) when the downwind trace u[2] changes from 2 to 0.
    pr = adv1d(2, 1)
    f = pr.rhs(np.array([2.0, 2.0, 2.0, 2.0]))
    g = pr.rhs(np.array([2.0, 2.0, 0.0, 2.0]))
    assert f[1] == g[1]
    assert f[0] == 0.0 and f[1] == 0.0


def test_free_stream():  # test_spatial.cpp:67-89 (advection part), acceptance 334-343
    pr = adv1d(6, 2, b=1.5)
    assert np.abs(pr.rhs(np.full(pr.dof, 2.5))).max() <= 1e-12
    for d, b in ((2, (1.0, 0.5)), (3, (1.0, 1.0, 1.0)), (3, (-0.3, 0.7, 1.1))):
        pr = O.Problem(d, 3, [5] * d, [0.0] * d, [1.0] * d, b)
        assert np.abs(pr.rhs(np.full(pr.dof, -0.6))).max() <= 1e-12


def test_conservation():  # test_spatial.cpp:91-119
    pr = adv1d(7, 2)
    u = pr.interpolate(lambda x, y, z: np.sin(2 * np.pi * x) + 0.2)
    assert abs(np.sum(pr.mass() * pr.rhs(u))) <= 1e-11
    for d, b in ((2, (1.0, 0.5)), (3, (1.0, 1.0, 1.0))):
        pr = O.Problem(d, 3, [4] * d, [0.0] * d, [1.0] * d, b)
        u = np.random.default_rng(5).uniform(-1, 1, pr.dof)
        assert abs(np.sum(pr.mass() * pr.rhs(u))) <= 1e-11


def test_dimension_reduction_2d():  # test_spatial.cpp:121-145
    cells, p = 5, 2
    f = lambda x: np.sin(2 * np.pi * x) + 0.3 * x * x
    s1 = adv1d(cells, p)
    r1 = s1.rhs(s1.interpolate(lambda x, y, z: f(x)))
    s2 = O.Problem(2, p, [cells, cells], [0, 0], [1, 1], (1.0, 0.0))
    r2 = s2.rhs(s2.interpolate(lambda x, y, z: f(x)))
    n = p + 1
    r2 = r2.reshape(cells, cells, n, n)  # [cy][cx][iy][ix]
    r1 = r1.reshape(cells, n)            # [cx][ix]
    assert np.abs(r2 - r1[None, :, None, :]).max() < 1e-12


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_dimension_reduction_3d(axis):  # EXTENSION: 3-D analogue of test_spatial.cpp:121-145
    cells, p = 4, 3
    n = p + 1
    f = lambda x: np.sin(2 * np.pi * x) + 0.3 * x * x
    s1 = adv1d(cells, p, b=0.8)
    r1 = s1.rhs(s1.interpolate(lambda x, y, z: f(x))).reshape(cells, n)
    b = [0.0, 0.0, 0.0]
    b[axis] = 0.8
    s3 = O.Problem(3, p, [cells] * 3, [0] * 3, [1] * 3, b)
    r3 = s3.rhs(s3.interpolate(lambda x, y, z: f((x, y, z)[axis])))
    r3 = r3.reshape(cells, cells, cells, n, n, n)  # [cz][cy][cx][iz][iy][ix]
    r3 = np.moveaxis(r3, (2 - axis, 5 - axis), (-2, -1))  # bring the active axis last
    assert np.abs(r3 - r1).max() < 1e-12


def test_consistency_order():  # test_spatial.cpp:147-167
    def err_at(cells):
        pr = adv1d(cells, 2)
        u = pr.interpolate(lambda x, y, z: np.sin(2 * np.pi * x))
        ex = pr.interpolate(lambda x, y, z: -2 * np.pi * np.cos(2 * np.pi * x))
        r = pr.rhs(u) - ex
        return math.sqrt(np.sum(r * r * pr.mass()))
    e8, e16 = err_at(8), err_at(16)
    assert e16 < 0.05 and 3.5 < e8 / e16 < 4.5


def test_jacobian_exact_linear():  # test_spatial.cpp:268-291
    pr = adv1d(6, 1)
    u = pr.interpolate(lambda x, y, z: np.cos(2 * np.pi * x))
    assert np.abs(pr.spatial_jvp(u, u) - pr.rhs(u)).max() < 1e-12
    v = np.random.default_rng(1).uniform(-1, 1, pr.dof)
    a = pr.spatial_jvp(u, v)
    b = pr.spatial_jvp(np.full(pr.dof, 0.8), v)
    assert np.abs(a - b).max() < 1e-13


def test_jacobian_one_ring():  # test_spatial.cpp:293-306
    pr = adv1d(8, 2)
    n = 3
    J = np.stack([pr.spatial_jvp(np.zeros(pr.dof), e) for e in np.eye(pr.dof)], axis=1)
    rows, cols = np.nonzero(J)
    rc, cc = rows // n, cols // n
    assert np.all((rc == cc) | ((cc + 1) % 8 == rc) | ((cc - 1) % 8 == rc))


# ---- slab residual (test_stdg.cpp) ------------------------------------------
def make_testeq(n_tau):
    return O.Problem(1, 1, [1], [0.0], [1.0], [0.0], O.TEST_EQUATION, n_tau=n_tau)


def test_st_residual_vanishes_at_rk_stages():  # test_stdg.cpp:42-51
    pr = make_testeq(2)
    U, un1, _, _ = pr.rk_step(2, O.A_FORM, 0.0, 0.1, [4.0])
    assert np.abs(pr.st_residual(0.0, 0.1, [4.0], U)).max() <= 1e-12


def test_st_residual_constant_and_dt_structure():  # test_stdg.cpp:53-73
    z = O.Problem(1, 1, [1], [0.0], [1.0], [0.0], O.ZERO_SYSTEM, n_tau=3)
    assert np.abs(z.st_residual(0.0, 0.25, [2.5], np.full(3, 2.5))).max() <= 1e-15
    adv = adv1d(4, 1, n_tau=3)
    dof = adv.dof
    U = np.linspace(-0.7, 1.3, 3 * dof)
    _, w = O.lgl(3)
    f = np.concatenate([w[i] * adv.rhs(U[i * dof:(i + 1) * dof]) for i in range(3)])
    diff = adv.st_residual(0.0, 0.2, np.zeros(dof), U) - adv.st_residual(0.0, 0.1, np.zeros(dof), U)
    assert np.abs(diff + 0.05 * f).max() <= 1e-14


def test_st_jacobian_hand_example():  # test_stdg.cpp:75-86
    pr = make_testeq(2)
    J = np.stack([pr.st_jvp(0.0, 0.0, np.full(2, 4.0), e) for e in np.eye(2)], axis=1)
    assert np.allclose(J, [[0.5, 0.5], [-0.5, 0.5]], rtol=1e-14, atol=1e-15)


def test_st_jacobian_fd():  # test_stdg.cpp:88-109
    adv = adv1d(4, 1, n_tau=3)
    dof = adv.dof
    un = np.linspace(0.1, 0.9, dof)
    U = np.sin(0.7 * np.arange(3 * dof) + 0.3)
    rng = np.random.default_rng(17)
    h = 1e-6
    for _ in range(3):
        v = rng.uniform(-1, 1, 3 * dof)
        fd = (adv.st_residual(0.2, 0.13, un, U + h * v) - adv.st_residual(0.2, 0.13, un, U - h * v)) / (2 * h)
        jv = adv.st_jvp(0.2, 0.13, U, v)
        assert np.abs(fd - jv).max() <= 1e-6 * (1 + np.abs(jv).max())


def test_stdg_equals_rk_step():  # test_stdg.cpp:111-135
    pr = make_testeq(2)
    _, un1, _, _ = pr.stdg_step(0.0, 0.1, [4.0])
    assert abs(un1[0] - 3.6199095) <= 1e-7 * 3.6199095
    _, rk1, _, _ = pr.rk_step(2, O.A_FORM, 0.0, 0.1, [4.0])
    assert abs(un1[0] - rk1[0]) <= 1e-11
    for n_tau in (2, 3):
        adv = adv1d(8, 2, n_tau=n_tau)
        u0 = adv.interpolate(lambda x, y, z: np.sin(2 * np.pi * x) + 0.3)
        Ua, ua, _, _ = adv.stdg_step(0.0, 0.05, u0)
        Ub, ub, _, _ = adv.rk_step(n_tau, O.A_INV_FORM, 0.0, 0.05, u0)
        assert np.linalg.norm(ua - ub) / np.linalg.norm(ub) <= 1e-10
        assert np.abs(Ua - Ub).max() <= 1e-9


def test_stdg_zero_system_bitwise():  # test_stdg.cpp:137-143
    z = O.Problem(1, 1, [1], [0.0], [1.0], [0.0], O.ZERO_SYSTEM, n_tau=3)
    _, un1, it, _ = z.stdg_step(0.0, 0.4, [2.5])
    assert it == 0 and un1[0] == 2.5


def test_st_jacobian_row_scaling_of_ainv_form():  # test_stdg.cpp:145-167
    dt = 0.07
    for p in (1, 2, 3):
        n_tau = p + 1
        adv = adv1d(1, p, n_tau=n_tau)
        dof = adv.dof
        U = np.linspace(-0.2, 1.0, n_tau * dof)
        E = np.eye(n_tau * dof)
        Jst = np.stack([adv.st_jvp(0.0, dt, U, e) for e in E], axis=1)
        Ja = np.stack([adv.stage_jvp(n_tau, O.A_INV_FORM, 0.0, dt, U, e) for e in E], axis=1)
        _, w = O.lgl(n_tau)
        scale = 0.5 * dt * np.kron(np.diag(w), np.eye(dof))
        assert np.abs(Jst - scale @ Ja).max() <= 1e-12
        # sparsity_of drops entries below 1e-14 x max-norm
        pat = lambda M: np.abs(M) > 1e-14 * np.abs(M).max()
        assert np.array_equal(pat(Jst), pat(Ja))


def test_stdg_testeq_eoc():  # test_stdg.cpp:169-192
    pr = make_testeq(3)

    def err(nsteps):
        u = np.array([4.0])
        dt = 1.0 / nsteps
        for k in range(nsteps):
            _, u, _, _ = pr.stdg_step(k * dt, dt, u)
        return abs(u[0] - 4 * math.exp(-1))
    assert abs(math.log2(err(8) / err(16)) - 3.96) <= 0.03 * 3.96


# ---- LoDG (test_lodg.cpp) ---------------------------------------------------
def test_rk_step_testeq_kat():  # test_lodg.cpp:38-55
    pr = make_testeq(2)
    A, _, _ = O.lobatto(2)
    Uo = np.linalg.solve(np.eye(2) + 0.1 * A, np.full(2, 4.0))
    assert abs(Uo[1] - 4.0 / 1.105) <= 1e-12 * Uo[1]
    for form in (O.A_FORM, O.A_INV_FORM):
        U, un1, it, _ = pr.rk_step(2, form, 0.0, 0.1, [4.0])
        assert abs(un1[0] - 3.6199095) <= 1e-7 * 3.6199095
        assert abs(un1[0] - Uo[1]) <= 1e-12 * Uo[1]
        assert np.allclose(U, Uo, rtol=1e-12, atol=0)
        assert it == 1


def test_rk_stiffly_accurate():  # test_lodg.cpp:64-81
    pr = make_testeq(2)
    for s in (2, 3, 4):
        U, un1, _, _ = pr.rk_step(s, O.A_FORM, 0.0, 0.2, [4.0])
        assert abs(un1[0] - U[-1]) <= 1e-12
    adv = adv1d(16, 2)
    u0 = adv.interpolate(lambda x, y, z: np.sin(2 * np.pi * x))
    for form in (O.A_FORM, O.A_INV_FORM):
        U, un1, _, _ = adv.rk_step(3, form, 0.0, 0.01, u0)
        assert np.abs(un1 - U[-adv.dof:]).max() <= 1e-12


def test_rk_forms_agree_and_linear_one_iteration():  # test_lodg.cpp:83-95, 123-132
    adv = adv1d(8, 2)
    u0 = adv.interpolate(lambda x, y, z: np.exp(np.sin(2 * np.pi * x)))
    for s in (2, 3):
        _, a, _, _ = adv.rk_step(s, O.A_FORM, 0.0, 0.05, u0)
        _, b, _, _ = adv.rk_step(s, O.A_INV_FORM, 0.0, 0.05, u0)
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-11
    adv = adv1d(8, 1)
    u0 = adv.interpolate(lambda x, y, z: np.cos(2 * np.pi * x))
    for form in (O.A_FORM, O.A_INV_FORM):
        assert adv.rk_step(2, form, 0.0, 0.1, u0)[2] == 1


def test_stage_jacobian_hand_example():  # test_lodg.cpp:97-121
    pr = make_testeq(2)
    U = np.full(2, 4.0)
    J = np.stack([pr.stage_jvp(2, O.A_FORM, 0.0, 1.0, U, e) for e in np.eye(2)], axis=1)
    assert np.allclose(J, [[1.5, -0.5], [0.5, 1.5]], rtol=1e-14)
    adv = adv1d(4, 1, n_tau=3)
    dof = adv.dof
    st = np.tile(np.linspace(-0.3, 1.1, dof), 3)
    E = np.eye(3 * dof)
    Ja = np.stack([adv.stage_jvp(3, O.A_FORM, 0.1, 0.2, st, e) for e in E], axis=1)
    Ji = np.stack([adv.stage_jvp(3, O.A_INV_FORM, 0.1, 0.2, st, e) for e in E], axis=1)
    A3, _, _ = O.lobatto(3)
    P = np.kron(np.linalg.inv(0.2 * A3), np.eye(dof))
    assert np.abs(P @ Ja - Ji).max() <= 1e-12


def test_nonconvergence_raises():  # test_lodg.cpp:179-194
    pr = make_testeq(2)
    with pytest.raises(O.OracleError) as ei:
        pr.rk_step(2, O.A_FORM, 0.5, 0.1, [4.0], max_iter=0)
    assert ei.value.code == 3


# ---- linear solvers (test_newton.cpp) ---------------------------------------
def test_gmres_vs_dense_spd():  # test_newton.cpp:50-58 (the only GMRES pin)
    rng = np.random.default_rng(3)
    R = rng.uniform(-1, 1, (50, 50))
    A = R @ R.T + 50 * np.eye(50)
    b = rng.uniform(-1, 1, 50)
    xd = O.lu_solve_dense(A, b)
    xg, it, rr = O.gmres_dense(A, b)
    assert np.abs(xd - xg).max() < 1e-8
    assert np.abs(xd - np.linalg.solve(A, b)).max() < 1e-10


def test_slab_gmres_matches_dense():  # GMRES branch vs dense LU on a slab (newton.hpp:51-86)
    adv = adv1d(8, 3)
    u0 = adv.interpolate(lambda x, y, z: np.sin(2 * np.pi * x))
    Ud, _, _, _ = adv.stdg_step(0.0, 0.005, u0, linear=O.DENSE_LU)
    Ug, _, it, lin = adv.stdg_step(0.0, 0.005, u0, linear=O.GMRES, gmres_tol=1e-13)
    assert np.abs(Ud - Ug).max() <= 1e-11 * np.abs(Ud).max()
    assert lin > 0


# ---- Burgers extension (NOT in the reference; parity unpinned) ---------------
def burgers(cells=8, p=3):
    return O.Problem(1, p, [cells], [0.0], [2 * np.pi], [0.0], O.BURGERS)


def test_burgers_free_stream_and_conservation():
    pr = burgers()
    assert np.abs(pr.rhs(np.full(pr.dof, 1.3))).max() <= 1e-12
    u = pr.interpolate(lambda x, y, z: 1 + 0.5 * np.sin(x)) + np.random.default_rng(2).normal(0, 0.01, pr.dof)
    F = pr.rhs(u)
    assert abs(np.sum(pr.mass() * F)) <= 1e-11
    # LLF interface + EC volume is entropy stable: d/dt sum(M u^2/2) <= 0
    assert np.sum(pr.mass() * u * F) <= 1e-12


def test_burgers_jvp_fd():
    pr = burgers()
    u = pr.interpolate(lambda x, y, z: 1 + 0.5 * np.sin(x))
    v = np.random.default_rng(4).uniform(-1, 1, pr.dof)
    h = 1e-6
    fd = (pr.rhs(u + h * v) - pr.rhs(u - h * v)) / (2 * h)
    jv = pr.spatial_jvp(u, v)
    assert np.abs(fd - jv).max() <= 1e-6 * (1 + np.abs(jv).max())
