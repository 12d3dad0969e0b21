"""GPU parity for the general flux models: the rotating
pulse (advdiff_model + interior penalty) and 2-D Euler, through the C ABI,
against the CPU oracle (tests/test_oracle_general.py pins the oracle), plus
the reference's acceptance criteria 5, 6 and 9 run on the device."""
import math

import numpy as np
import pytest

import oracle as O
from paper_2201_05800_b200 import configs as C
from paper_2201_05800_b200 import _lib as L

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2201_05800_b200.api import (  # noqa: E402
    AdmissibilityError, NewtonConfig, SlabOperator,
)

TOL_OP = 1e-12
TOL_SOLVE = 1e-10


def rel(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")


def pulse_pair(cells, p, n_tau=None, eps=0.001, field=L.STG_FIELD_ROTATING, vel=(0.0, 0.0),
               dim=2, eta=0.0):
    n_tau = n_tau or p + 1
    cells = [cells] * dim if np.isscalar(cells) else list(cells)
    op = SlabOperator(dim, p, n_tau, cells, [0.0] * dim, [1.0] * dim, velocity=vel,
                      model=L.STG_MODEL_ADVDIFF, velocity_field=field, eps=eps, eta=eta)
    pr = O.Problem(dim, p, cells, [0.0] * dim, [1.0] * dim, velocity=vel, model=O.ADVDIFF,
                   field=field, eps=eps, eta=eta, n_tau=n_tau)
    return op, pr


def euler_pair(cells, p, n_tau=2):
    op = SlabOperator(2, p, n_tau, [cells, cells], [-10.0, -10.0], [10.0, 10.0],
                      model=L.STG_MODEL_EULER)
    pr = O.Problem(2, p, [cells, cells], [-10.0, -10.0], [10.0, 10.0], model=O.EULER,
                   n_tau=n_tau)
    return op, pr


def pulse_u(pr, t=0.0):
    X = pr.coords()
    return C.rotating_pulse_exact(t, X[:, 0], X[:, 1])


def vortex_u(pr):
    X = pr.coords()
    return C.vortex_initial(X[:, 0], X[:, 1]).reshape(-1)


GENERAL = [
    ("pulse p1", lambda: pulse_pair((5, 4), 1)),
    ("pulse p2", lambda: pulse_pair(6, 2)),
    ("pulse p3", lambda: pulse_pair((4, 7), 3)),
    ("advdiff const 2d", lambda: pulse_pair((5, 3), 2, field=L.STG_FIELD_CONSTANT,
                                            vel=(0.7, -1.3), eps=0.05)),
    ("advdiff 1d", lambda: pulse_pair(7, 3, field=L.STG_FIELD_CONSTANT, vel=(1.5,), eps=0.02,
                                      dim=1)),
    ("advection var b (eps 0)", lambda: pulse_pair(5, 2, eps=0.0)),
    ("pulse eta", lambda: pulse_pair(4, 2, eta=3.5)),
    ("euler p1", lambda: euler_pair(4, 1)),
    ("euler p2", lambda: euler_pair(5, 2, n_tau=3)),
]


def state_of(op, pr, seed=0):
    rng = np.random.default_rng(seed)
    if op.model == L.STG_MODEL_EULER:
        u = vortex_u(pr)
        return u * (1.0 + 0.01 * rng.uniform(-1, 1, u.size))
    return pulse_u(pr) + 0.1 * rng.uniform(-1, 1, pr.dof)


@pytest.mark.parametrize("name,make", GENERAL, ids=[g[0] for g in GENERAL])
def test_spatial_rhs_parity(name, make):
    op, pr = make()
    assert op.n_sdof == pr.dof
    u = state_of(op, pr)
    assert rel(op.spatial_rhs(dev(u)), pr.rhs(u)) <= TOL_OP


@pytest.mark.parametrize("name,make", GENERAL, ids=[g[0] for g in GENERAL])
def test_slab_residual_and_stage_residual_parity(name, make):
    op, pr = make()
    nt = op.n_tau
    un = state_of(op, pr, 1)
    U = np.concatenate([state_of(op, pr, 2 + j) for j in range(nt)])
    dt = 0.01
    assert rel(op.st_residual(0.0, dt, dev(un), dev(U)), pr.st_residual(0.0, dt, un, U)) <= TOL_OP
    if nt in (2, 3, 4):
        for form in (L.STG_FORM_A, L.STG_FORM_A_INV):
            got = op.stage_residual(form, 0.0, dt, dev(un), dev(U))
            assert rel(got, pr.stage_residual(nt, form, 0.0, dt, un, U)) <= TOL_OP


def test_linear_jvp_parity():
    op, pr = pulse_pair(6, 2)
    U = np.concatenate([pulse_u(pr)] * op.n_tau)
    v = np.random.default_rng(3).uniform(-1, 1, op.n_dof)
    assert rel(op.st_jvp(0.0, 0.02, dev(U), dev(v)), pr.st_jvp(0.0, 0.02, U, v)) <= TOL_OP


def test_euler_jvp_close_to_central_difference():
    op, pr = euler_pair(4, 1)
    u = vortex_u(pr)
    v = np.random.default_rng(42).uniform(-1.0, 1.0, pr.dof)
    Jv = op.spatial_jvp(dev(u), dev(v)).cpu().numpy()
    h = 1e-6
    fd = (pr.rhs(u + h * v) - pr.rhs(u - h * v)) / (2 * h)
    assert np.abs(fd - Jv).max() <= 1e-5 * np.abs(fd).max()  # test_spatial.cpp:308-326


def test_free_stream_and_conservation_on_device():  # test_spatial.cpp:67-118
    op, pr = pulse_pair(5, 3)
    assert np.abs(op.spatial_rhs(dev(np.full(op.n_sdof, -0.6))).cpu().numpy()).max() <= 1e-12
    op, pr = euler_pair(4, 2)
    F = op.spatial_rhs(dev(vortex_u(pr))).cpu().numpy()
    mF = pr.mass() * F
    for comp in range(4):
        assert abs(mF[comp::4].sum()) <= 1e-11


def test_admissibility_error_names_temporal_node():  # stdg.hpp:41-50, models.hpp:108-113
    op, pr = euler_pair(2, 1)
    good = np.tile([1.0, 0.3, -0.2, 2.5], op.n_sdof // 4)
    bad = np.tile([1.0, 4.0, 0.0, 1.0], op.n_sdof // 4)
    U = np.concatenate([good, bad])
    with pytest.raises(AdmissibilityError, match="temporal node 1"):
        op.st_residual(0.0, 0.01, dev(good), dev(U))
    # the handle recovers
    v = vortex_u(pr)
    V = np.concatenate([v, v * 1.01])
    assert rel(op.st_residual(0.0, 0.01, dev(v), dev(V)), pr.st_residual(0.0, 0.01, v, V)) <= TOL_OP


def test_admissibility_error_inside_a_solve():
    # inside stdg_step the flag is checked at the Newton step's sync points
    # (not after every apply): the same error surfaces from the same call,
    # and the handle solves normally afterwards
    op, pr = euler_pair(2, 1)
    bad = np.tile([1.0, 4.0, 0.0, 1.0], op.n_sdof // 4)  # negative pressure
    nc = NewtonConfig(abs_tol=1e-10, rel_tol=1e-10, gmres_tol=1e-12)
    with pytest.raises(AdmissibilityError, match="temporal node"):
        op.stdg_step(0.0, 0.01, dev(bad), nc)
    v = vortex_u(pr)
    U, u1, info = op.stdg_step(0.0, 0.01, dev(v), nc)
    assert info.newton_iterations >= 1
    Uo, _, _, _ = pr.stdg_step(0.0, 0.01, v, abs_tol=1e-10, rel_tol=1e-10, linear=O.DENSE_LU)
    assert rel(U, Uo) <= 1e-8


def test_general_model_preconditioner_resolution():
    op, pr = pulse_pair(4, 1)
    v = dev(np.ones(op.n_dof))
    with pytest.raises(ValueError):  # temporal blocks: constant-velocity advection only
        op.st_precond_apply(0.1, v, precond=L.STG_PRECOND_TBLOCK)
    a = op.st_precond_apply(0.1, v)  # AUTO -> element blocks for advdiff
    b = op.st_precond_apply(0.1, v, precond=L.STG_PRECOND_EBLOCK)
    assert torch.equal(a, b)
    eo, _ = euler_pair(4, 1)  # nonlinear Euler: no block preconditioner (AUTO = identity)
    ve = dev(np.ones(eo.n_dof))
    assert float((eo.st_precond_apply(0.1, ve, dev(np.tile([1.0, 0.3, -0.2, 2.5], eo.n_dof // 4)))
                  - ve).abs().max()) == 0.0
    with pytest.raises(ValueError):
        eo.st_precond_apply(0.1, ve, dev(np.ones(eo.n_dof)), precond=L.STG_PRECOND_EBLOCK)


@pytest.mark.parametrize("cells,p,nt,field,vel", [(6, 2, 3, L.STG_FIELD_ROTATING, (0.0, 0.0)),
                                                  (5, 1, 2, L.STG_FIELD_CONSTANT, (0.7, -1.1))])
def test_general_eblock_is_exact_local_inverse(cells, p, nt, field, vel):
    """advdiff element blocks (coloured probing, kernels_precond.cu) = the exact
    inverse of each element's local Jacobian block, read off the oracle's J.v."""
    op, pr = pulse_pair(cells, p, n_tau=nt, field=field, vel=vel, eps=0.01)
    ns, npc = op.n_sdof, (p + 1) ** 2
    dt = 0.03
    rng = np.random.default_rng(5)
    x = rng.standard_normal(nt * ns)
    y = op.st_precond_apply(dt, dev(x), precond=L.STG_PRECOND_EBLOCK).cpu().numpy()
    U0 = np.zeros(nt * ns)
    for cell in (0, cells + 1, cells * cells - 1):  # the velocity field varies per cell
        loc = np.array([t * ns + cell * npc + k for t in range(nt) for k in range(npc)])
        Lblk = np.zeros((loc.size, loc.size))
        for c, i in enumerate(loc):
            e = np.zeros(nt * ns)
            e[i] = 1.0
            Lblk[:, c] = pr.st_jvp(0.0, dt, U0, e)[loc]
        assert rel(y[loc], np.linalg.solve(Lblk, x[loc])) <= 1e-11, cell


def test_pulse_eblock_same_solution_fewer_iterations():
    op, pr = pulse_pair(16, 2)
    u = dev(pulse_u(pr))
    res = {}
    for pc in (L.STG_PRECOND_NONE, L.STG_PRECOND_EBLOCK):
        nc = NewtonConfig(abs_tol=1e-13, rel_tol=1e-13, gmres_tol=1e-13, gmres_max_it=5000,
                          precond=pc)
        U, u1, info = op.stdg_step(0.0, 1.0 / 16, u, nc)
        res[pc] = (U.cpu().numpy(), info.linear_iterations)
    assert rel(res[L.STG_PRECOND_EBLOCK][0], res[L.STG_PRECOND_NONE][0]) <= TOL_SOLVE
    assert res[L.STG_PRECOND_EBLOCK][1] * 5 < res[L.STG_PRECOND_NONE][1], res


def test_pulse_slab_solves_match_oracle():
    op, pr = pulse_pair(8, 2)
    u = pulse_u(pr)
    kw = dict(abs_tol=1e-13, rel_tol=1e-13, linear=O.GMRES, gmres_tol=1e-14, gmres_max_it=5000)
    Uo, uo, _, _ = pr.stdg_step(0.0, 0.0625, u, **kw)
    nc = NewtonConfig(abs_tol=1e-13, rel_tol=1e-13, gmres_tol=1e-14, gmres_max_it=5000)
    U, u1, info = op.stdg_step(0.0, 0.0625, dev(u), nc)
    assert rel(U, Uo) <= TOL_SOLVE
    for form in (L.STG_FORM_A, L.STG_FORM_A_INV):
        Uo, uo, _, _ = pr.rk_step(3, form, 0.0, 0.0625, u, **kw)
        U, u1, info = op.rk_step(form, 0.0, 0.0625, dev(u), nc)
        assert rel(U, Uo) <= TOL_SOLVE
        assert rel(u1, uo) <= TOL_SOLVE


def test_euler_stage_solve_matches_oracle():
    op, pr = euler_pair(8, 1)
    u = vortex_u(pr)
    Uo, uo, _, _ = pr.rk_step(2, 0, 0.0, 0.05, u, abs_tol=1e-12, rel_tol=1e-13,
                              linear=O.GMRES, gmres_tol=1e-9, gmres_max_it=5000)
    nc = NewtonConfig(abs_tol=1e-12, rel_tol=1e-13, gmres_tol=1e-9, gmres_max_it=5000)
    U, u1, info = op.rk_step(L.STG_FORM_A, 0.0, 0.05, dev(u), nc)
    # both Newton iterations converge to ||R||_inf <= 1e-12 with FD J.v
    assert rel(u1, uo) <= 1e-10


def test_criterion5_pulse_step_equivalence_on_device():  # acceptance.cpp:221-261
    for n_tau in (2, 3):
        op, pr = pulse_pair(8, n_tau - 1, n_tau=n_tau)
        u = dev(pulse_u(pr))
        nc = NewtonConfig(abs_tol=1e-13, rel_tol=1e-13, gmres_tol=1e-14, gmres_max_it=5000)
        t, dt = 0.0, 0.125
        for _ in range(4):
            _, lo, _ = op.rk_step(L.STG_FORM_A, t, dt, u, nc)
            _, st, _ = op.stdg_step(t, dt, u, nc)
            gap = float((lo - st).abs().max() / (1.0 + st.abs().max()))
            assert gap <= 1e-9
            u, t = st, t + dt


PULSE_TABLE = [(2, 8, 4.66e-2, 4.46e-2), (2, 16, 3.49e-2, 3.39e-2),
               (3, 8, 2.42e-2, 2.41e-2), (3, 16, 5.36e-3, 5.38e-3)]  # acceptance.cpp:265-269


@pytest.mark.parametrize("n_tau,N,lodg_ref,stdg_ref", PULSE_TABLE)
def test_criterion6_pulse_error_table_on_device(n_tau, N, lodg_ref, stdg_ref):
    op, pr = pulse_pair(N, n_tau - 1, n_tau=n_tau)
    m = pr.mass()
    exact = pulse_u(pr, 1.0)
    nc = NewtonConfig(gmres_tol=1e-12, gmres_max_it=5000)
    for method, ref in (("lodg", lodg_ref), ("stdg", stdg_ref)):
        u, dt = dev(pulse_u(pr)), 1.0 / N
        for k in range(N):
            if method == "lodg":
                _, u, _ = op.rk_step(L.STG_FORM_A, k * dt, dt, u, nc)
            else:
                _, u, _ = op.stdg_step(k * dt, dt, u, nc)
        d = u.cpu().numpy() - exact
        err = math.sqrt(float(np.dot(m, d * d)))
        assert abs(err / ref - 1.0) <= 0.25, (method, err, ref)


def _euler_vortex(n_steps, dt, cells=16):  # experiments.hpp:188-262 (lodg, A-form)
    op, pr = euler_pair(cells, 1, n_tau=2)
    u = dev(vortex_u(pr))
    min_rho, max_newton, t = float(u[0::4].min()), 0, 0.0
    nc = NewtonConfig(gmres_tol=1e-8, gmres_max_it=5000)
    for _ in range(n_steps):
        _, u, info = op.rk_step(L.STG_FORM_A, t, dt, u, nc)
        t += dt
        max_newton = max(max_newton, info.newton_iterations)
        min_rho = min(min_rho, float(u[0::4].min()))
    X = pr.coords()
    xb = X[:, 0] - t
    xb -= 20.0 * np.floor((xb + 10.0) / 20.0)
    rho_exact = C.vortex_initial(xb, X[:, 1])[:, 0]
    m = pr.mass()[0::4]
    err = math.sqrt(float(np.dot(m, (u[0::4].cpu().numpy() - rho_exact) ** 2)))
    return err, min_rho, max_newton


def test_criterion9_euler_vortex_on_device():  # acceptance.cpp:451-466
    e_full, rho_full, nit = _euler_vortex(10, 0.05)
    assert rho_full > 0.0 and nit <= 10
    e_half, rho_half, _ = _euler_vortex(20, 0.025)
    assert rho_half > 0.0
    assert e_half / e_full <= 1.005
