"""GPU: the d = 1 upwind block sweep (STG_PRECOND_SWEEP, kernels_precond.cu
k_eblock2 + k_sweep_win) against dense numpy solves built from the oracle's
exact Burgers Jacobian.

P = J without its downwind part: the element blocks plus each element's
inflow coupling to its left neighbour (rows at node 0, columns at the left
neighbour's node N).  The sweep solves P z = x around the periodic ring up
to the fp32 storage of the blocks (a preconditioner; the GMRES it serves
stays fp64) and the 32-element window of its recurrence (the transfer
through 32 elements is ~1e-23 at these CFL numbers).  Small meshes (rings
shorter than the window included) compare with np.linalg.solve; c3-sized
rings check the residual P z - x with J z from the oracle and the downwind
part from the LLF derivative (spatial.hpp:20-25 with f = u^2/2).
"""
import numpy as np
import pytest

import oracle as O
from paper_2201_05800_b200 import configs as C
from paper_2201_05800_b200 import _lib as L

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2201_05800_b200.api import NewtonConfig, SlabOperator  # noqa: E402

TOL_F32 = 2e-5  # fp32 element blocks and couplings
TOL_SOLVE = 1e-10


def rel(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")


def burgers(cells, degree=3):
    cfg = C.Config(f"bg{cells}", 1, degree, 4, (cells,), (0.0,), (2 * np.pi,), (0.0,), 1e-4,
                   "burgers", 2, model=L.STG_MODEL_BURGERS)
    pr = O.Problem(1, degree, [cells], [0.0], [2 * np.pi], [0.0], model=O.BURGERS, n_tau=4)
    return cfg, SlabOperator(**cfg.kwargs()), pr


def state(cfg, seed=5, amp=0.05):
    un = C.initial_state(cfg)
    rng = np.random.default_rng(seed)
    return np.concatenate([un + amp * rng.uniform(-1, 1, un.size) for _ in range(cfg.n_tau)])


def downwind_action(cfg, dt, U, z):
    """The Jacobian's downwind part applied to z: rows (r, node N) of element
    e, columns (j, node 0) of element e + 1; S = -(dt/2) M_tau (diagonal),
    coupling -(2/h)(1/w_N) dH/du_R at each temporal node."""
    n1, nt, K = cfg.degree + 1, cfg.n_tau, cfg.cells[0]
    ns = K * n1
    h = (cfg.upper[0] - cfg.lower[0]) / K
    xi, w = O.lgl(n1)
    tau_w = O.lgl(nt)[1]
    out = np.zeros_like(z)
    for t in range(nt):
        Ut = U[t * ns:(t + 1) * ns].reshape(K, n1)
        zt = z[t * ns:(t + 1) * ns].reshape(K, n1)
        uL, uR = Ut[:, -1], np.roll(Ut[:, 0], -1)
        aL, aR = np.abs(uL), np.abs(uR)
        dH = np.where(aL >= aR, 0.5 * uR - 0.5 * aL,
                      0.5 * uR + 0.5 * np.sign(uR) * (uL - uR) - 0.5 * aR)
        coup = -(2.0 / h) * (1.0 / w[-1]) * dH
        S = -0.5 * dt * tau_w[t]
        blk = np.zeros((K, n1))
        blk[:, -1] = S * coup * np.roll(zt[:, 0], -1)
        out[t * ns:(t + 1) * ns] = blk.ravel()
    return out


def dense_J(pr, dt, U):
    n = U.size
    J = np.zeros((n, n))
    for k in range(n):
        e = np.zeros(n)
        e[k] = 1.0
        J[:, k] = pr.st_jvp(0.0, dt, U, e)
    return J


@pytest.mark.parametrize("cells,dt", [(16, 0.1), (130, 0.02), (300, 0.01)])
def test_sweep_is_exact_lower_block_solve(cells, dt):
    cfg, op, pr = burgers(cells)
    U = state(cfg)
    J = dense_J(pr, dt, U)
    D = np.stack([downwind_action(cfg, dt, U, e) for e in np.eye(U.size)], axis=1)
    # the downwind formula is exactly the Jacobian's entries at those positions
    n1, ns = cfg.degree + 1, cells * (cfg.degree + 1)
    mask = np.zeros_like(J, dtype=bool)
    for t in range(cfg.n_tau):
        for e in range(cells):
            r = t * ns + e * n1 + n1 - 1
            for j in range(cfg.n_tau):
                mask[r, j * ns + ((e + 1) % cells) * n1] = True
    assert np.abs(D[~mask]).max() == 0.0
    assert np.abs(D[mask] - J[mask]).max() <= 1e-12 * np.abs(J).max()
    P = J - D
    x = np.random.default_rng(9).standard_normal(U.size)
    z = op.st_precond_apply(dt, dev(x), dev(U), precond=L.STG_PRECOND_SWEEP).cpu().numpy()
    assert rel(z, np.linalg.solve(P, x)) <= TOL_F32
    # and it is not the block-Jacobi answer (the coupling is live)
    zb = op.st_precond_apply(dt, dev(x), dev(U), precond=L.STG_PRECOND_EBLOCK).cpu().numpy()
    assert rel(zb, np.linalg.solve(P, x)) > 1e-3


@pytest.mark.parametrize("cells", [40000, 65536])
def test_sweep_residual_at_large_ring(cells):
    """Many CTAs (chunk windows reaching into the previous chunk); c3 size."""
    cfg, op, pr = burgers(cells)
    dt = 1e-4
    U = state(cfg, amp=0.01)
    x = np.random.default_rng(3).standard_normal(U.size)
    z = op.st_precond_apply(dt, dev(x), dev(U), precond=L.STG_PRECOND_SWEEP).cpu().numpy()
    Pz = pr.st_jvp(0.0, dt, U, z) - downwind_action(cfg, dt, U, z)
    assert rel(Pz, x) <= TOL_F32
    # repeated applies are deterministic
    z2 = op.st_precond_apply(dt, dev(x), dev(U), precond=L.STG_PRECOND_SWEEP).cpu().numpy()
    assert np.array_equal(z, z2)


def test_sweep_without_jumps_in_negative_flow_is_block_jacobi():
    """u < 0 with no jumps: dH/du_L = (u_0 - u_L)/2 = 0 at every face, so the
    inflow couplings vanish and the sweep is the element-block Jacobi."""
    cfg, op, pr = burgers(64)
    U = np.concatenate([np.full(cfg.n_sdof, -2.0 - 0.1 * t) for t in range(cfg.n_tau)])
    x = np.random.default_rng(4).standard_normal(U.size)
    a = op.st_precond_apply(0.01, dev(x), dev(U), precond=L.STG_PRECOND_SWEEP).cpu().numpy()
    b = op.st_precond_apply(0.01, dev(x), dev(U), precond=L.STG_PRECOND_EBLOCK).cpu().numpy()
    assert rel(a, b) <= 1e-14


def test_sweep_newton_same_solution_fewer_iterations():
    cfg = C.CONFIGS["c3"].scaled((4096,))
    op = SlabOperator(**cfg.kwargs())
    un = dev(C.initial_state(cfg))
    sols, its = [], []
    for pc in (L.STG_PRECOND_EBLOCK, L.STG_PRECOND_SWEEP):
        nc = NewtonConfig(abs_tol=1e-13, rel_tol=1e-12, gmres_tol=1e-12, precond=pc)
        U, _, info = op.stdg_step(0.0, 4 * cfg.dt, un, nc)
        sols.append(U.cpu().numpy())
        its.append(info.linear_iterations)
    assert rel(sols[1], sols[0]) <= TOL_SOLVE
    assert its[1] < 0.7 * its[0], its


def test_sweep_rejected_where_unsupported():
    op = SlabOperator(**C.CONFIGS["c4"].scaled((8, 8, 8)).kwargs())
    v = dev(np.ones(op.n_dof))
    with pytest.raises(ValueError):
        op.st_precond_apply(0.002, v, precond=L.STG_PRECOND_SWEEP)


@pytest.mark.parametrize("form", [L.STG_FORM_A, L.STG_FORM_A_INV])
def test_sweep_stage_solves_match_block_jacobi(form):
    """The sweep's couplings are built from the solve's own temporal mix (a
    full S for the A-form stage system): Burgers rk_step with SWEEP and with
    the element blocks alone converge to the same stages."""
    cfg = C.CONFIGS["c3"].scaled((2048,))
    op = SlabOperator(**cfg.kwargs())
    u = dev(C.initial_state(cfg))
    sols, its = [], []
    for pc in (L.STG_PRECOND_EBLOCK, L.STG_PRECOND_SWEEP):
        nc = NewtonConfig(abs_tol=1e-13, rel_tol=1e-12, gmres_tol=1e-12, precond=pc)
        U, _, info = op.rk_step(form, 0.0, 4 * cfg.dt, u, nc)
        sols.append(U.cpu().numpy())
        its.append(info.linear_iterations)
    assert rel(sols[1], sols[0]) <= TOL_SOLVE
    assert its[1] < its[0], its


@pytest.mark.parametrize("tight", [False, True], ids=["default_budget", "tight_budget"])
def test_lagged_blocks_are_rebuilt_when_the_state_changes(tight):
    """The Burgers element blocks (and sweep couplings) of one step serve the
    next few steps of a march (STG_PRECOND_LAG_STEPS).  A handle that is then
    given an unrelated state still returns the fresh-handle solution: blocks
    that cost clearly more GMRES steps are rebuilt, and with an iteration
    budget the stale blocks cannot meet the solve is repeated with blocks
    built at the current state (newton(), stg.cpp)."""
    cfg = C.CONFIGS["c3"].scaled((4096,))
    x = np.asarray(C.initial_state(cfg))
    n = x.size
    # a shock-forming state far from the smooth initial one
    s = np.linspace(0.0, 2 * np.pi, n, endpoint=False)
    other = dev(1.5 + 1.2 * np.sin(3 * s) + 0.4 * np.cos(7 * s))
    kw = dict(abs_tol=1e-12, rel_tol=1e-10, gmres_tol=1e-8, fd_eps=1e-7)
    fresh = SlabOperator(**cfg.kwargs())
    Uf, uf, inf = fresh.stdg_step(0.0, 4 * cfg.dt, other, NewtonConfig(**kw))
    if tight:  # barely what the fresh blocks need per Newton iteration
        kw["gmres_max_it"] = -(-inf.linear_iterations // inf.newton_iterations) + 2
        Uf, uf, inf = SlabOperator(**cfg.kwargs()).stdg_step(0.0, 4 * cfg.dt, other,
                                                             NewtonConfig(**kw))
    op = SlabOperator(**cfg.kwargs())
    op.stdg_step(0.0, cfg.dt, dev(x), NewtonConfig(**kw))  # blocks built at the smooth state
    Ul, ul, inl = op.stdg_step(0.0, 4 * cfg.dt, other, NewtonConfig(**kw))
    assert rel(Ul, Uf.cpu().numpy()) <= 1e-7  # both solved to the inexact-Newton tolerance
    assert inl.final_residual <= max(1e-12, 1e-10 * inl.residual_history[0])
    # and a march keeps converging with the blocks of its first step
    u = dev(x)
    for k in range(6):
        _, u, info = op.stdg_step(k * cfg.dt, cfg.dt, u, NewtonConfig(**kw))
        assert info.final_residual <= max(1e-12, 1e-10 * info.residual_history[0])
