"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): ||x_gpu - x_cpu||_inf / ||x_cpu||_inf <= 1e-12
for R(U) and J.v; <= 1e-10 for converged slab solutions at the same solver
tolerances.  Oracle-sized cases run every kernel family; the full c4 / c2
sizes are compared directly (the oracle finishes them in seconds) and through
size-independent properties (free stream, linearity, determinism).
"""
import os

import numpy as np
import pytest

import oracle as O
from paper_2201_05800_b200 import configs as C
from paper_2201_05800_b200 import _lib as L

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2201_05800_b200.api import (  # noqa: E402
    NewtonConfig, NonconvergenceError, SlabOperator,
)

TOL_OP = 1e-12
TOL_SOLVE = 1e-10


def rel(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")


def pair(cfg, kernel=L.STG_KERNEL_AUTO):
    op = SlabOperator(**cfg.kwargs(), kernel=kernel)
    pr = O.Problem(cfg.dim, cfg.degree, list(cfg.cells), list(cfg.lower), list(cfg.upper),
                   list(cfg.velocity), model=cfg.model, n_tau=cfg.n_tau)
    return op, pr


def make(dim, degree, n_tau, cells, velocity, model=L.STG_MODEL_ADVECTION, dt=0.01, u0=None):
    lower = (0.0,) * dim
    upper = (1.0,) * dim if model == L.STG_MODEL_ADVECTION else (2 * np.pi,)
    return C.Config(f"t{dim}{degree}{n_tau}", dim, degree, n_tau, tuple(cells), lower, upper,
                    tuple(velocity), dt, u0 or ("burgers" if model else "sin2pi_x"), 7,
                    model=model)


CASES = [
    C.CONFIGS["c1"],                                            # exact c1
    C.CONFIGS["c2"].scaled((8, 8)),                             # c2 physics, small mesh
    C.CONFIGS["c4"].scaled((8, 8, 8)),                          # c4 physics, small mesh
    C.CONFIGS["c3"].scaled((64,)),                              # Burgers
    make(3, 3, 4, (16, 4, 4), (-0.7, 0.4, -1.1)),               # fast kernel, upwind on both sides
    make(3, 3, 4, (6, 5, 3), (0.3, -1.2, 0.8)),                 # generic (nx % 8 != 0)
    make(3, 2, 3, (4, 3, 5), (1.0, 0.5, -0.25)),
    make(2, 2, 3, (5, 7), (-1.0, 0.3)),
    make(2, 3, 2, (4, 4), (0.0, 1.0)),
    make(1, 2, 3, (9,), (-1.5,)),
    make(1, 5, 6, (7,), (0.8,)),
    make(3, 4, 5, (3, 2, 2), (1.0, -1.0, 0.5)),
    # 2-D plane kernel (cells % 32 == 0): negative / zero velocities, and
    # single-cell axes (a cell is its own periodic neighbour)
    make(2, 4, 5, (16, 4), (-0.8, -0.3)),
    make(2, 2, 3, (8, 4), (0.0, -1.2)),
    make(2, 3, 4, (1, 32), (0.7, 0.4)),
    make(2, 3, 4, (32, 1), (-0.7, 0.4)),
    # fast 3-D kernel with one-cell y / z axes
    make(3, 3, 4, (8, 1, 1), (1.0, 0.5, -0.5)),
    make(3, 3, 4, (8, 2, 1), (-1.0, 1.0, 1.0)),
]
IDS = [c.name if c.name[0] == "c" else f"d{c.dim}p{c.degree}nt{c.n_tau}{c.cells}" for c in CASES]


def kernels_for(cfg):
    ks = [L.STG_KERNEL_GENERIC]
    if cfg.dim == 3 and cfg.degree == 3 and cfg.n_tau == 4 and cfg.cells[0] % 8 == 0:
        ks.append(L.STG_KERNEL_FAST)
    return ks


@pytest.mark.parametrize("cfg", CASES, ids=IDS)
def test_st_residual_parity(cfg):
    U = C.random_slab(cfg)
    un = C.initial_state(cfg)
    for k in kernels_for(cfg):
        op, pr = pair(cfg, k)
        ref = pr.st_residual(0.0, cfg.dt, un, U)
        got = op.st_residual(0.0, cfg.dt, dev(un), dev(U))
        assert rel(got, ref) <= TOL_OP, (k, rel(got, ref))


@pytest.mark.parametrize("cfg", CASES, ids=IDS)
def test_st_jvp_parity(cfg):
    U = C.random_slab(cfg)
    if cfg.model == L.STG_MODEL_BURGERS:
        U = 1.0 + 0.3 * U
    v = np.random.default_rng(11).uniform(-1, 1, cfg.n_dof)
    for k in kernels_for(cfg):
        op, pr = pair(cfg, k)
        ref = pr.st_jvp(0.0, cfg.dt, U, v)
        got = op.st_jvp(0.0, cfg.dt, dev(U), dev(v))
        assert rel(got, ref) <= TOL_OP, (k, rel(got, ref))


@pytest.mark.parametrize("cfg", CASES, ids=IDS)
@pytest.mark.parametrize("form", [L.STG_FORM_A, L.STG_FORM_A_INV])
def test_stage_residual_and_jvp_parity(cfg, form):
    if cfg.n_tau > 4:
        pytest.skip("lobatto_tableau closed forms stored for s <= 4 (operators.hpp:76-112)")
    U = C.random_slab(cfg)
    if cfg.model == L.STG_MODEL_BURGERS:
        U = 1.0 + 0.3 * U
    u = C.initial_state(cfg)
    v = np.random.default_rng(5).uniform(-1, 1, cfg.n_dof)
    for k in kernels_for(cfg):
        op, pr = pair(cfg, k)
        ref = pr.stage_residual(cfg.n_tau, form, 0.0, cfg.dt, u, U)
        got = op.stage_residual(form, 0.0, cfg.dt, dev(u), dev(U))
        assert rel(got, ref) <= TOL_OP, ("residual", k, rel(got, ref))
        ref = pr.stage_jvp(cfg.n_tau, form, 0.0, cfg.dt, U, v)
        got = op.stage_jvp(form, 0.0, cfg.dt, dev(U), dev(v))
        assert rel(got, ref) <= TOL_OP, ("jvp", k, rel(got, ref))


@pytest.mark.parametrize("cfg", CASES[:4], ids=IDS[:4])
def test_spatial_rhs_parity(cfg):
    op, pr = pair(cfg)
    u = C.initial_state(cfg) + np.random.default_rng(3).uniform(-0.1, 0.1, cfg.n_sdof)
    assert rel(op.spatial_rhs(dev(u)), pr.rhs(u)) <= TOL_OP
    v = np.random.default_rng(4).uniform(-1, 1, cfg.n_sdof)
    assert rel(op.spatial_jvp(dev(u), dev(v)), pr.spatial_jvp(u, v)) <= TOL_OP


def test_spatial_single_cell_kat():  # test_spatial.cpp:56-65 on the device
    op = SlabOperator(1, 1, 2, (1,), (0.0,), (1.0,), (1.0,))
    A = np.array([[-1.0, 1.0], [1.0, -1.0]])
    for u in (np.array([1.0, 0.0]), np.array([0.3, -0.7])):
        assert np.abs(op.spatial_rhs(dev(u)).cpu().numpy() - A @ u).max() < 1e-14


# ---- full-size configs ---------------------------------------------------------
@pytest.mark.parametrize("name", ["c4", "c2"])
def test_full_size_residual_parity(name):
    cfg = C.CONFIGS[name]
    O.set_threads(O.max_threads())
    op, pr = pair(cfg)
    U = C.random_slab(cfg)
    un = C.initial_state(cfg)
    ref = pr.st_residual(0.0, cfg.dt, un, U)
    got = op.st_residual(0.0, cfg.dt, dev(un), dev(U))
    assert rel(got, ref) <= TOL_OP
    v = np.random.default_rng(cfg.seed + 100).uniform(-1, 1, cfg.n_dof)
    ref = pr.st_jvp(0.0, cfg.dt, U, v)
    got = op.st_jvp(0.0, cfg.dt, dev(U), dev(v))
    assert rel(got, ref) <= TOL_OP


@pytest.mark.parametrize("name", ["c4", "c2"])
def test_full_size_properties(name):
    cfg = C.CONFIGS[name]
    op = SlabOperator(**cfg.kwargs())
    # free stream: U = 1 (x) c with u_n = c gives R = 0 (SBP telescoping + D1 = 0)
    c = dev(np.full(cfg.n_sdof, 0.37))
    U = c.repeat(cfg.n_tau)
    assert op.st_residual(0.0, cfg.dt, c, U).abs().max().item() <= 1e-12
    # linearity: R(U1 + U2; un1 + un2) = R(U1; un1) + R(U2; un2)
    U1, U2 = dev(C.random_slab(cfg, 1)), dev(C.random_slab(cfg, 2))
    u1, u2 = dev(C.initial_state(cfg)), dev(np.cos(C.initial_state(cfg)))
    lhs = op.st_residual(0.0, cfg.dt, u1 + u2, U1 + U2)
    rhs = op.st_residual(0.0, cfg.dt, u1, U1) + op.st_residual(0.0, cfg.dt, u2, U2)
    assert rel(lhs, rhs.cpu().numpy()) <= 1e-13
    # J v = R(v) - R(0) for the linear model
    z = torch.zeros_like(U1)
    jv = op.st_jvp(0.0, cfg.dt, None, U2)
    diff = op.st_residual(0.0, cfg.dt, u1, U2) - op.st_residual(0.0, cfg.dt, u1, z)
    assert rel(jv, diff.cpu().numpy()) <= 1e-13
    # determinism: bitwise identical reruns
    a = op.st_residual(0.0, cfg.dt, u1, U1)
    b = op.st_residual(0.0, cfg.dt, u1, U1)
    assert torch.equal(a, b)


def test_fast_and_generic_kernels_agree_full_c4():
    cfg = C.CONFIGS["c4"]
    fast = SlabOperator(**cfg.kwargs(), kernel=L.STG_KERNEL_FAST)
    gen = SlabOperator(**cfg.kwargs(), kernel=L.STG_KERNEL_GENERIC)
    U, un = dev(C.random_slab(cfg)), dev(C.initial_state(cfg))
    a = fast.st_residual(0.0, cfg.dt, un, U)
    b = gen.st_residual(0.0, cfg.dt, un, U)
    assert rel(a, b.cpu().numpy()) <= 1e-13


@pytest.mark.parametrize("cfg", [
    C.CONFIGS["c4"].scaled((8, 8, 8)),
    make(3, 3, 4, (16, 8, 6), (-0.7, 0.4, -1.1)),      # z-downwind neighbours: pipelined waits
    make(3, 2, 3, (6, 5, 4), (1.0, 1.0, 1.0)),         # generic kernel: plain host path
], ids=["c4small", "negvel", "generic"])
def test_host_buffer_variant_matches_device(cfg):
    op = SlabOperator(**cfg.kwargs())
    U, un = C.random_slab(cfg), C.initial_state(cfg)
    a = op.st_residual_host(0.0, cfg.dt, un, U)
    b = op.st_residual(0.0, cfg.dt, dev(un), dev(U)).cpu().numpy()
    assert np.array_equal(a, b)


@pytest.mark.parametrize("cfg", [
    make(3, 3, 4, (16, 8, 6), (-0.7, 0.4, -1.1)),      # fast kernel, z-downwind neighbours
    make(3, 3, 4, (8, 8, 10), (0.3, -0.4, 1.1)),       # chunks of unequal size (10 layers, K = 8)
    make(2, 4, 5, (40, 32), (1.0, 0.5)),               # plane kernel: staged copies around it
    make(1, 3, 4, (16384,), (1.0,), dt=1e-4),          # lane kernel
], ids=["negvel", "ragged", "d2", "d1"])
def test_pageable_and_pinned_host_buffers_agree(cfg):
    """Pageable caller memory goes through the library's page-locked mirrors
    and worker threads (hostcopy.hpp), page-locked memory straight to the
    copy engines: R(U), the slab step and the stage step return the same bits
    as the device-resident calls either way, call after call."""
    assert cfg.n_dof * 8 >= 1 << 20  # large enough for the staged path
    op = SlabOperator(**cfg.kwargs())
    U, un = C.random_slab(cfg), C.initial_state(cfg)
    Rd = op.st_residual(0.0, cfg.dt, dev(un), dev(U)).cpu().numpy()
    pU = torch.empty(cfg.n_dof, dtype=torch.float64, pin_memory=True)
    pu = torch.empty(cfg.n_sdof, dtype=torch.float64, pin_memory=True)
    pR = torch.empty(cfg.n_dof, dtype=torch.float64, pin_memory=True)
    pU.numpy()[:] = U
    pu.numpy()[:] = un
    for _ in range(3):
        assert np.array_equal(op.st_residual_host(0.0, cfg.dt, un, U), Rd)
        pR.zero_()
        op.st_residual_host(0.0, cfg.dt, pu.numpy(), pU.numpy(), out=pR.numpy())
        assert np.array_equal(pR.numpy(), Rd)
        # mixed: page-locked inputs, pageable result
        assert np.array_equal(op.st_residual_host(0.0, cfg.dt, pu.numpy(), pU.numpy()), Rd)
    nc = NewtonConfig(abs_tol=0.0, rel_tol=1e-9, gmres_tol=1e-10)
    Ud, ud, _ = op.stdg_step(0.0, cfg.dt, dev(un), nc)
    Uh, uh, _ = op.stdg_step_host(0.0, cfg.dt, un, nc)
    assert np.array_equal(Uh, Ud.cpu().numpy()) and np.array_equal(uh, ud.cpu().numpy())
    Uh, uh, _ = op.stdg_step_host(0.0, cfg.dt, pu.numpy(), nc)
    assert np.array_equal(Uh, Ud.cpu().numpy()) and np.array_equal(uh, ud.cpu().numpy())
    Sd, sd, _ = op.rk_step(L.STG_FORM_A_INV, 0.0, cfg.dt, dev(un), nc)
    Sh, sh, _ = op.rk_step_host(L.STG_FORM_A_INV, 0.0, cfg.dt, un, nc)
    assert np.array_equal(Sh, Sd.cpu().numpy()) and np.array_equal(sh, sd.cpu().numpy())


@pytest.mark.parametrize("n", [1 << 18, (1 << 20) + 12345, 5 * (1 << 20) + 777, 9 << 20])
def test_stg_memcpy_pageable_round_trip(n):
    """stg_memcpy and stg_host_alloc (the memory helpers FFI callers use):
    pageable arrays of 2 MiB and more go through the staged ring (several
    slot-sized chunks, ragged tails), page-locked ones straight to the copy
    engine; a round trip through the device returns the same bits."""
    import ctypes
    lib = L.load()
    rng = np.random.default_rng(n)
    src = rng.standard_normal(n)
    d = ctypes.c_void_p()
    assert lib.stg_device_alloc(n, ctypes.byref(d)) == 0
    try:
        assert lib.stg_memcpy(d, src.ctypes.data, n, 0) == 0
        back = np.zeros(n)
        assert lib.stg_memcpy(back.ctypes.data, d, n, 1) == 0
        assert np.array_equal(back, src)
        # against torch's own copy of the same device memory
        p = ctypes.c_void_p()
        assert lib.stg_host_alloc(n, ctypes.byref(p)) == 0
        try:
            pin = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)), (n,))
            pin[:] = 0.0
            assert lib.stg_memcpy(p, d, n, 1) == 0
            assert np.array_equal(pin, src)
            pin[:] = src[::-1]
            assert lib.stg_memcpy(d, p, n, 0) == 0
            assert lib.stg_memcpy(back.ctypes.data, d, n, 1) == 0
            assert np.array_equal(back, src[::-1])
        finally:
            assert lib.stg_host_free(p) == 0
    finally:
        assert lib.stg_device_free(d) == 0


# ---- solvers ---------------------------------------------------------------------
def test_c1_slab_solve_vs_oracle():
    cfg = C.CONFIGS["c1"]
    op, pr = pair(cfg)
    un = C.initial_state(cfg)
    Uo, uo, _, _ = pr.stdg_step(0.0, cfg.dt, un, linear=O.DENSE_LU)
    cfgn = NewtonConfig(abs_tol=1e-14, rel_tol=1e-13, gmres_tol=1e-13)
    U, un1, info = op.stdg_step(0.0, cfg.dt, dev(un), cfgn)
    assert rel(U, Uo) <= TOL_SOLVE
    assert rel(un1, uo) <= TOL_SOLVE
    assert info.newton_iterations >= 1 and info.linear_iterations > 0
    assert np.allclose(U[-cfg.n_sdof:].cpu().numpy(), un1.cpu().numpy(), rtol=0, atol=0)


def test_gmres_matches_oracle_gmres_small_3d():
    cfg = C.CONFIGS["c4"].scaled((8, 8, 8))
    op, pr = pair(cfg)
    un = C.initial_state(cfg)
    cfgn = dict(abs_tol=0.0, rel_tol=1e-12, gmres_tol=1e-13)
    Uo, uo, _, lino = pr.stdg_step(0.0, cfg.dt, un, linear=O.GMRES, **cfgn)
    U, un1, info = op.stdg_step(0.0, cfg.dt, dev(un), NewtonConfig(**cfgn))
    assert rel(U, Uo) <= TOL_SOLVE


@pytest.mark.parametrize("form", [L.STG_FORM_A, L.STG_FORM_A_INV])
def test_rk_step_vs_oracle_and_equivalence(form):
    # test_stdg.cpp:111-135 on the device: STDG slab == LoDG stages
    cfg = make(1, 2, 3, (8,), (1.0,), dt=0.05)
    op, pr = pair(cfg)
    u0 = np.sin(2 * np.pi * C.node_coords(cfg)[:, 0]) + 0.3
    tight = NewtonConfig(abs_tol=1e-14, rel_tol=1e-13, gmres_tol=1e-14)
    Ua, ua, _ = op.stdg_step(0.0, cfg.dt, dev(u0), tight)
    Ub, ub, info = op.rk_step(form, 0.0, cfg.dt, dev(u0), tight)
    assert rel(ua, ub.cpu().numpy()) <= 1e-10
    assert rel(Ua, Ub.cpu().numpy()) <= 1e-9
    Uo, uo, _, _ = pr.rk_step(3, form, 0.0, cfg.dt, u0, linear=O.DENSE_LU)
    assert rel(ub, uo) <= TOL_SOLVE


def test_lodg_stages_match_stdg_slab_small_c5():
    # c5 physics on a small mesh: stage solution == slab solution to 1e-10
    cfg = C.CONFIGS["c5"].scaled((8, 8, 8))
    op = SlabOperator(**cfg.kwargs())
    un = dev(C.initial_state(cfg))
    tight = NewtonConfig(abs_tol=0.0, rel_tol=1e-13, gmres_tol=1e-14)
    Ua, ua, _ = op.stdg_step(0.0, cfg.dt, un, tight)
    Ub, ub, _ = op.rk_step(L.STG_FORM_A_INV, 0.0, cfg.dt, un, tight)
    assert rel(Ub, Ua.cpu().numpy()) <= TOL_SOLVE
    assert rel(ub, ua.cpu().numpy()) <= TOL_SOLVE


def test_burgers_newton_vs_oracle():
    cfg = C.CONFIGS["c3"].scaled((64,))
    op, pr = pair(cfg)
    un = C.initial_state(cfg)
    Uo, uo, ito, _ = pr.stdg_step(0.0, 1e-3, un, linear=O.DENSE_LU, abs_tol=1e-13, rel_tol=1e-13)
    U, un1, info = op.stdg_step(0.0, 1e-3, dev(un),
                                NewtonConfig(abs_tol=1e-13, rel_tol=1e-13, gmres_tol=1e-14))
    assert info.newton_iterations >= 2  # nonlinear
    assert rel(U, Uo) <= TOL_SOLVE


@pytest.mark.parametrize("name,cells,pcs", [
    ("c4", (8, 8, 8), [L.STG_PRECOND_NONE, L.STG_PRECOND_TBLOCK, L.STG_PRECOND_EBLOCK]),
    ("c2", (16, 16), [L.STG_PRECOND_NONE, L.STG_PRECOND_TBLOCK, L.STG_PRECOND_EBLOCK]),
    ("c1", (64,), [L.STG_PRECOND_NONE, L.STG_PRECOND_EBLOCK]),
    ("c3", (256,), [L.STG_PRECOND_NONE, L.STG_PRECOND_EBLOCK, L.STG_PRECOND_SWEEP]),
])
def test_preconditioners_same_solution_fewer_iterations(name, cells, pcs):
    cfg = C.CONFIGS[name].scaled(cells)
    op = SlabOperator(**cfg.kwargs())
    un = dev(C.initial_state(cfg))
    dt = cfg.dt if name != "c3" else 1e-3
    sols, its = [], []
    for pc in pcs:
        nc = NewtonConfig(abs_tol=1e-13, rel_tol=1e-12, gmres_tol=1e-13, precond=pc,
                          gmres_max_it=5000)
        U, u1, info = op.stdg_step(0.0, dt, un, nc)
        sols.append(U.cpu().numpy())
        its.append(info.linear_iterations)
    for i in range(1, len(pcs)):
        assert rel(sols[i], sols[0]) <= TOL_SOLVE
        assert its[i] < its[i - 1], its


@pytest.mark.parametrize("velocity", [(1.0, 1.0, 1.0), (-0.7, 0.4, -1.1)])
@pytest.mark.parametrize("cells", [(2, 2, 2), (4, 2, 2), (2, 2, 8)])
def test_fdm_element_block_is_exact_local_inverse(velocity, cells):
    """d = 3 EBLOCK (fast diagonalisation, kernels_fdm.cu) = the exact inverse
    of the element-local Jacobian block, which is read off the oracle's J.v
    (columns supported on one element; periodic meshes of 8 cells: the
    two-half kernel, and 16 / 32 cells: fdm3_kernel with the direct temporal
    solve)."""
    cfg = make(3, 3, 4, cells, velocity, dt=0.02)
    op, pr = pair(cfg)
    ns, npc, nt = op.n_sdof, 64, 4
    loc = np.array([t * ns + k for t in range(nt) for k in range(npc)])  # element 0
    Lblk = np.zeros((nt * npc, nt * npc))
    U0 = np.zeros(nt * ns)
    for c, i in enumerate(loc):
        e = np.zeros(nt * ns)
        e[i] = 1.0
        Lblk[:, c] = pr.st_jvp(0.0, cfg.dt, U0, e)[loc]
    x = np.random.default_rng(5).standard_normal(nt * ns)
    y = op.st_precond_apply(cfg.dt, dev(x), precond=L.STG_PRECOND_EBLOCK).cpu().numpy()
    for cell in range(int(np.prod(cells))):
        idx = loc + cell * npc
        ref = np.linalg.solve(Lblk, x[idx])
        assert rel(y[idx], ref) <= 1e-11, cell


@pytest.mark.parametrize("dim,cells,velocity,degree", [
    (3, (2, 2, 4), (1.0, 1.0, 1.0), 3),      # fdm3 with the couplings folded in
    (3, (4, 2, 2), (-0.7, 0.4, -1.1), 3),    # ... upwind on both sides
    (3, (8, 4, 2), (0.3, -1.2, 0.8), 3),     # ... 64 cells: several segments per row
    (3, (2, 2, 2), (-0.7, 0.4, -1.1), 3),    # fdm (two-half) blocks, upwind on both sides
    (2, (8, 4), (1.0, 0.5), 4),              # fdm2i blocks + k_offdiag<2,5,5>
    (2, (4, 4), (-0.6, 1.1), 3),             # fdm2 blocks + k_offdiag<2,4,4>
])
def test_poly_precond_is_the_neumann_series(dim, cells, velocity, degree):
    """STG_PRECOND_POLY (the AUTO choice for d >= 2 advection) applies
    sum_{i=0..m} (I - P0^-1 J)^i P0^-1 with P0 the exact element blocks and m
    its terms (STG_POLY_TERMS, default 7): checked against the series formed
    in numpy from the oracle's J.v and
    dense block solves.  d = 3 meshes of 16k cells run the fused fdm3 +
    neighbour-coupling kernel, the others k_offdiag + the block apply."""
    cfg = make(dim, degree, degree + 1, cells, velocity, dt=0.02)
    op, pr = pair(cfg)
    ns, nt = op.n_sdof, degree + 1
    npc = (degree + 1) ** dim
    loc = np.array([t * ns + k for t in range(nt) for k in range(npc)])
    U0 = np.zeros(nt * ns)
    Lblk = np.zeros((nt * npc, nt * npc))
    for c, i in enumerate(loc):
        e = np.zeros(nt * ns)
        e[i] = 1.0
        Lblk[:, c] = pr.st_jvp(0.0, cfg.dt, U0, e)[loc]
    Li = np.linalg.inv(Lblk)

    def p0(v):
        out = np.empty_like(v)
        for cell in range(int(np.prod(cells))):
            idx = loc + cell * npc
            out[idx] = Li @ v[idx]
        return out

    x = np.random.default_rng(5).standard_normal(nt * ns)
    z = p0(x)
    y = z.copy()
    for _ in range(int(os.environ.get("STG_POLY_TERMS", "7"))):
        y = z + y - p0(pr.st_jvp(0.0, cfg.dt, U0, y))
    got = op.st_precond_apply(cfg.dt, dev(x), precond=L.STG_PRECOND_POLY).cpu().numpy()
    assert rel(got, y) <= 1e-11
    ya = op.st_precond_apply(cfg.dt, dev(x)).cpu().numpy()  # AUTO picks it
    assert np.array_equal(ya, got)


def test_fdm_eblock_stage_solves():
    cfg = C.CONFIGS["c5"].scaled((8, 8, 8))
    op = SlabOperator(**cfg.kwargs())
    un = dev(C.initial_state(cfg))
    for form in (L.STG_FORM_A, L.STG_FORM_A_INV):
        res = []
        for pc in (L.STG_PRECOND_TBLOCK, L.STG_PRECOND_EBLOCK):
            # a linear stage system: one Newton step at a realistic GMRES tolerance
            nc = NewtonConfig(abs_tol=0.0, rel_tol=1e-11, gmres_tol=1e-12, precond=pc)
            U, _, info = op.rk_step(form, 0.0, cfg.dt, un, nc)
            res.append((U.cpu().numpy(), info.linear_iterations, info.newton_iterations))
        assert rel(res[1][0], res[0][0]) <= TOL_SOLVE
        assert res[1][2] == res[0][2] == 1
        assert res[1][1] < res[0][1], (form, res[0][1], res[1][1])


def test_preconditioned_stage_solve_matches_slab():
    cfg = C.CONFIGS["c5"].scaled((8, 8, 8))
    op = SlabOperator(**cfg.kwargs())
    un = dev(C.initial_state(cfg))
    tight = NewtonConfig(abs_tol=0.0, rel_tol=1e-13, gmres_tol=1e-14,
                         precond=L.STG_PRECOND_TBLOCK)
    Ua, _, _ = op.stdg_step(0.0, cfg.dt, un, tight)
    for form in (L.STG_FORM_A, L.STG_FORM_A_INV):
        Ub, _, _ = op.rk_step(form, 0.0, cfg.dt, un, tight)
        assert rel(Ub, Ua.cpu().numpy()) <= TOL_SOLVE


def test_burgers_fd_jvp_close_to_exact():
    cfg = C.CONFIGS["c3"].scaled((64,))
    op = SlabOperator(**cfg.kwargs())
    U = dev(1.0 + 0.3 * C.random_slab(cfg))
    v = dev(np.random.default_rng(1).uniform(-1, 1, cfg.n_dof))
    ex = op.st_jvp(0.0, 1e-3, U, v)
    fd = op.st_jvp(0.0, 1e-3, U, v, fd_eps=1e-7)
    assert rel(fd, ex.cpu().numpy()) <= 1e-6


def test_nonconvergence_and_bad_input_errors():
    cfg = C.CONFIGS["c1"]
    op = SlabOperator(**cfg.kwargs())
    un = dev(C.initial_state(cfg))
    with pytest.raises(NonconvergenceError, match="stdg_step element at t=0") as ei:
        op.stdg_step(0.0, cfg.dt, un, NewtonConfig(max_iter=0))
    assert len(ei.value.residual_history) == 1  # newton.hpp:40-48 carries the history
    with pytest.raises(ValueError):
        op.stdg_step(0.0, -1.0, un)
    with pytest.raises(ValueError):
        op.st_residual(0.0, cfg.dt, un, dev(np.zeros(cfg.n_dof - 1)))
    with pytest.raises(ValueError):
        SlabOperator(3, 3, 4, (8, 8, 8), (0, 0, 0), (1, 1, 1), (1, 1, 1),
                     kernel=L.STG_KERNEL_FAST).stage_residual  # ok to construct
        SlabOperator(3, 3, 3, (6, 6, 6), (0, 0, 0), (1, 1, 1), (1, 1, 1),
                     kernel=L.STG_KERNEL_FAST).st_residual(
            0.0, 0.01, dev(np.zeros(6 ** 3 * 64)), dev(np.zeros(3 * 6 ** 3 * 64)))


def test_launch_counter_counts_native_kernels():
    cfg = C.CONFIGS["c4"].scaled((8, 8, 8))
    op = SlabOperator(**cfg.kwargs())
    n0 = op.kernel_launches()
    op.st_residual(0.0, cfg.dt, dev(C.initial_state(cfg)), dev(C.random_slab(cfg)))
    assert op.kernel_launches() == n0 + 1


@pytest.mark.parametrize("cells,degree,n_tau,vel", [((64,), 3, 4, (1.0,)), ((16,), 2, 3, (-0.8,)),
                                                    ((40,), 4, 5, (1.3,))])
def test_fused_small_solve_matches_host_driven(cells, degree, n_tau, vel):
    """kernels_small.cu (one-CTA Newton-GMRES, AUTO) == the host-driven solver
    (STG_KERNEL_GENERIC) for slab and stage solves, both preconditioners."""
    cfg = make(1, degree, n_tau, cells, vel, dt=0.005)
    fused = SlabOperator(**cfg.kwargs())
    host = SlabOperator(**cfg.kwargs(), kernel=L.STG_KERNEL_GENERIC)
    pr = O.Problem(1, degree, list(cells), [0.0], [1.0], list(vel), n_tau=n_tau)
    un = C.initial_state(cfg)
    for pc in (L.STG_PRECOND_AUTO, L.STG_PRECOND_NONE):
        nc = NewtonConfig(abs_tol=0.0, rel_tol=1e-11, gmres_tol=1e-12, precond=pc)
        Uf, uf, inf_f = fused.stdg_step(0.0, cfg.dt, dev(un), nc)
        Uh, uh, inf_h = host.stdg_step(0.0, cfg.dt, dev(un), nc)
        assert rel(Uf, Uh.cpu().numpy()) <= TOL_SOLVE
        assert rel(uf, uh.cpu().numpy()) <= TOL_SOLVE
        assert inf_f.newton_iterations == inf_h.newton_iterations
        assert abs(inf_f.linear_iterations - inf_h.linear_iterations) <= 1
        Uo, _, _, _ = pr.stdg_step(0.0, cfg.dt, un, linear=O.DENSE_LU if pr.dof * n_tau < 600
                                   else O.GMRES, abs_tol=0.0, rel_tol=1e-11, gmres_tol=1e-13)
        assert rel(Uf, Uo) <= TOL_SOLVE
        if n_tau in (2, 3, 4):
            for form in (L.STG_FORM_A, L.STG_FORM_A_INV):
                Uf, uf, _ = fused.rk_step(form, 0.0, cfg.dt, dev(un), nc)
                Uh, uh, _ = host.rk_step(form, 0.0, cfg.dt, dev(un), nc)
                assert rel(Uf, Uh.cpu().numpy()) <= TOL_SOLVE
                assert rel(uf, uh.cpu().numpy()) <= TOL_SOLVE


def test_fused_small_solve_errors_match():
    cfg = C.CONFIGS["c1"]
    op = SlabOperator(**cfg.kwargs())
    un = dev(C.initial_state(cfg))
    with pytest.raises(NonconvergenceError) as e:
        op.stdg_step(0.5, cfg.dt, un, NewtonConfig(max_iter=0))
    assert "stdg_step element at t=0.5" in str(e.value)
    assert len(e.value.residual_history) == 1
    with pytest.raises(RuntimeError, match="GMRES did not converge"):
        op.stdg_step(0.0, cfg.dt, un, NewtonConfig(gmres_max_it=1, gmres_tol=1e-14,
                                                   precond=L.STG_PRECOND_NONE))


@pytest.mark.parametrize("model,n_tau,degree", [(L.STG_MODEL_ADVECTION, 4, 3),
                                                (L.STG_MODEL_BURGERS, 4, 3),
                                                (L.STG_MODEL_BURGERS, 3, 2),
                                                (L.STG_MODEL_ADVECTION, 5, 1)])
def test_large_1d_lane_kernel_parity(model, n_tau, degree):
    """slab1d_lane_kernel (d = 1, >= 4096 elements): R(U), J.v (exact and FD
    paths), stage residuals vs the oracle."""
    cfg = make(1, degree, n_tau, (5003,), (0.9,), model=model, dt=1e-3)
    op, pr = pair(cfg)
    rng = np.random.default_rng(11)
    un = C.initial_state(cfg)
    U = np.concatenate([un + 0.05 * rng.uniform(-1, 1, un.size) for _ in range(n_tau)])
    v = rng.uniform(-1, 1, U.size)
    assert rel(op.st_residual(0.0, cfg.dt, dev(un), dev(U)), pr.st_residual(0.0, cfg.dt, un, U)) <= TOL_OP
    assert rel(op.st_jvp(0.0, cfg.dt, dev(U), dev(v)), pr.st_jvp(0.0, cfg.dt, U, v)) <= TOL_OP
    if n_tau in (2, 3, 4):
        for form in (L.STG_FORM_A, L.STG_FORM_A_INV):
            got = op.stage_residual(form, 0.0, cfg.dt, dev(un), dev(U))
            assert rel(got, pr.stage_residual(n_tau, form, 0.0, cfg.dt, un, U)) <= TOL_OP


def test_full_c3_residual_parity():
    cfg = C.CONFIGS["c3"]
    op, pr = pair(cfg)
    un = C.initial_state(cfg)
    U = np.concatenate([un] * cfg.n_tau) + 0.01 * np.random.default_rng(2).uniform(-1, 1, cfg.n_dof)
    assert rel(op.st_residual(0.0, cfg.dt, dev(un), dev(U)), pr.st_residual(0.0, cfg.dt, un, U)) <= TOL_OP


@pytest.mark.parametrize("cells,velocity,degree", [
    ((4, 3), (1.0, -0.5), 4),      # 12 cells: the dense block (kernels_precond.cu)
    ((8, 4), (1.0, -0.5), 4),      # 32 cells: fdm2i_kernel <5, 5, 1, 2> (in place)
    ((16, 4), (-0.8, 0.3), 4),
    ((8, 8), (1.0, 0.5), 4),
    ((8, 4), (0.0, 0.7), 4),       # b_x = 0: V_x has no FDM form -> dense block
    ((8, 4), (0.6, -1.1), 3),      # n = 4, n_tau = 4: fdm2_kernel <4, 4, 0, 2>
    ((16, 2), (1.0, 1.0), 2),      # n = 3, n_tau = 3: fdm2i_kernel <3, 3, 1, 1>
])
@pytest.mark.parametrize("variant", ["default", "STG_NO_FDM2I"])
def test_2d_element_block_is_exact_local_inverse(cells, velocity, degree, variant, monkeypatch):
    """d = 2 EBLOCK (fast diagonalisation, kernels_fdm.cu fdm2_kernel, or the
    shared dense block) = the exact inverse of the element-local block read
    off the oracle's J.v.  STG_NO_FDM2I selects the tiled fdm2_kernel (read
    at each preconditioner build)."""
    if variant != "default":
        monkeypatch.setenv(variant, "1")
    cfg = make(2, degree, degree + 1, cells, velocity, dt=0.003)
    op, pr = pair(cfg)
    ns, npc, nt = op.n_sdof, (degree + 1) ** 2, degree + 1
    loc = np.array([t * ns + k for t in range(nt) for k in range(npc)])  # element 0
    Lblk = np.zeros((nt * npc, nt * npc))
    U0 = np.zeros(nt * ns)
    for c, i in enumerate(loc):
        e = np.zeros(nt * ns)
        e[i] = 1.0
        Lblk[:, c] = pr.st_jvp(0.0, cfg.dt, U0, e)[loc]
    x = np.random.default_rng(9).standard_normal(nt * ns)
    y = op.st_precond_apply(cfg.dt, dev(x), precond=L.STG_PRECOND_EBLOCK).cpu().numpy()
    for cell in range(int(np.prod(cells))):
        idx = loc + cell * npc
        assert rel(y[idx], np.linalg.solve(Lblk, x[idx])) <= 1e-11, cell


def test_fused_fd_jvp_matches_host_driven_and_exact():
    """d = 1 Burgers, >= 4096 elements: the fused central difference (one lane
    kernel, <v,v> on the device) agrees with the host-driven difference and
    with the exact linearisation to FD accuracy; slab and both stage forms."""
    cfg = make(1, 3, 4, (5003,), (0.0,), model=L.STG_MODEL_BURGERS, dt=1e-4)
    fused = SlabOperator(**cfg.kwargs())
    host = SlabOperator(**cfg.kwargs(), kernel=L.STG_KERNEL_GENERIC)
    rng = np.random.default_rng(4)
    un = C.initial_state(cfg)
    U = dev(np.concatenate([un + 0.05 * rng.uniform(-1, 1, un.size) for _ in range(4)]))
    v = dev(rng.uniform(-1, 1, cfg.n_dof))
    a = fused.st_jvp(0.0, cfg.dt, U, v, fd_eps=1e-7).cpu().numpy()
    b = host.st_jvp(0.0, cfg.dt, U, v, fd_eps=1e-7).cpu().numpy()
    ex = fused.st_jvp(0.0, cfg.dt, U, v).cpu().numpy()  # exact linearisation
    assert rel(a, b) <= 1e-7
    assert rel(a, ex) <= 1e-6
    for form in (L.STG_FORM_A, L.STG_FORM_A_INV):
        a = fused.stage_jvp(form, 0.0, cfg.dt, U, v, fd_eps=1e-7).cpu().numpy()
        ex = fused.stage_jvp(form, 0.0, cfg.dt, U, v).cpu().numpy()
        assert rel(a, ex) <= 1e-6


def test_c3_fused_solve_matches_host_driven():
    cfg = C.CONFIGS["c3"]
    fused = SlabOperator(**cfg.kwargs())
    host = SlabOperator(**cfg.kwargs(), kernel=L.STG_KERNEL_GENERIC)
    u = dev(C.initial_state(cfg))
    nc = NewtonConfig(abs_tol=1e-12, rel_tol=1e-10, gmres_tol=1e-6, fd_eps=1e-7)
    _, uf, inf_f = fused.stdg_step(0.0, cfg.dt, u, nc)
    _, uh, inf_h = host.stdg_step(0.0, cfg.dt, u, nc)
    # inexact Newton to ||R||_inf <= 1e-12: both land on the same solution
    assert rel(uf, uh.cpu().numpy()) <= 1e-9
    assert inf_f.newton_iterations == inf_h.newton_iterations


def _random_configs(n, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        d = int(rng.integers(1, 4))
        p = int(rng.integers(1, 5 if d < 3 else 5))
        nt = int(rng.integers(2, 7))
        if d == 1:
            cells = (int(rng.choice([1, 2, 3, 7, 16, 33, 64])),)
        elif d == 2:
            cells = tuple(int(x) for x in rng.choice([1, 2, 3, 4, 5, 8, 16, 32], 2))
        else:
            cells = tuple(int(x) for x in rng.choice([1, 2, 3, 4, 8], 3))
        vel = tuple(float(v) for v in rng.choice([-1.3, -0.4, 0.0, 0.6, 1.1], d))
        out.append(make(d, p, nt, cells, vel, dt=float(rng.uniform(1e-3, 5e-2))))
    return out


SWEEP = _random_configs(40)


@pytest.mark.parametrize("cfg", SWEEP, ids=[f"{c.dim}d-p{c.degree}-nt{c.n_tau}-{c.cells}"
                                            for c in SWEEP])
def test_random_sweep_parity(cfg):
    """Seeded sweep over (d, N, n_tau, mesh, velocity signs incl. 0): R(U),
    J.v and both stage residuals vs the oracle, with whatever kernel AUTO
    selects for the shape."""
    op, pr = pair(cfg)
    rng = np.random.default_rng(7)
    un = rng.uniform(-1, 1, cfg.n_sdof)
    U = rng.uniform(-1, 1, cfg.n_dof)
    v = rng.uniform(-1, 1, cfg.n_dof)
    assert rel(op.st_residual(0.0, cfg.dt, dev(un), dev(U)), pr.st_residual(0.0, cfg.dt, un, U)) <= TOL_OP
    assert rel(op.st_jvp(0.0, cfg.dt, None, dev(v)), pr.st_jvp(0.0, cfg.dt, U, v)) <= TOL_OP
    if cfg.n_tau in (2, 3, 4):
        for form in (L.STG_FORM_A, L.STG_FORM_A_INV):
            got = op.stage_residual(form, 0.0, cfg.dt, dev(un), dev(U))
            assert rel(got, pr.stage_residual(cfg.n_tau, form, 0.0, cfg.dt, un, U)) <= TOL_OP


@pytest.mark.parametrize("name", ["c1", "c4@8"])
def test_device_integrate_matches_step_loop(name):
    """stg_stdg_integrate / stg_rk_integrate (stdg.hpp:152-173, lodg.hpp:158-181)
    march on the device and reproduce a host loop of steps bit for bit."""
    cfg = C.CONFIGS["c1"] if name == "c1" else C.CONFIGS["c4"].scaled((8, 8, 8))
    op = SlabOperator(**cfg.kwargs())
    u0 = dev(C.initial_state(cfg))
    nc = NewtonConfig(abs_tol=0.0, rel_tol=1e-10, gmres_tol=1e-11)
    n, t0, t1 = 3, 0.1, 0.1 + 3 * cfg.dt
    uf, states, sols, info = op.stdg_integrate(t0, u0, t1, n, nc, keep_states=True,
                                               keep_solutions=True)
    u, tot = u0, 0
    for k in range(n):
        U, u, inf = op.stdg_step(t0 + (t1 - t0) * k / n, (t1 - t0) / n, u, nc)
        assert torch.equal(states[k + 1], u)
        assert torch.equal(sols[k], U)
        tot += inf.newton_iterations
    assert torch.equal(uf, u) and torch.equal(states[0], u0)
    assert info.newton_iterations == tot
    uf2, _, _, _ = op.rk_integrate(L.STG_FORM_A_INV, t0, u0, t1, n, nc)
    u = u0
    for k in range(n):
        _, u, _ = op.rk_step(L.STG_FORM_A_INV, t0 + (t1 - t0) * k / n, (t1 - t0) / n, u, nc)
    assert torch.equal(uf2, u)
    with pytest.raises(ValueError):
        op.stdg_integrate(0.0, u0, 1.0, 0, nc)


@pytest.mark.parametrize("form", [L.STG_FORM_A, L.STG_FORM_A_INV])
@pytest.mark.parametrize("name,cells", [("c5", (8, 8, 8)), ("c2", (16, 16))])
def test_poly_stage_solves_match_element_blocks(form, name, cells):
    """AUTO (the polynomial preconditioner; the A-form's full S takes the
    unfused neighbour-coupling kernel, the A^-1-form the fused block apply)
    and the element blocks alone give the same stage solution."""
    cfg = C.CONFIGS[name].scaled(cells)
    op = SlabOperator(**cfg.kwargs())
    u = dev(C.initial_state(cfg))
    sols, its = [], []
    for pc in (L.STG_PRECOND_EBLOCK, L.STG_PRECOND_AUTO):
        nc = NewtonConfig(abs_tol=0.0, rel_tol=1e-11, gmres_tol=1e-13, precond=pc)
        U, _, info = op.rk_step(form, 0.0, cfg.dt, u, nc)
        sols.append(U.cpu().numpy())
        its.append(info.linear_iterations)
    assert rel(sols[1], sols[0]) <= TOL_SOLVE
    assert its[1] < its[0], its
