"""GPU: the device-side GMRES driver (stg.cpp gmres; Eigen's GMRES branch,
newton.hpp:68-77, is what it replaces).

The driver keeps the Hessenberg column, the Givens rotations and the stopping
test on the device and enqueues Arnoldi step k+1 before it has read step k;
kernels of a step that is no longer needed return at entry (skip flag).  These
tests check the mechanisms one by one:
* restarted cycles (restart 3-5, every preconditioner) converge to the oracle's
  solution (flexible GMRES forms x from the preconditioned basis);
* the results are BITWISE identical with speculation off (STG_GMRES_SYNC=1)
  and with programmatic dependent launch off (STG_NO_PDL=1): neither changes
  any arithmetic;
* forcing the second Gram-Schmidt pass on every step
  (STG_GMRES_REORTH_TOL=0.5) gives the same converged solutions;
* the d = 2 solve with the fast-diagonalisation element block (fdm2_kernel,
  default) matches the one with the dense element block (STG_NO_FDM2=1) and
  the oracle.
The knobs are read once per process, so each variant is a subprocess
(tests/_gmres_runner.py).  The forced-second-pass run found a real bug: a
Jacobian action that reduces into the step's scratch (the unfused FD J.v)
clobbered the raw dots a re-orthogonalisation re-reads; such actions are now
never run speculatively and the scalar reductions use their own slot.
"""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from paper_2201_05800_b200 import configs as C

pytestmark = pytest.mark.gpu

RUNNER = Path(__file__).with_name("_gmres_runner.py")
TOL_SOLVE = 1e-10
KEYS = ["fdm30", "fdm3", "tblock4", "none30", "gmres_st", "c3", "c3f", "c2", "c2rk"]


def run(tmp_path_factory, **env):
    out = tmp_path_factory.mktemp("gmres") / "res.npz"
    e = dict(os.environ)
    e.update(env)
    subprocess.run([sys.executable, str(RUNNER), str(out)], env=e, check=True, timeout=600)
    return dict(np.load(out))


@pytest.fixture(scope="module")
def base(tmp_path_factory):
    return run(tmp_path_factory)


@pytest.fixture(scope="module")
def oracle_c4():
    cfg = C.CONFIGS["c4"].scaled((8, 8, 8))
    pr = O.Problem(cfg.dim, cfg.degree, list(cfg.cells), list(cfg.lower), list(cfg.upper),
                   list(cfg.velocity), n_tau=cfg.n_tau)
    Uo, _, _, _ = pr.stdg_step(0.0, cfg.dt, C.initial_state(cfg), linear=O.GMRES, abs_tol=0.0,
                               rel_tol=1e-12, gmres_tol=1e-13)
    return Uo


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


@pytest.mark.parametrize("name", ["fdm30", "fdm3", "tblock4", "none30"])
def test_restarted_and_preconditioned_solves_match_oracle(base, oracle_c4, name):
    assert rel(base[name], oracle_c4) <= TOL_SOLVE
    newton, linear = base[name + "_its"]
    assert newton == 1 and linear >= 1


def test_restart_costs_iterations_not_accuracy(base):
    # GMRES(3) needs at least as many Arnoldi steps as GMRES(30)
    assert base["fdm3_its"][1] >= base["fdm30_its"][1]
    assert base["tblock4_its"][1] > base["fdm30_its"][1]


def test_gmres_st_nonzero_guess_residual(base):
    # the ABI linear solve from a non-zero guess: residual check on the oracle
    cfg = C.CONFIGS["c4"].scaled((8, 8, 8))
    pr = O.Problem(cfg.dim, cfg.degree, list(cfg.cells), list(cfg.lower), list(cfg.upper),
                   list(cfg.velocity), n_tau=cfg.n_tau)
    rng = np.random.default_rng(5)
    b = rng.uniform(-1, 1, cfg.n_dof)
    x = base["gmres_st"]
    r = b - pr.st_jvp(0.0, cfg.dt, np.zeros(cfg.n_dof), x)
    assert np.linalg.norm(r) <= 1e-10 * np.linalg.norm(b)


@pytest.mark.parametrize("knob", ["STG_GMRES_SYNC", "STG_NO_PDL", "STG_GMRES_NO_PREDICT",
                                  "STG_NO_LAZY_GUESS", "STG_NEWTON_SYNC_FIRST"])
def test_speculation_and_pdl_change_no_arithmetic(base, tmp_path_factory, knob):
    other = run(tmp_path_factory, **{knob: "1"})
    for k in KEYS:
        assert np.array_equal(other[k], base[k]), f"{knob}: {k} differs"
        assert np.array_equal(other[k + "_its"], base[k + "_its"]), f"{knob}: {k} iterations"


def test_forced_reorthogonalisation_same_solutions(base, tmp_path_factory):
    other = run(tmp_path_factory, STG_GMRES_REORTH_TOL="0.5")
    for k in KEYS:
        assert rel(other[k], base[k]) <= TOL_SOLVE, k


@pytest.mark.parametrize("knob", ["STG_NO_FDM2", "STG_NO_FDM2I"])
def test_fdm2_solve_matches_dense_element_block(base, tmp_path_factory, knob):
    # d = 2: the element-block inverse by in-place fast diagonalisation
    # (fdm2i_kernel, default), by the tiled one (fdm2_kernel, STG_NO_FDM2I)
    # and by the dense block (k_eblock_dense, STG_NO_FDM2) are the same
    # operator, so the solves agree and take the same number of iterations
    other = run(tmp_path_factory, **{knob: "1"})
    for k in ["c2", "c2rk"]:
        assert rel(other[k], base[k]) <= TOL_SOLVE, k
    assert base["c2_its"][1] == other["c2_its"][1]


def test_c2_solve_matches_oracle(base):
    cfg = C.CONFIGS["c2"].scaled((32, 8))
    pr = O.Problem(cfg.dim, cfg.degree, list(cfg.cells), list(cfg.lower), list(cfg.upper),
                   list(cfg.velocity), n_tau=cfg.n_tau)
    Uo, _, _, _ = pr.stdg_step(0.0, cfg.dt, C.initial_state(cfg), linear=O.GMRES, abs_tol=0.0,
                               rel_tol=1e-12, gmres_tol=1e-13)
    assert rel(base["c2"], Uo) <= TOL_SOLVE
