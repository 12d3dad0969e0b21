"""CPU ORACLE -- test infrastructure only.

ctypes binding over ``oracle/build/liboracle.so`` (built from
``stdg_oracle.hpp``, a plain-C++ restatement of the reference ``stdgsem``
hot path).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline legs may import this package; the product
(``paper_2201_05800_b200``) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "liboracle.so"
NATIVE_PATH = HERE / "build" / "liboracle_native.so"

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)


def build(force: bool = False) -> Path:
    """Compile the oracle with its Makefile (system g++, -fopenmp)."""
    if force or not LIB_PATH.exists() or (
        LIB_PATH.stat().st_mtime
        < max((HERE / f).stat().st_mtime for f in ("stdg_oracle.hpp", "oracle_capi.cpp"))
    ):
        subprocess.run(["make", "-C", str(HERE), "-s"], check=True)
    return LIB_PATH


_LIB = None
_USE_NATIVE = False


def use_native() -> bool:
    """Switch to the -march=native build (the CPU-baseline legs of bench.py;
    BASELINE.md), compiled on this host.  Must run before the first lib()
    call; returns False (portable build kept) if the native build fails."""
    global _USE_NATIVE
    if _LIB is not None:
        return _USE_NATIVE
    try:
        subprocess.run(["make", "-B", "-C", str(HERE), "-s", "native"], check=True,
                       capture_output=True, timeout=600)
        _USE_NATIVE = NATIVE_PATH.exists()
    except Exception:
        _USE_NATIVE = False
    return _USE_NATIVE


def flags() -> str:
    return "-O3 -march=native" if _USE_NATIVE else "-O3 -march=x86-64-v3"


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is None:
        if not _USE_NATIVE:
            build()
        L = ctypes.CDLL(str(NATIVE_PATH if _USE_NATIVE else LIB_PATH))
        L.or_last_error.restype = ctypes.c_char_p
        L.or_dof.restype = ctypes.c_longlong
        L.or_dof.argtypes = [ctypes.c_void_p]
        L.or_destroy.argtypes = [ctypes.c_void_p]
        L.or_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _ip, _dp, _dp, _dp,
                                ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
        L.or_create_general.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _ip, _dp, _dp,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                        ctypes.POINTER(ctypes.c_void_p)]
        L.or_eta.restype = ctypes.c_double
        L.or_eta.argtypes = [ctypes.c_void_p]
        for name in ("or_spatial_rhs",):
            getattr(L, name).argtypes = [ctypes.c_void_p, ctypes.c_double, _dp, _dp]
        L.or_spatial_jvp.argtypes = [ctypes.c_void_p, ctypes.c_double, _dp, _dp, _dp]
        L.or_st_residual.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double, _dp, _dp, _dp]
        L.or_st_jvp.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double, _dp, _dp, _dp]
        L.or_stage_residual.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                        ctypes.c_double, _dp, _dp, _dp]
        L.or_stage_jvp.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                   ctypes.c_double, _dp, _dp, _dp]
        L.or_stdg_step.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double, _dp, _dp, _ip,
                                   _dp, _dp, _ip]
        L.or_rk_step.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                 ctypes.c_double, _dp, _dp, _ip, _dp, _dp, _ip]
        L.or_mass.argtypes = [ctypes.c_void_p, _dp]
        L.or_node_coords.argtypes = [ctypes.c_void_p, _dp]
        L.or_eval_interpolant.argtypes = [ctypes.c_int, _dp, ctypes.c_double, _dp]
        L.or_gmres_dense.argtypes = [ctypes.c_int, _dp, _dp, _dp, ctypes.c_int, ctypes.c_double,
                                     ctypes.c_int, _ip, _dp]
        L.or_lu_solve_dense.argtypes = [ctypes.c_int, _dp, _dp, _dp]
        L.or_sbp_defect.argtypes = [ctypes.c_int, _dp]
        _LIB = L
    return _LIB


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[oracle code {code}] {msg}")
        self.code = code


def _check(code: int) -> None:
    if code != 0:
        raise OracleError(code, lib().or_last_error().decode())


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def set_threads(n: int) -> int:
    return lib().or_set_threads(int(n))


def max_threads() -> int:
    return lib().or_max_threads()


# ---- 1-D numerics (quadrature.hpp / operators.hpp) -------------------------
def lgl(n: int):
    x = np.zeros(n)
    w = np.zeros(n)
    _check(lib().or_lgl(n, _p(x), _p(w)))
    return x, w


def barycentric(n: int):
    bw = np.zeros(n)
    _check(lib().or_barycentric(n, _p(bw)))
    return bw


def diff_matrix(n: int) -> np.ndarray:
    D = np.zeros((n, n))
    _check(lib().or_diff_matrix(n, _p(D)))
    return D


def eval_interpolant(n: int, coeffs, tau: float) -> float:
    out = np.zeros(1)
    _check(lib().or_eval_interpolant(n, _p(_f64(coeffs)), float(tau), _p(out)))
    return float(out[0])


def sbp_defect(n: int) -> float:
    out = np.zeros(1)
    _check(lib().or_sbp_defect(n, _p(out)))
    return float(out[0])


def lobatto(s: int):
    A = np.zeros((s, s))
    b = np.zeros(s)
    c = np.zeros(s)
    _check(lib().or_lobatto(s, _p(A), _p(b), _p(c)))
    return A, b, c


def to_butcher(n: int):
    A = np.zeros((n, n))
    b = np.zeros(n)
    c = np.zeros(n)
    _check(lib().or_to_butcher(n, _p(A), _p(b), _p(c)))
    return A, b, c


def gmres_dense(A, b, restart=30, tol=1e-12, max_it=1000):
    A = _f64(A)
    b = _f64(b)
    n = b.size
    x = np.zeros(n)
    it = ctypes.c_int(0)
    rr = ctypes.c_double(0)
    _check(lib().or_gmres_dense(n, _p(A), _p(b), _p(x), restart, tol, max_it,
                                ctypes.byref(it), ctypes.byref(rr)))
    return x, it.value, rr.value


def lu_solve_dense(A, b):
    A = _f64(A)
    b = _f64(b)
    x = np.zeros(b.size)
    _check(lib().or_lu_solve_dense(b.size, _p(A), _p(b), _p(x)))
    return x


# ---- problems ---------------------------------------------------------------
ADVECTION, BURGERS, TEST_EQUATION, ZERO_SYSTEM = 0, 1, 2, 3
ADVDIFF, EULER = 4, 5               # general flux models (models.hpp:40-159)
FIELD_CONSTANT, FIELD_ROTATING = 0, 1  # velocity b constant / rotating_field()
A_FORM, A_INV_FORM = 0, 1
AUTO, DENSE_LU, GMRES = 0, 1, 3


class Problem:
    """A DG space + model + temporal SBP operators (n_tau nodes)."""

    def __init__(self, d, p, cells, lower, upper, velocity=(0.0, 0.0, 0.0), model=ADVECTION,
                 n_tau=None, field=FIELD_CONSTANT, eps=0.0, eta=0.0, gamma=1.4):
        """model ADVECTION / BURGERS / TEST_EQUATION / ZERO_SYSTEM, or the general
        flux models ADVDIFF (advdiff_model: b constant or rotating_field, eps >= 0,
        interior penalty eta; eta <= 0 -> 10 p^2) and EULER (euler_model(gamma),
        r = 4 conservative components per node)."""
        self.d = int(d)
        self.p = int(p)
        self.n_tau = int(n_tau if n_tau is not None else p + 1)
        c = (ctypes.c_int * 3)(*(list(cells) + [1] * (3 - len(cells))))
        lo = _f64(list(lower) + [0.0] * (3 - len(lower)))
        hi = _f64(list(upper) + [1.0] * (3 - len(upper)))
        b = _f64(list(velocity) + [0.0] * (3 - len(velocity)))
        h = ctypes.c_void_p()
        self.r = 4 if model == EULER else 1
        if model in (ADVDIFF, EULER):
            _check(lib().or_create_general(self.d, self.p, self.n_tau, c, _p(lo), _p(hi),
                                           0 if model == ADVDIFF else 1, self.r, int(field),
                                           _p(b), float(eps), float(eta), float(gamma),
                                           ctypes.byref(h)))
        else:
            _check(lib().or_create(self.d, self.p, self.n_tau, c, _p(lo), _p(hi), _p(b),
                                   int(model), ctypes.byref(h)))
        self._h = h
        self.dof = int(lib().or_dof(h))
        self.model = model
        self.eta = float(lib().or_eta(h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib().or_destroy(h)
            self._h = None

    def mass(self):
        m = np.zeros(self.dof)
        _check(lib().or_mass(self._h, _p(m)))
        return m

    def coords(self):
        """Node coordinates, one row per (cell, node) (components share a node)."""
        x = np.zeros((self.dof // self.r, 3))
        _check(lib().or_node_coords(self._h, _p(x)))
        return x

    def rhs(self, u, t=0.0):
        u = _f64(u)
        F = np.zeros(self.dof)
        _check(lib().or_spatial_rhs(self._h, float(t), _p(u), _p(F)))
        return F

    def spatial_jvp(self, u, v, t=0.0):
        u, v = _f64(u), _f64(v)
        out = np.zeros(self.dof)
        _check(lib().or_spatial_jvp(self._h, float(t), _p(u), _p(v), _p(out)))
        return out

    def st_residual(self, t_n, dt, u_n, U):
        u_n, U = _f64(u_n), _f64(U)
        R = np.zeros(self.n_tau * self.dof)
        _check(lib().or_st_residual(self._h, float(t_n), float(dt), _p(u_n), _p(U), _p(R)))
        return R

    def st_jvp(self, t_n, dt, U, v):
        U, v = _f64(U), _f64(v)
        out = np.zeros(self.n_tau * self.dof)
        _check(lib().or_st_jvp(self._h, float(t_n), float(dt), _p(U), _p(v), _p(out)))
        return out

    def stage_residual(self, s, form, t, dt, u, U):
        u, U = _f64(u), _f64(U)
        R = np.zeros(s * self.dof)
        _check(lib().or_stage_residual(self._h, s, form, float(t), float(dt), _p(u), _p(U), _p(R)))
        return R

    def stage_jvp(self, s, form, t, dt, U, v):
        U, v = _f64(U), _f64(v)
        out = np.zeros(s * self.dof)
        _check(lib().or_stage_jvp(self._h, s, form, float(t), float(dt), _p(U), _p(v), _p(out)))
        return out

    @staticmethod
    def _cfg(abs_tol, rel_tol, gmres_tol, max_iter, linear, restart, gmres_max_it):
        d = _f64([abs_tol, rel_tol, gmres_tol])
        i = (ctypes.c_int * 4)(max_iter, linear, restart, gmres_max_it)
        return d, i

    def stdg_step(self, t_n, dt, u_n, abs_tol=1e-12, rel_tol=1e-12, max_iter=50, linear=AUTO,
                  restart=30, gmres_tol=1e-12, gmres_max_it=1000):
        u_n = _f64(u_n)
        d, i = self._cfg(abs_tol, rel_tol, gmres_tol, max_iter, linear, restart, gmres_max_it)
        U = np.zeros(self.n_tau * self.dof)
        un1 = np.zeros(self.dof)
        io = (ctypes.c_int * 2)()
        _check(lib().or_stdg_step(self._h, float(t_n), float(dt), _p(u_n), _p(d), i, _p(U),
                                  _p(un1), io))
        return U, un1, io[0], io[1]

    def rk_step(self, s, form, t, dt, u, abs_tol=1e-12, rel_tol=1e-12, max_iter=50, linear=AUTO,
                restart=30, gmres_tol=1e-12, gmres_max_it=1000):
        u = _f64(u)
        d, i = self._cfg(abs_tol, rel_tol, gmres_tol, max_iter, linear, restart, gmres_max_it)
        U = np.zeros(s * self.dof)
        un1 = np.zeros(self.dof)
        io = (ctypes.c_int * 2)()
        _check(lib().or_rk_step(self._h, s, form, float(t), float(dt), _p(u), _p(d), i, _p(U),
                                _p(un1), io))
        return U, un1, io[0], io[1]

    def interpolate(self, f):
        """Nodal interpolation (mesh.hpp:145-165): f maps (dof,3) coords -> values."""
        x = self.coords()
        return _f64(f(x[:, 0], x[:, 1], x[:, 2]))
