"""CPU checks of the C-ABI library: it builds, loads, exports every symbol the
header declares, validates descriptors before touching CUDA, refuses to run
without a device (no CPU fallback), and its host constants are bitwise equal
to the oracle's restatement of quadrature.hpp / operators.hpp."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from paper_2201_05800_b200 import _lib as L
from paper_2201_05800_b200 import build as B

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    B.build()
    return L.load()


def header_symbols():
    txt = (ROOT / "include" / "stg_cuda.h").read_text()
    return sorted(set(re.findall(r"\b(stg_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported(lib):
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/stg_cuda.h but not exported"
    assert sorted(L.EXPORTS) == syms


def test_invalid_descriptor_rejected_before_cuda(lib):
    d = L.StgDesc()
    d.dim, d.degree, d.n_tau, d.model = 4, 3, 4, 0  # d = 4 is invalid
    d.cells[:] = [4, 4, 4]
    d.lower[:] = [0, 0, 0]
    d.upper[:] = [1, 1, 1]
    h = ctypes.c_void_p()
    assert lib.stg_create(ctypes.byref(d), ctypes.byref(h)) == L.STG_ERR_INVALID
    assert b"d in" in lib.stg_last_error(None)
    d.dim = 2
    d.upper[:] = [1, 0, 1]  # upper <= lower on y
    assert lib.stg_create(ctypes.byref(d), ctypes.byref(h)) == L.STG_ERR_INVALID
    d.upper[:] = [1, 1, 1]
    d.model = 1  # Burgers is 1-D only
    assert lib.stg_create(ctypes.byref(d), ctypes.byref(h)) == L.STG_ERR_INVALID


@pytest.mark.parametrize("field,msg", [
    (dict(model=L.STG_MODEL_ADVDIFF, dim=3), b"d in {1, 2}"),
    (dict(model=L.STG_MODEL_ADVDIFF, eps=-1e-3), b"eps >= 0"),
    (dict(model=L.STG_MODEL_ADVDIFF, velocity_field=7), b"velocity field"),
    (dict(model=L.STG_MODEL_ADVDIFF, dim=1, velocity_field=L.STG_FIELD_ROTATING), b"d = 2"),
    (dict(model=L.STG_MODEL_EULER, dim=1), b"dimension mismatch"),
    (dict(model=L.STG_MODEL_EULER, gamma=0.9), b"gamma > 1"),
    (dict(model=9), b"unknown model"),
    (dict(cells=[1 << 15, 1 << 14, 1]), b"2^31"),
    (dict(cells=[1 << 16, 1 << 15, 1]), b"too many cells"),
])
def test_invalid_v2_descriptors(lib, field, msg):  # models.hpp:68-124, mesh.hpp:39
    """ABI v2 descriptor validation (general models, size guard) happens before
    any CUDA call, so it runs on CPU too."""
    d = L.StgDesc()
    d.dim, d.degree, d.n_tau, d.model = 2, 3, 4, L.STG_MODEL_ADVECTION
    d.cells[:] = [4, 4, 1]
    d.lower[:] = [0, 0, 0]
    d.upper[:] = [1, 1, 1]
    for k, v in field.items():
        if k == "cells":
            d.cells[:] = v
        else:
            setattr(d, k, v)
    h = ctypes.c_void_p()
    assert lib.stg_create(ctypes.byref(d), ctypes.byref(h)) == L.STG_ERR_INVALID
    assert msg in lib.stg_last_error(None), lib.stg_last_error(None)


def test_no_cpu_fallback_without_device(lib):
    from conftest import cuda_available
    if cuda_available():
        pytest.skip("device present")
    d = L.StgDesc()
    d.dim, d.degree, d.n_tau, d.model = 1, 3, 4, 0
    d.cells[:] = [8, 1, 1]
    d.lower[:] = [0, 0, 0]
    d.upper[:] = [1, 1, 1]
    d.velocity[:] = [1, 0, 0]
    h = ctypes.c_void_p()
    assert lib.stg_create(ctypes.byref(d), ctypes.byref(h)) == L.STG_ERR_CUDA


def test_host_alloc_argument_checks(lib):
    """stg_host_alloc / stg_host_free: n = 0 gives a null pointer, n < 0 is
    invalid, and without a device a real allocation fails with STG_ERR_CUDA
    (the C++ mirror's Vec then falls back to malloc)."""
    from conftest import cuda_available
    p = ctypes.c_void_p(1)
    assert lib.stg_host_alloc(0, ctypes.byref(p)) == L.STG_OK and not p.value
    assert lib.stg_host_alloc(-1, ctypes.byref(p)) == L.STG_ERR_INVALID
    assert lib.stg_host_free(None) == L.STG_OK
    code = lib.stg_host_alloc(1 << 10, ctypes.byref(p))
    if cuda_available():
        assert code == L.STG_OK and p.value
        assert lib.stg_host_free(p) == L.STG_OK
    else:
        assert code == L.STG_ERR_CUDA and not p.value


def test_newton_config_defaults(lib):  # newton.hpp:30-38
    c = L.StgNewtonConfig()
    lib.stg_newton_config_default(ctypes.byref(c))
    assert (c.abs_tol, c.rel_tol, c.max_iter, c.gmres_restart, c.gmres_tol, c.gmres_max_it) == (
        1e-12, 1e-12, 50, 30, 1e-12, 1000)


@pytest.mark.parametrize("n", range(2, 8))
def test_constants_bitwise_equal_to_oracle(lib, n):
    x = np.zeros(n)
    w = np.zeros(n)
    D = np.zeros((n, n))
    assert lib.stg_lgl_rule(n, x.ctypes.data, w.ctypes.data) == 0
    assert lib.stg_diff_matrix(n, D.ctypes.data) == 0
    xo, wo = O.lgl(n)
    assert np.array_equal(x, xo) and np.array_equal(w, wo)
    assert np.array_equal(D, O.diff_matrix(n))


@pytest.mark.parametrize("s", [2, 3, 4])
def test_tableau_bitwise_equal_to_oracle(lib, s):
    A = np.zeros((s, s))
    b = np.zeros(s)
    c = np.zeros(s)
    assert lib.stg_lobatto_tableau(s, A.ctypes.data, b.ctypes.data, c.ctypes.data) == 0
    Ao, bo, co = O.lobatto(s)
    assert np.array_equal(A, Ao) and np.array_equal(b, bo) and np.array_equal(c, co)


def test_tableau_beyond_closed_forms(lib):  # to_butcher path, operators.hpp:55-72
    s = 5
    A = np.zeros((s, s))
    b = np.zeros(s)
    c = np.zeros(s)
    assert lib.stg_lobatto_tableau(s, A.ctypes.data, b.ctypes.data, c.ctypes.data) == 0
    Ao, bo, co = O.to_butcher(s)
    assert np.abs(A - Ao).max() < 1e-13 and np.abs(b - bo).max() < 1e-15


def test_lgl_rejects_small_n(lib):  # test_quadrature.cpp:66-69
    x = np.zeros(2)
    assert lib.stg_lgl_rule(1, x.ctypes.data, x.ctypes.data) == L.STG_ERR_INVALID


def test_package_fails_loudly_without_library(monkeypatch, tmp_path):
    monkeypatch.setattr(L, "LIB_PATH", tmp_path / "missing.so")
    monkeypatch.setattr(L, "_LIB", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        L.load()
