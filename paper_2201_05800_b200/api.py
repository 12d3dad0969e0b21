"""Python mirror of the reference ``stdgsem`` interface for the slab hot path.

Same names, argument meaning and error behaviour as the reference C++ free
functions (file:line cited per function), backed by the CUDA library through
the C ABI (include/stg_cuda.h).  Vectors are CUDA float64 torch tensors in the
reference layout (stage-major blocks, cell x-fastest, node x-fastest); torch
is used only for device memory and streams.  There is no CPU fallback.

Exception mapping (status code -> reference exception type):
  STG_ERR_INVALID        -> ValueError            (std::invalid_argument)
  STG_ERR_RUNTIME        -> RuntimeError          (std::runtime_error)
  STG_ERR_NONCONVERGENCE -> NonconvergenceError   (newton.hpp:40-48)
  STG_ERR_CUDA           -> CudaError
  STG_ERR_ADMISSIBILITY  -> AdmissibilityError    (models.hpp:15-20)
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib as L

try:  # torch provides device memory and streams (plumbing only)
    import torch
except Exception:  # pragma: no cover
    torch = None


class NonconvergenceError(RuntimeError):
    """newton.hpp:40-48: carries the last Newton iterate and the residual
    history (rethrown with the slab / step context, stdg.hpp:132-137,
    lodg.hpp:132-137)."""

    def __init__(self, what: str, residual_history=(), last_iterate=None):
        super().__init__(what)
        self.residual_history = list(residual_history)
        self.last_iterate = last_iterate


class CudaError(RuntimeError):
    pass


class AdmissibilityError(RuntimeError):
    """A model was evaluated at a nonphysical state (models.hpp:15-20); the
    message names the temporal node (stdg.hpp:41-50)."""


class LinearMethod:  # newton.hpp:28
    auto_select = L.STG_LINEAR_AUTO
    gmres = L.STG_LINEAR_GMRES


class JacobianForm:  # lodg.hpp:20
    a_form = L.STG_FORM_A
    a_inv_form = L.STG_FORM_A_INV


@dataclass
class NewtonConfig:  # newton.hpp:30-38 (+ fd_eps for nonlinear J v)
    abs_tol: float = 1e-12
    rel_tol: float = 1e-12
    max_iter: int = 50
    linear: int = LinearMethod.auto_select
    gmres_restart: int = 30
    gmres_tol: float = 1e-12
    gmres_max_it: int = 1000
    fd_eps: float = 0.0
    precond: int = L.STG_PRECOND_AUTO  # right preconditioner, STG_PRECOND_* (stg_cuda.h)

    def to_c(self) -> L.StgNewtonConfig:
        return L.StgNewtonConfig(self.abs_tol, self.rel_tol, self.max_iter, self.linear,
                                 self.gmres_restart, self.gmres_tol, self.gmres_max_it, self.fd_eps,
                                 self.precond)


@dataclass
class SolveInfo:
    newton_iterations: int
    linear_iterations: int
    final_residual: float
    residual_history: list


def _raise(h, code: int, lib) -> None:
    if code == L.STG_OK:
        return
    msg = lib.stg_last_error(h).decode(errors="replace")
    if code == L.STG_ERR_INVALID:
        raise ValueError(msg)
    if code == L.STG_ERR_NONCONVERGENCE:
        raise NonconvergenceError(msg)
    if code == L.STG_ERR_CUDA:
        raise CudaError(msg)
    if code == L.STG_ERR_ADMISSIBILITY:
        raise AdmissibilityError(msg)
    raise RuntimeError(msg)


def _ptr(t, n: Optional[int] = None, what: str = "tensor") -> int:
    if torch is None or not isinstance(t, torch.Tensor):
        raise TypeError(f"{what}: expected a CUDA float64 torch tensor")
    if not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise ValueError(f"{what}: expected a contiguous CUDA float64 tensor")
    if n is not None and t.numel() != n:
        raise ValueError(f"{what}: expected {n} entries, got {t.numel()}")
    return t.data_ptr()


def _np(a, n: int, what: str) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.size != n:
        raise ValueError(f"{what}: expected {n} entries, got {a.size}")
    return a


def _out(a, n: int, what: str) -> np.ndarray:
    """A caller-owned host output buffer: written in place, so no copies."""
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous \
            or not a.flags.writeable:
        raise ValueError(f"{what}: expected a writable contiguous float64 array")
    if a.size != n:
        raise ValueError(f"{what}: expected {n} entries, got {a.size}")
    return a


class SlabOperator:
    """One problem handle: DG space + model + temporal operators (n_tau nodes).

    Wraps stg_create (assemble_semidiscrete spatial.hpp:352-385 together with
    sbp_operators operators.hpp:33-44 and lobatto_tableau operators.hpp:76-112).
    """

    def __init__(self, dim: int, degree: int, n_tau: int, cells: Sequence[int],
                 lower: Sequence[float], upper: Sequence[float],
                 velocity: Sequence[float] = (0.0, 0.0, 0.0), model: int = L.STG_MODEL_ADVECTION,
                 kernel: int = L.STG_KERNEL_AUTO, velocity_field: int = L.STG_FIELD_CONSTANT,
                 eps: float = 0.0, eta: float = 0.0, gamma: float = 0.0):
        self._lib = L.load()
        pad = lambda v, fill: list(v) + [fill] * (3 - len(v))
        d = L.StgDesc()
        d.dim, d.degree, d.n_tau, d.model = int(dim), int(degree), int(n_tau), int(model)
        d.cells[:] = [int(c) for c in pad(cells, 1)]
        d.lower[:] = [float(x) for x in pad(lower, 0.0)]
        d.upper[:] = [float(x) for x in pad(upper, 1.0)]
        d.velocity[:] = [float(x) for x in pad(velocity, 0.0)]
        d.velocity_field, d.eps, d.eta, d.gamma = int(velocity_field), float(eps), float(eta), \
            float(gamma)
        h = ctypes.c_void_p()
        _raise(None, self._lib.stg_create(ctypes.byref(d), ctypes.byref(h)), self._lib)
        self._h = h
        self.dim, self.degree, self.n_tau, self.model = d.dim, d.degree, d.n_tau, d.model
        ns, nd = ctypes.c_longlong(), ctypes.c_longlong()
        self._lib.stg_sizes(h, ctypes.byref(ns), ctypes.byref(nd))
        self.n_sdof, self.n_dof = ns.value, nd.value
        if kernel != L.STG_KERNEL_AUTO:
            self.set_kernel(kernel)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.stg_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- plumbing --
    def _call(self, fn, *args):
        if torch is not None and torch.cuda.is_available():
            self._lib.stg_set_stream(self._h, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        _raise(self._h, fn(self._h, *args), self._lib)

    def set_kernel(self, kernel: int):
        _raise(self._h, self._lib.stg_set_kernel(self._h, int(kernel)), self._lib)

    def kernel_launches(self) -> int:
        return int(self._lib.stg_kernel_launches(self._h))

    def constants(self):
        n1 = self.degree + 1
        x = np.zeros(n1)
        w = np.zeros(n1)
        Dt = np.zeros((self.n_tau, self.n_tau))
        self._lib.stg_constants(self._h, x.ctypes.data, w.ctypes.data, Dt.ctypes.data)
        return x, w, Dt

    def _new(self, n):
        return torch.empty(n, dtype=torch.float64, device="cuda")

    # -- operator applies (device tensors) --
    def spatial_rhs(self, u, t: float = 0.0, out=None):
        """SemiDiscreteSystem::rhs (system.hpp:21, spatial.hpp:107-266)."""
        out = self._new(self.n_sdof) if out is None else out
        self._call(self._lib.stg_spatial_rhs, float(t), _ptr(u, self.n_sdof, "u"),
                   _ptr(out, self.n_sdof, "F"))
        return out

    def spatial_jvp(self, u, v, t: float = 0.0, out=None):
        out = self._new(self.n_sdof) if out is None else out
        up = _ptr(u, self.n_sdof, "u") if u is not None else None
        self._call(self._lib.stg_spatial_jvp, float(t), up, _ptr(v, self.n_sdof, "v"),
                   _ptr(out, self.n_sdof, "Jv"))
        return out

    def st_residual(self, t_n: float, dt: float, u_n, U, out=None):
        """st_residual (stdg.hpp:56-76)."""
        out = self._new(self.n_dof) if out is None else out
        self._call(self._lib.stg_st_residual, float(t_n), float(dt), _ptr(u_n, self.n_sdof, "u_n"),
                   _ptr(U, self.n_dof, "U"), _ptr(out, self.n_dof, "R"))
        return out

    def st_jvp(self, t_n: float, dt: float, U, v, fd_eps: float = 0.0, out=None):
        """st_jacobian (stdg.hpp:79-110) applied to v, matrix-free."""
        out = self._new(self.n_dof) if out is None else out
        Up = _ptr(U, self.n_dof, "U") if U is not None else None
        self._call(self._lib.stg_st_jvp, float(t_n), float(dt), Up, _ptr(v, self.n_dof, "v"),
                   _ptr(out, self.n_dof, "Jv"), float(fd_eps))
        return out

    def stage_residual(self, form: int, t: float, dt: float, u, U, out=None):
        """rk_step residual (lodg.hpp:104-122)."""
        out = self._new(self.n_dof) if out is None else out
        self._call(self._lib.stg_stage_residual, int(form), float(t), float(dt),
                   _ptr(u, self.n_sdof, "u"), _ptr(U, self.n_dof, "U"), _ptr(out, self.n_dof, "R"))
        return out

    def stage_jvp(self, form: int, t: float, dt: float, U, v, fd_eps: float = 0.0, out=None):
        """stage_jacobian (lodg.hpp:43-85) applied to v, matrix-free."""
        out = self._new(self.n_dof) if out is None else out
        Up = _ptr(U, self.n_dof, "U") if U is not None else None
        self._call(self._lib.stg_stage_jvp, int(form), float(t), float(dt), Up,
                   _ptr(v, self.n_dof, "v"), _ptr(out, self.n_dof, "Jv"), float(fd_eps))
        return out

    def gmres_st(self, t_n: float, dt: float, U, b, x=None, restart: int = 30, tol: float = 1e-12,
                 max_it: int = 1000, precond: int = L.STG_PRECOND_AUTO):
        """linear_solve GMRES branch (newton.hpp:68-77) on the slab Jacobian."""
        x = torch.zeros(self.n_dof, dtype=torch.float64, device="cuda") if x is None else x
        it = ctypes.c_int(0)
        rr = ctypes.c_double(0.0)
        Up = _ptr(U, self.n_dof, "U") if U is not None else None
        self._call(self._lib.stg_gmres_st, float(t_n), float(dt), Up, _ptr(b, self.n_dof, "b"),
                   _ptr(x, self.n_dof, "x"), int(restart), float(tol), int(max_it), int(precond),
                   ctypes.byref(it), ctypes.byref(rr))
        return x, it.value, rr.value

    def st_precond_apply(self, dt: float, v, U=None, precond: int = L.STG_PRECOND_AUTO,
                         out=None):
        """out = P^-1 v for the block-Jacobi right preconditioner gmres_st uses."""
        out = self._new(self.n_dof) if out is None else out
        Up = _ptr(U, self.n_dof, "U") if U is not None else None
        self._call(self._lib.stg_st_precond_apply, float(dt), Up, int(precond),
                   _ptr(v, self.n_dof, "in"), _ptr(out, self.n_dof, "out"))
        return out

    def _step(self, fn, head, u, cfg, U, u_next, what):
        cfg = cfg or NewtonConfig()
        U = self._new(self.n_dof) if U is None else U
        u_next = self._new(self.n_sdof) if u_next is None else u_next
        info = L.StgSolveInfo()
        c = cfg.to_c()
        self._lib.stg_set_stream(self._h, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        code = fn(self._h, *head, _ptr(u, self.n_sdof, what), ctypes.byref(c),
                  _ptr(U, self.n_dof, "U"), _ptr(u_next, self.n_sdof, "u_next"), ctypes.byref(info))
        if code == L.STG_ERR_NONCONVERGENCE:  # U holds the last iterate
            raise NonconvergenceError(self._lib.stg_last_error(self._h).decode(),
                                      _info(info).residual_history, U)
        _raise(self._h, code, self._lib)
        return U, u_next, _info(info)

    def _integrate(self, fn, head, u0, t_end, n_steps, cfg, keep_states, keep_solutions):
        cfg = cfg or NewtonConfig()
        u_final = self._new(self.n_sdof)
        states = self._new((n_steps + 1) * self.n_sdof) if keep_states else None
        sols = self._new(n_steps * self.n_dof) if keep_solutions else None
        info = L.StgSolveInfo()
        c = cfg.to_c()
        self._lib.stg_set_stream(self._h, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        code = fn(self._h, *head, _ptr(u0, self.n_sdof, "u0"), float(t_end), int(n_steps),
                  ctypes.byref(c), _ptr(u_final, self.n_sdof, "u_final"),
                  None if states is None else states.data_ptr(),
                  None if sols is None else sols.data_ptr(), ctypes.byref(info))
        if code == L.STG_ERR_NONCONVERGENCE:  # the failing step's last iterate is in sols
            raise NonconvergenceError(self._lib.stg_last_error(self._h).decode(),
                                      _info(info).residual_history)
        _raise(self._h, code, self._lib)
        if states is not None:
            states = states.view(n_steps + 1, self.n_sdof)
        if sols is not None:
            sols = sols.view(n_steps, self.n_dof)
        return u_final, states, sols, _info(info)

    def stdg_integrate(self, t0: float, u0, t_end: float, n_steps: int,
                       cfg: Optional[NewtonConfig] = None, keep_states: bool = False,
                       keep_solutions: bool = False):
        """stdg_integrate (stdg.hpp:152-173), marched on the device: returns
        (u_final, states or None, slab solutions or None, SolveInfo totals)."""
        return self._integrate(self._lib.stg_stdg_integrate, (float(t0),), u0, t_end, n_steps,
                               cfg, keep_states, keep_solutions)

    def rk_integrate(self, form: int, t0: float, u0, t_end: float, n_steps: int,
                     cfg: Optional[NewtonConfig] = None, keep_states: bool = False,
                     keep_solutions: bool = False):
        """integrate (lodg.hpp:158-181), marched on the device."""
        return self._integrate(self._lib.stg_rk_integrate, (int(form), float(t0)), u0, t_end,
                               n_steps, cfg, keep_states, keep_solutions)

    def stdg_step(self, t_n: float, dt: float, u_n, cfg: Optional[NewtonConfig] = None, U=None,
                  u_next=None):
        """stdg_step (stdg.hpp:120-143): returns (U, u_next, SolveInfo)."""
        return self._step(self._lib.stg_stdg_step, (float(t_n), float(dt)), u_n, cfg, U, u_next,
                          "u_n")

    def rk_step(self, form: int, t: float, dt: float, u, cfg: Optional[NewtonConfig] = None,
                U=None, u_next=None):
        """rk_step (lodg.hpp:89-149): returns (stages U, u_next, SolveInfo)."""
        return self._step(self._lib.stg_rk_step, (int(form), float(t), float(dt)), u, cfg, U,
                          u_next, "u")

    # -- host-buffer variants (reference-facing e2e path) --
    def st_residual_host(self, t_n: float, dt: float, u_n, U, out=None) -> np.ndarray:
        u_n = _np(u_n, self.n_sdof, "u_n")
        U = _np(U, self.n_dof, "U")
        out = np.empty(self.n_dof) if out is None else out
        _raise(self._h, self._lib.stg_st_residual_host(self._h, float(t_n), float(dt),
                                                       u_n.ctypes.data, U.ctypes.data,
                                                       out.ctypes.data), self._lib)
        return out

    def _step_host(self, fn, head, u, cfg, U, u_next, what):
        u = _np(u, self.n_sdof, what)
        U = np.empty(self.n_dof) if U is None else _out(U, self.n_dof, "U")
        u_next = np.empty(self.n_sdof) if u_next is None else _out(u_next, self.n_sdof, "u_next")
        info = L.StgSolveInfo()
        c = (cfg or NewtonConfig()).to_c()
        code = fn(self._h, *head, u.ctypes.data, ctypes.byref(c), U.ctypes.data,
                  u_next.ctypes.data, ctypes.byref(info))
        if code == L.STG_ERR_NONCONVERGENCE:  # U holds the last iterate
            raise NonconvergenceError(self._lib.stg_last_error(self._h).decode(),
                                      _info(info).residual_history, U)
        _raise(self._h, code, self._lib)
        return U, u_next, _info(info)

    def stdg_step_host(self, t_n: float, dt: float, u_n, cfg: Optional[NewtonConfig] = None,
                       U=None, u_next=None):
        """stdg_step from host buffers (stg_stdg_step_host): H2D of u_n, the
        device solve, D2H of U and u_next, all inside the call.  U / u_next
        may be caller-owned (pinned or pageable) float64 arrays."""
        return self._step_host(self._lib.stg_stdg_step_host, (float(t_n), float(dt)), u_n, cfg,
                               U, u_next, "u_n")

    def rk_step_host(self, form: int, t: float, dt: float, u, cfg: Optional[NewtonConfig] = None,
                     U=None, u_next=None):
        """rk_step from host buffers (stg_rk_step_host)."""
        return self._step_host(self._lib.stg_rk_step_host, (int(form), float(t), float(dt)), u,
                               cfg, U, u_next, "u")


def _info(i: L.StgSolveInfo) -> SolveInfo:
    return SolveInfo(i.newton_iterations, i.linear_iterations, i.final_residual,
                     [i.residual_history[k] for k in range(i.n_history)])


# ---------------------------------------------------------------------------
# Reference-named free functions (stdgsem namespace)
# ---------------------------------------------------------------------------
@dataclass
class Mesh:  # mesh.hpp:14-35 (d = 3 is an extension)
    d: int
    lower: list
    upper: list
    cells: list


def uniform_mesh(d: int, lower, upper, cells) -> Mesh:  # mesh.hpp:37-55
    lower, upper, cells = list(lower), list(upper), list(cells)
    if d < 1 or d > 3:
        raise ValueError("uniform_mesh: d in {1,2,3}")
    if len(lower) != d or len(upper) != d or len(cells) != d:
        raise ValueError("uniform_mesh: inconsistent sizes")
    for a in range(d):
        if not upper[a] > lower[a]:
            raise ValueError("uniform_mesh: need upper > lower")
        if cells[a] < 1:
            raise ValueError("uniform_mesh: need cells >= 1")
    return Mesh(d, lower, upper, cells)


@dataclass
class DgSpace:  # mesh.hpp:59-91
    mesh: Mesh
    p: int
    r: int = 1

    def nodes_per_cell(self) -> int:
        return (self.p + 1) ** self.mesh.d

    def dof(self) -> int:
        return int(np.prod(self.mesh.cells)) * self.nodes_per_cell() * self.r


def dg_space(mesh: Mesh, p: int, r: int = 1) -> DgSpace:  # mesh.hpp:93-110
    if p < 1:
        raise ValueError("dg_space: the GPU path needs p >= 1")
    if r < 1:
        raise ValueError("dg_space: need r >= 1")
    return DgSpace(mesh, int(p), int(r))


@dataclass
class FluxModel:  # models.hpp:23-36 (constant-velocity advection, or Burgers)
    kind: int
    velocity: list = field(default_factory=list)
    linear: bool = True


def advection_model(b) -> FluxModel:  # models.hpp:60-66
    return FluxModel(L.STG_MODEL_ADVECTION, [float(x) for x in b], True)


def burgers_model() -> FluxModel:  # EXTENSION (not in the reference)
    return FluxModel(L.STG_MODEL_BURGERS, [0.0], False)


class SemiDiscreteSystem:
    """system.hpp:16-23: rhs(t, u) and a matrix-free jacobian(t, u)."""

    def __init__(self, space: DgSpace, model: FluxModel):
        self.space, self.model = space, model
        self.dof = space.dof()
        self._ops = {}

    def op(self, n_tau: int) -> SlabOperator:
        if n_tau not in self._ops:
            m = self.space.mesh
            self._ops[n_tau] = SlabOperator(m.d, self.space.p, n_tau, m.cells, m.lower, m.upper,
                                            self.model.velocity, self.model.kind)
        return self._ops[n_tau]

    def rhs(self, t: float, u):
        return self.op(2).spatial_rhs(u, t)

    def jacobian(self, t: float, u):
        o = self.op(2)
        return lambda v: o.spatial_jvp(u, v, t)


def assemble_semidiscrete(space: DgSpace, model: FluxModel) -> SemiDiscreteSystem:
    if space.r != 1:
        raise ValueError("assemble_semidiscrete: component mismatch (scalar models, r = 1)")
    if model.kind == L.STG_MODEL_ADVECTION and len(model.velocity) != space.mesh.d:
        raise ValueError("assemble_semidiscrete: dimension mismatch")
    if model.kind == L.STG_MODEL_BURGERS and space.mesh.d != 1:
        raise ValueError("assemble_semidiscrete: Burgers is 1-D only")
    return SemiDiscreteSystem(space, model)


@dataclass
class SbpOperators:  # operators.hpp:16-22
    n: int


def sbp_operators(n: int) -> SbpOperators:  # operators.hpp:33-44
    if n < 2:
        raise ValueError("sbp_operators: need n >= 2")
    return SbpOperators(int(n))


@dataclass
class ButcherTableau:  # operators.hpp:24-30
    s: int


def lobatto_tableau(s: int) -> ButcherTableau:  # operators.hpp:76-112
    if s not in (2, 3, 4):
        raise ValueError("lobatto_tableau: closed forms stored for s in {2,3,4}")
    return ButcherTableau(int(s))


@dataclass
class TimeElementSystem:  # stdg.hpp:21-29
    system: SemiDiscreteSystem
    ops: SbpOperators
    t_n: float
    dt: float
    u_n: object

    def n_tau(self) -> int:
        return self.ops.n


def st_residual(sys: TimeElementSystem, U):  # stdg.hpp:56-76
    op = sys.system.op(sys.ops.n)
    if U.numel() != op.n_dof:
        raise ValueError(f"st_residual: expected {op.n_dof} unknowns")
    return op.st_residual(sys.t_n, sys.dt, sys.u_n, U)


def st_jacobian(sys: TimeElementSystem, U, fd_eps: float = 0.0):  # stdg.hpp:79-110
    op = sys.system.op(sys.ops.n)
    if U.numel() != op.n_dof:
        raise ValueError(f"st_jacobian: expected {op.n_dof} unknowns")
    return lambda v: op.st_jvp(sys.t_n, sys.dt, U, v, fd_eps)


@dataclass
class StdgStepResult:  # stdg.hpp:112-116
    U: object
    u_next: object
    newton_iterations: int
    linear_iterations: int = 0


def stdg_step(system: SemiDiscreteSystem, ops: SbpOperators, t_n: float, u_n, dt: float,
              cfg: Optional[NewtonConfig] = None) -> StdgStepResult:  # stdg.hpp:120-143
    if not dt > 0:
        raise ValueError("stdg_step: dt > 0 required")
    U, un1, info = system.op(ops.n).stdg_step(t_n, dt, u_n, cfg)
    return StdgStepResult(U, un1, info.newton_iterations, info.linear_iterations)


@dataclass
class StdgTrajectory:  # stdg.hpp:145-150
    times: list
    states: list
    element_solutions: list
    total_newton_iterations: int = 0


def stdg_integrate(system, ops, t0, u0, t_end, n_steps, cfg=None) -> StdgTrajectory:
    """stdg_integrate (stdg.hpp:152-173): sequential slabs."""
    if n_steps < 1:
        raise ValueError("stdg_integrate: n_steps >= 1 required")
    times = [t0 + (t_end - t0) * k / n_steps for k in range(n_steps + 1)]
    # marched on the device (stg_stdg_integrate): no host round trip per slab
    _, states, sols, info = system.op(ops.n).stdg_integrate(t0, u0, t_end, n_steps, cfg,
                                                            keep_states=True, keep_solutions=True)
    return StdgTrajectory(times, [states[k] for k in range(n_steps + 1)],
                          [sols[k] for k in range(n_steps)], info.newton_iterations)


@dataclass
class RkStepResult:  # lodg.hpp:33-38
    u_next: object
    stages: object
    newton_iterations: int
    t_next: float
    linear_iterations: int = 0


def rk_step(system: SemiDiscreteSystem, tab: ButcherTableau, t: float, u, dt: float,
            cfg: Optional[NewtonConfig] = None, jac_form: int = JacobianForm.a_form) -> RkStepResult:
    """rk_step (lodg.hpp:89-149); stages returned stage-major in one tensor."""
    if not dt > 0:
        raise ValueError("rk_step: dt > 0 required")
    U, un1, info = system.op(tab.s).rk_step(jac_form, t, dt, u, cfg)
    return RkStepResult(un1, U, info.newton_iterations, t + dt, info.linear_iterations)


@dataclass
class RkTrajectory:  # lodg.hpp:151-156
    times: list
    states: list
    stage_solutions: list
    total_newton_iterations: int = 0


def integrate(system, tab, t0, u0, t_end, n_steps, cfg=None, jac_form=JacobianForm.a_form):
    """integrate (lodg.hpp:158-181)."""
    if n_steps < 1:
        raise ValueError("integrate: n_steps >= 1 required")
    times = [t0 + (t_end - t0) * k / n_steps for k in range(n_steps + 1)]
    # marched on the device (stg_rk_integrate)
    _, states, sols, info = system.op(tab.s).rk_integrate(jac_form, t0, u0, t_end, n_steps, cfg,
                                                          keep_states=True, keep_solutions=True)
    return RkTrajectory(times, [states[k] for k in range(n_steps + 1)],
                        [sols[k] for k in range(n_steps)], info.newton_iterations)


# ---------------------------------------------------------------------------
# Host-side field helpers (mesh.hpp:82-90, 113-181); layout as the library:
# cell x-fastest (d = 3 extended), node x-fastest, component innermost
# ---------------------------------------------------------------------------
@dataclass
class DiscreteField:  # mesh.hpp:113-117
    space: DgSpace
    coeffs: np.ndarray
    time_tag: float = 0.0


def node_coords(space: DgSpace) -> np.ndarray:
    """node_coord (mesh.hpp:82-90) of every (cell, node): (n_cells * n^d, 3),
    evaluated as lower + (c + 0.5 (1 + xi)) h in the reference's operation
    order (bitwise equal to it)."""
    from . import configs as C
    m = space.mesh
    return C.grid_coords(m.d, space.p, m.cells, m.lower, m.upper)


def interpolate(space: DgSpace, f, t: float = 0.0) -> DiscreteField:
    """interpolate (mesh.hpp:145-157): f(X) maps the (n_nodes, 3) coordinate
    array to (n_nodes,) or (n_nodes, r) values."""
    X = node_coords(space)
    val = np.asarray(f(X), dtype=np.float64).reshape(X.shape[0], -1)
    if val.shape[1] != space.r:
        raise ValueError(f"interpolate: f returned {val.shape[1]} components, space has r = {space.r}")
    return DiscreteField(space, np.ascontiguousarray(val.reshape(-1)), float(t))


def interpolate_scalar(space: DgSpace, f, t: float = 0.0) -> DiscreteField:
    """interpolate_scalar (mesh.hpp:159-165)."""
    return interpolate(space, lambda X: np.asarray(f(X), dtype=np.float64).reshape(-1, 1), t)


def global_mass(space: DgSpace) -> np.ndarray:
    """global_mass (mesh.hpp:125-141): cell volume / 2^d times the tensor LGL
    weights, replicated across the r components."""
    m = space.mesh
    n = space.p + 1
    lib = L.load()
    x, w = np.zeros(n), np.zeros(n)
    if lib.stg_lgl_rule(n, x.ctypes.data, w.ctypes.data) != 0:
        raise ValueError("lgl_rule failed")
    vol = 1.0
    for a in range(m.d):
        vol *= (m.upper[a] - m.lower[a]) / m.cells[a]
    vol_scale = vol / 2.0 ** m.d
    wn = w.copy()
    for _ in range(1, m.d):  # node x-fastest: w[ix] * w[iy] (* w[iz])
        wn = np.multiply.outer(w, wn).reshape(-1)
    cell = np.repeat(vol_scale * wn, space.r)
    return np.tile(cell, int(np.prod(m.cells)))


def l2_norm(field: DiscreteField) -> float:  # mesh.hpp:167-172
    return float(np.sqrt(np.dot(field.coeffs * field.coeffs, global_mass(field.space))))


def l2_error(field: DiscreteField, exact, t: float) -> float:  # mesh.hpp:174-181
    ref = interpolate(field.space, lambda X: exact(X, t), t)
    return l2_norm(DiscreteField(field.space, field.coeffs - ref.coeffs, t))
