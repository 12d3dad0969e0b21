"""The BASELINE.json workloads (c1..c5) and their synthetic inputs.

Inputs are generated on the host in the reference flat layout (mesh.hpp:70-81)
with numpy's PCG64 (``np.random.default_rng(seed)``): U ~ uniform[-1, 1) for
R(U) / J.v, and u_n = nodal interpolation of the config's u0 at the LGL nodes
(interpolate_scalar, mesh.hpp:145-165).  BASELINE.json gives only the seeds;
the generator is pinned here and documented in DESIGN.md.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib as L


@dataclass(frozen=True)
class Config:
    name: str
    dim: int
    degree: int
    n_tau: int
    cells: tuple
    lower: tuple
    upper: tuple
    velocity: tuple
    dt: float
    u0: str
    seed: int
    model: int = L.STG_MODEL_ADVECTION
    gmres_tol: float = 1e-10
    note: str = ""

    @property
    def n_cells(self) -> int:
        return int(np.prod(self.cells))

    @property
    def n_sdof(self) -> int:
        return self.n_cells * (self.degree + 1) ** self.dim

    @property
    def n_dof(self) -> int:
        return self.n_tau * self.n_sdof

    def scaled(self, cells) -> "Config":
        """Same physics on a smaller mesh (for oracle-sized parity cases)."""
        return replace(self, cells=tuple(cells), name=f"{self.name}@{'x'.join(map(str, cells))}")

    def kwargs(self) -> dict:
        return dict(dim=self.dim, degree=self.degree, n_tau=self.n_tau, cells=self.cells,
                    lower=self.lower, upper=self.upper, velocity=self.velocity, model=self.model)


TWO_PI = 2.0 * math.pi
CONFIGS = {
    "c1": Config("c1", 1, 3, 4, (64,), (0.0,), (1.0,), (1.0,), 0.005, "sin2pi_x", 0,
                 gmres_tol=1e-12, note="1-D advection, GMRES(30) slab to 1e-12, 1000 R(U)"),
    "c2": Config("c2", 2, 4, 5, (256, 256), (0.0, 0.0), (1.0, 1.0), (1.0, 0.5), 0.001,
                 "sin2pix_sin2piy", 1, note="2-D advection N=4: 8,192,000 DOF per slab"),
    "c3": Config("c3", 1, 3, 4, (65536,), (0.0,), (TWO_PI,), (0.0,), 1e-4, "burgers", 2,
                 model=L.STG_MODEL_BURGERS, note="1-D Burgers EC+LLF, Newton-GMRES, 10 slabs"),
    "c4": Config("c4", 3, 3, 4, (32, 32, 32), (0.0,) * 3, (1.0,) * 3, (1.0, 1.0, 1.0), 0.002,
                 "sin2pi_xyz", 3, note="3-D + t advection N=3 (the north-star target)"),
    "c5": Config("c5", 3, 3, 4, (32, 32, 32), (0.0,) * 3, (1.0,) * 3, (1.0, 1.0, 1.0), 0.002,
                 "sin2pi_xyz", 3, note="Lobatto IIIC s=4 stage system on the c4 mesh"),
}


def lgl_nodes(n: int) -> np.ndarray:
    lib = L.load()
    x = np.zeros(n)
    w = np.zeros(n)
    if lib.stg_lgl_rule(n, x.ctypes.data, w.ctypes.data) != 0:
        raise ValueError("lgl_rule failed")
    return x


def node_coords(cfg: Config) -> np.ndarray:
    """(n_sdof, 3) node coordinates, node_coord (mesh.hpp:82-90) order."""
    n = cfg.degree + 1
    xi = lgl_nodes(n)
    h = [(cfg.upper[a] - cfg.lower[a]) / cfg.cells[a] for a in range(cfg.dim)]
    shape_c = list(reversed(cfg.cells))          # [cz][cy][cx]
    out = np.zeros((cfg.n_sdof, 3))
    grids = []
    for a in range(cfg.dim):
        c = np.arange(cfg.cells[a])
        grids.append(cfg.lower[a] + (c[:, None] + 0.5 * (1.0 + xi[None, :])) * h[a])  # [c][i]
    if cfg.dim == 1:
        out[:, 0] = grids[0].reshape(-1)
    elif cfg.dim == 2:
        cy, cx, iy, ix = np.meshgrid(np.arange(cfg.cells[1]), np.arange(cfg.cells[0]),
                                     np.arange(n), np.arange(n), indexing="ij")
        out[:, 0] = grids[0][cx, ix].reshape(-1)
        out[:, 1] = grids[1][cy, iy].reshape(-1)
    else:
        cz, cy, cx, iz, iy, ix = np.meshgrid(*(np.arange(s) for s in shape_c),
                                             np.arange(n), np.arange(n), np.arange(n),
                                             indexing="ij")
        out[:, 0] = grids[0][cx, ix].reshape(-1)
        out[:, 1] = grids[1][cy, iy].reshape(-1)
        out[:, 2] = grids[2][cz, iz].reshape(-1)
    return out


def initial_state(cfg: Config) -> np.ndarray:
    """u0 at the LGL nodes (the u_n of the first slab)."""
    X = node_coords(cfg)
    x, y, z = X[:, 0], X[:, 1], X[:, 2]
    if cfg.u0 == "sin2pi_x":
        return np.sin(TWO_PI * x)
    if cfg.u0 == "sin2pix_sin2piy":
        return np.sin(TWO_PI * x) * np.sin(TWO_PI * y)
    if cfg.u0 == "sin2pi_xyz":
        return np.sin(TWO_PI * (x + y + z))
    if cfg.u0 == "burgers":
        rng = np.random.default_rng(cfg.seed)
        return 1.0 + 0.5 * np.sin(x) + 0.01 * rng.standard_normal(cfg.n_sdof)
    raise ValueError(cfg.u0)


def random_slab(cfg: Config, seed: int | None = None) -> np.ndarray:
    """U ~ uniform[-1, 1) over the slab (n_dof), PCG64(seed)."""
    rng = np.random.default_rng(cfg.seed if seed is None else seed)
    return rng.uniform(-1.0, 1.0, cfg.n_dof)


def residual_bytes(cfg: Config) -> int:
    """Algorithmic bytes of one R(U): read U and u_n, write R."""
    return 8 * (2 * cfg.n_dof + cfg.n_sdof)


def jvp_bytes(cfg: Config) -> int:
    return 16 * cfg.n_dof


# ---- initial data of the reference experiments (host side) -----------------
def rotating_pulse_exact(t, x, y, eps=0.001):
    """Analytic rotating-pulse solution (models.hpp:162-170), vectorised."""
    x0, y0 = np.asarray(x) - 0.5, np.asarray(y) - 0.5
    xq = x0 * np.cos(4.0 * t) + y0 * np.sin(4.0 * t) + 0.25
    yq = -x0 * np.sin(4.0 * t) + y0 * np.cos(4.0 * t)
    s2 = 0.004 + 4.0 * eps * t
    return (0.004 / s2) * np.exp(-(xq * xq + yq * yq) / s2)


def vortex_initial(x, y, Sv=5.0, M=0.5, gamma=1.4):
    """Isentropic vortex conservative state (rho, rho v1, rho v2, e), evaluated
    as printed in models.hpp:173-190; returns an (..., 4) array."""
    x, y = np.asarray(x, dtype=np.float64), np.asarray(y, dtype=np.float64)
    f = 1.0 - x * x - y * y
    rho_base = 1.0 - Sv * Sv * (gamma - 1.0) * M * M * np.exp(f) / (8.0 * math.pi * math.pi)
    if np.any(~(rho_base > 0.0)):
        raise ValueError("vortex_initial: density formula nonpositive")
    rho = rho_base ** (1.0 / (gamma - 1.0))
    v1 = 1.0 - Sv * y * np.exp(f / 2.0) / (2.0 * math.pi)
    v2 = Sv * x * np.exp(f / 2.0) / (2.0 * math.pi)
    P = rho ** gamma / (gamma * M * M)
    e = P / (gamma - 1.0) + 0.5 * (v1 * v1 + v2 * v2) / rho
    return np.stack([rho, rho * v1, rho * v2, e], axis=-1)


def grid_coords(dim, degree, cells, lower, upper) -> np.ndarray:
    """Node coordinates (n_cells * n^d, 3) in the reference order (mesh.hpp:70-90)."""
    cfg = Config("grid", dim, degree, 2, tuple(cells), tuple(lower), tuple(upper),
                 (0.0,) * dim, 0.0, "none", 0)
    return node_coords(cfg)
