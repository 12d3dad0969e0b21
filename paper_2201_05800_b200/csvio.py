"""The reference's deterministic CSV formats (csv.hpp:14-109) for slab
results fetched from the device: ``# stdgsem-csv v1 <label>`` header, values
printed with ``%.16g`` (C printf semantics; Python's %-formatting is correctly
rounded like glibc's, so the bytes match the C++ writers in
include/stdgsem_csv.hpp).  EXTENSION: d = 3 writes ``x,y,z``."""
from __future__ import annotations

import math
from typing import Sequence

import numpy as np

from .configs import lgl_nodes
from . import _lib as L


def fmt_g(v: float) -> str:  # csv.hpp:14-18
    return "%.16g" % float(v)


def _host(a) -> np.ndarray:
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    return np.asarray(a, dtype=np.float64)


def _lgl_weights(n: int) -> np.ndarray:
    x = np.zeros(n)
    w = np.zeros(n)
    L.load().stg_lgl_rule(n, x.ctypes.data, w.ctypes.data)
    return w


class Grid:
    """Uniform periodic mesh + LGL nodes (mesh.hpp:14-91), r components per
    node, component innermost (coeff_index, mesh.hpp:78-81)."""

    def __init__(self, d: int, p: int, cells: Sequence[int], lower: Sequence[float],
                 upper: Sequence[float], r: int = 1):
        self.d, self.p, self.r = int(d), int(p), int(r)
        self.cells, self.lower, self.upper = list(cells), list(lower), list(upper)
        self.n1 = self.p + 1
        self.npc = self.n1 ** self.d
        self.n_cells = int(np.prod(self.cells))
        self.dof = self.n_cells * self.npc * self.r

    def index(self, cell: int, node: int, comp: int) -> int:
        return (cell * self.npc + node) * self.r + comp

    def coord_header(self) -> str:
        return {1: "x", 2: "x,y", 3: "x,y,z"}[self.d]

    def coords(self):
        xi = lgl_nodes(self.n1)
        for cell in range(self.n_cells):
            for node in range(self.npc):
                c, q, x = cell, node, []
                for a in range(self.d):
                    ca, qa = c % self.cells[a], q % self.n1
                    c //= self.cells[a]
                    q //= self.n1
                    h = (self.upper[a] - self.lower[a]) / float(self.cells[a])
                    x.append(self.lower[a] + (ca + 0.5 * (1.0 + xi[qa])) * h)
                yield cell, node, x


def _open(path: str, label: str):
    f = open(path, "w", newline="\n")
    f.write(f"# stdgsem-csv v1 {label}\n")
    return f


def write_field_csv(g: Grid, coeffs, path: str, label: str = "field") -> None:
    """write_field_csv (csv.hpp:29-46)."""
    u = _host(coeffs)
    if u.size != g.dof:
        raise ValueError("write_field_csv: coefficient size mismatch")
    with _open(path, label) as f:
        f.write(f"{g.coord_header()},component,value\n")
        for cell, node, x in g.coords():
            xs = ",".join(fmt_g(v) for v in x)
            for comp in range(g.r):
                f.write(f"{xs},{comp},{fmt_g(u[g.index(cell, node, comp)])}\n")


def write_trajectory_csv(g: Grid, times, states, path: str, label: str = "trajectory") -> None:
    """write_trajectory_csv (csv.hpp:49-73): global mass-weighted L2 norm."""
    if len(states) != len(times):
        raise ValueError("write_trajectory_csv: size mismatch")
    w = _lgl_weights(g.n1)
    hprod = 1.0
    for a in range(g.d):
        hprod *= (g.upper[a] - g.lower[a]) / float(g.cells[a])
    vol_scale = hprod / math.pow(2.0, g.d)
    with _open(path, label) as f:
        f.write("step,t" + "".join(f",norm_c{c}" for c in range(g.r)) + "\n")
        for k, st in enumerate(states):
            u = _host(st)
            if u.size != g.dof:
                raise ValueError("write_trajectory_csv: state size mismatch")
            row = f"{k},{fmt_g(times[k])}"
            for comp in range(g.r):
                acc = 0.0
                for cell in range(g.n_cells):  # the reference's summation order
                    for node in range(g.npc):
                        wn = w[node % g.n1]
                        if g.d >= 2:
                            wn *= w[(node // g.n1) % g.n1]
                        if g.d >= 3:
                            wn *= w[node // (g.n1 * g.n1)]
                        v = u[g.index(cell, node, comp)]
                        acc += vol_scale * wn * v * v
                row += f",{fmt_g(math.sqrt(acc))}"
            f.write(row + "\n")


def write_elements_csv(g: Grid, n_tau: int, times, element_solutions, path: str,
                       label: str = "elements") -> None:
    """write_elements_csv (csv.hpp:77-109): one row per (element, stage, node,
    component)."""
    if len(element_solutions) + 1 != len(times):
        raise ValueError("write_elements_csv: size mismatch")
    tau = lgl_nodes(n_tau)
    coords = list(g.coords())
    with _open(path, label) as f:
        f.write(f"element,stage,tau,t,{g.coord_header()},component,value\n")
        for n, U in enumerate(element_solutions):
            U = _host(U)
            dt = times[n + 1] - times[n]
            for j in range(n_tau):
                t = times[n] + 0.5 * dt * (1.0 + tau[j])
                head = f"{n},{j},{fmt_g(tau[j])},{fmt_g(t)},"
                for cell, node, x in coords:
                    xs = ",".join(fmt_g(v) for v in x)
                    for comp in range(g.r):
                        val = U[j * g.dof + g.index(cell, node, comp)]
                        f.write(f"{head}{xs},{comp},{fmt_g(val)}\n")
