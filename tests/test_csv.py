"""CSV output formats: byte-identical to the reference
writers.  Pinned by the reference's own KAT strings (test_experiments.cpp:
132-160); the C++ (include/stdgsem_csv.hpp) and Python writers must agree byte
for byte on larger 1/2/3-D cases.  CPU only."""
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2201_05800_b200 import csvio
from paper_2201_05800_b200 import build as B

ROOT = Path(__file__).resolve().parents[1]


def test_reference_kat_strings(tmp_path):  # test_experiments.cpp:132-160
    g = csvio.Grid(1, 1, [2], [0.0], [1.0])
    coeffs = np.array([1.0, 2.0, 3.0, 4.0])
    csvio.write_field_csv(g, coeffs, tmp_path / "f.csv")
    assert (tmp_path / "f.csv").read_text() == (
        "# stdgsem-csv v1 field\nx,component,value\n0,0,1\n0.5,0,2\n0.5,0,3\n1,0,4\n")
    times = [0.0, 0.5, 1.0]
    csvio.write_trajectory_csv(g, times, [coeffs] * 3, tmp_path / "t.csv")
    traj = (tmp_path / "t.csv").read_text()
    assert traj.startswith("# stdgsem-csv v1 trajectory\nstep,t,norm_c0\n0,0,")
    assert traj.count("\n") == 5
    elems = [np.linspace(0.0, 7.0, 8), np.linspace(8.0, 15.0, 8)]
    csvio.write_elements_csv(g, 2, times, elems, tmp_path / "e.csv")
    e = (tmp_path / "e.csv").read_text()
    assert e.startswith("# stdgsem-csv v1 elements\nelement,stage,tau,t,x,component,value\n"
                        "0,0,-1,0,0,0,0\n")
    assert e.count("\n") == 18
    # deterministic reruns (test_experiments.cpp:47-55)
    csvio.write_elements_csv(g, 2, times, elems, tmp_path / "e2.csv")
    assert (tmp_path / "e2.csv").read_text() == e


CPP = r'''
#include <cmath>
#include <random>
#include "stdgsem_csv.hpp"
using namespace stdgsem::gpu::csv;
int main(int argc, char** argv) {
  const std::string dir = argv[1];
  struct C { int d, p; std::vector<int> cells; int r; };
  const C cases[] = {{1, 3, {5}, 1}, {2, 2, {3, 2}, 1}, {3, 1, {2, 3, 2}, 1}, {2, 1, {3, 2}, 4},
                     {1, 2, {3}, 2}};
  int i = 0;
  for (const C& c : cases) {
    Grid g;
    g.d = c.d; g.p = c.p; g.cells = c.cells; g.r = c.r;
    g.lower.assign(size_t(c.d), 0.25); g.upper.assign(size_t(c.d), 1.75);
    std::vector<double> u(static_cast<size_t>(g.dof()));
    for (size_t k = 0; k < u.size(); ++k) u[k] = std::sin(0.37 * double(k)) * 1e-3 + 1.0 / (k + 3);
    const std::string s = dir + "/cpp" + std::to_string(i);
    write_field_csv(g, u, s + "_f.csv");
    write_trajectory_csv(g, {0.0, 0.125}, {u, u}, s + "_t.csv");
    std::vector<double> U(u.size() * 3);
    for (size_t k = 0; k < U.size(); ++k) U[k] = std::cos(0.11 * double(k));
    write_elements_csv(g, 3, {0.0, 0.2}, {U}, s + "_e.csv");
    ++i;
  }
  return 0;
}
'''


def test_cpp_and_python_writers_agree(tmp_path):
    B.build()
    src = tmp_path / "csv_writer.cpp"
    src.write_text(CPP)
    exe = tmp_path / "csv_writer"
    cxx = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else shutil.which("g++")
    lib = ROOT / "paper_2201_05800_b200"
    subprocess.run([cxx, "-std=c++17", "-O2", f"-I{ROOT / 'include'}", str(src), f"-L{lib}",
                    "-lstg_cuda", f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    subprocess.run([str(exe), str(tmp_path)], check=True)
    cases = [(1, 3, [5], 1), (2, 2, [3, 2], 1), (3, 1, [2, 3, 2], 1), (2, 1, [3, 2], 4),
             (1, 2, [3], 2)]
    for i, (d, p, cells, r) in enumerate(cases):
        g = csvio.Grid(d, p, cells, [0.25] * d, [1.75] * d, r=r)
        k = np.arange(g.dof, dtype=np.float64)
        u = np.sin(0.37 * k) * 1e-3 + 1.0 / (k + 3)
        kk = np.arange(3 * g.dof, dtype=np.float64)
        U = np.cos(0.11 * kk)
        s = tmp_path / f"py{i}"
        csvio.write_field_csv(g, u, f"{s}_f.csv")
        csvio.write_trajectory_csv(g, [0.0, 0.125], [u, u], f"{s}_t.csv")
        csvio.write_elements_csv(g, 3, [0.0, 0.2], [U], f"{s}_e.csv")
        for kind in ("f", "t", "e"):
            a = (tmp_path / f"cpp{i}_{kind}.csv").read_bytes()
            b = Path(f"{s}_{kind}.csv").read_bytes()
            assert a == b, (d, kind)


def test_multicomponent_rows_and_header(tmp_path):
    """r > 1 (Euler, r = 4): every row carries its component index in
    coeff_index order (csv.hpp:39-44, 57-71, 97-104) and the trajectory has a
    norm per component.  The 1-cell, p = 1, r = 2 case written out by hand."""
    g = csvio.Grid(1, 1, [1], [0.0], [1.0], r=2)
    u = np.array([1.0, -2.0, 3.0, 0.5])  # (node 0: c0, c1), (node 1: c0, c1)
    csvio.write_field_csv(g, u, tmp_path / "f.csv")
    assert (tmp_path / "f.csv").read_text() == (
        "# stdgsem-csv v1 field\nx,component,value\n0,0,1\n0,1,-2\n1,0,3\n1,1,0.5\n")
    csvio.write_trajectory_csv(g, [0.0], [u], tmp_path / "t.csv")
    # global mass: w = (1, 1), vol_scale = 1/2 -> norms sqrt((1 + 9)/2), sqrt((4 + 0.25)/2)
    assert (tmp_path / "t.csv").read_text() == (
        "# stdgsem-csv v1 trajectory\nstep,t,norm_c0,norm_c1\n"
        f"0,0,{csvio.fmt_g(np.sqrt(5.0))},{csvio.fmt_g(np.sqrt(2.125))}\n")
    U = np.arange(8.0)
    csvio.write_elements_csv(g, 2, [0.0, 1.0], [U], tmp_path / "e.csv")
    lines = (tmp_path / "e.csv").read_text().splitlines()
    assert lines[2:6] == ["0,0,-1,0,0,0,0", "0,0,-1,0,0,1,1", "0,0,-1,0,1,0,2", "0,0,-1,0,1,1,3"]
    assert lines[6] == "0,1,1,1,0,0,4" and len(lines) == 10
