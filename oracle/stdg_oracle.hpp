// ===========================================================================
// stdg_oracle.hpp -- CPU ORACLE (TEST INFRASTRUCTURE ONLY).
//
// A plain-C++20 restatement (no Eigen) of the hot path of the reference
// space-time DG-SEM library `stdgsem` (/root/reference/proj/include/stdgsem).
// It is the CHECKER for the CUDA product in paper_2201_05800_b200/: only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may load it.  Nothing in the product links or calls it.
//
// Pinning: the reference cannot be compiled here (Eigen3, doctest and CLI11 are
// absent).  This restatement is pinned against every
// inline known-answer test the reference's own test suite holds for the path
// (tests/test_oracle_pins.py mirrors test_quadrature.cpp, test_operators.cpp,
// test_spatial.cpp, test_stdg.cpp, test_lodg.cpp, test_newton.cpp).
//
// EXTENSIONS (not in the reference, labelled where they appear):
//   * d = 3 tensor-product meshes (the reference throws for d not in {1,2},
//     mesh.hpp:39); layout generalises mesh.hpp:22-25 / mesh.hpp:70-81.
//   * Burgers with an entropy-conservative two-point volume flux
//     (flux differencing) and LLF interface flux -- "parity unpinned" by the
//     reference, pinned by reduction identities (see tests).
//   * matrix-free GMRES(m) (the reference calls Eigen::GMRES on an assembled
//     matrix, newton.hpp:68-77; Eigen is third-party and absent).
// ===========================================================================
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace stdg_oracle {

using Vec = std::vector<double>;

// Row-major small dense matrix.
struct Mat {
  int rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int r, int c) : rows(r), cols(c), a(size_t(r) * c, 0.0) {}
  double& operator()(int i, int j) { return a[size_t(i) * cols + j]; }
  double operator()(int i, int j) const { return a[size_t(i) * cols + j]; }
};

// --------------------------------------------------------------------------
// Quadrature -- quadrature.hpp:35-144
// --------------------------------------------------------------------------
// legendre_pair: quadrature.hpp:35-44
inline void legendre_pair(int m, double x, double& pm, double& pm1) {
  pm = 1.0;
  pm1 = 0.0;
  for (int k = 0; k < m; ++k) {
    const double next = ((2 * k + 1) * x * pm - double(k) * pm1) / double(k + 1);
    pm1 = pm;
    pm = next;
  }
}

inline double legendre(int m, double x) {
  double pm, pm1;
  legendre_pair(m, x, pm, pm1);
  return pm;
}

// legendre_derivs: quadrature.hpp:56-62
inline void legendre_derivs(int m, double x, double& dp, double& ddp) {
  double pm, pm1;
  legendre_pair(m, x, pm, pm1);
  const double x2m1 = x * x - 1.0;
  dp = double(m) * (x * pm - pm1) / x2m1;
  ddp = (2.0 * x * dp - double(m * (m + 1)) * pm) / (-x2m1);
}

struct Rule {
  int n = 0;
  Vec nodes, weights;
};

// lgl_rule: quadrature.hpp:66-105 (Newton on P'_m from Chebyshev-Gauss-Lobatto
// guesses, |dx| < 1e-15 or 100 iterations, explicit symmetrisation 90-99).
inline Rule lgl_rule(int n) {
  if (n < 2) throw std::invalid_argument("lgl_rule: need n >= 2 nodes");
  Rule r;
  r.n = n;
  r.nodes.assign(n, 0.0);
  r.weights.assign(n, 0.0);
  r.nodes[0] = -1.0;
  r.nodes[n - 1] = 1.0;
  const int m = n - 1;
  const double pi = 3.14159265358979323846;
  for (int i = 1; i < n - 1; ++i) {
    double x = -std::cos(pi * double(i) / double(m));
    for (int it = 0; it < 100; ++it) {
      double dp, ddp;
      legendre_derivs(m, x, dp, ddp);
      const double dx = dp / ddp;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    r.nodes[i] = x;
  }
  for (int i = 0; i < n; ++i) {
    const double sym = (r.nodes[i] - r.nodes[n - 1 - i]) / 2.0;
    if (2 * i < n - 1) {
      r.nodes[i] = sym;
      r.nodes[n - 1 - i] = -sym;
    } else if (2 * i == n - 1) {
      r.nodes[i] = 0.0;
    }
  }
  for (int i = 0; i < n; ++i) {
    const double p = legendre(m, r.nodes[i]);
    r.weights[i] = 2.0 / (double(n) * double(m) * p * p);
  }
  return r;
}

// lagrange_basis barycentric weights: quadrature.hpp:107-124 (rescaled so the
// largest magnitude is 1).
inline Vec barycentric_weights(const Rule& r) {
  const int n = r.n;
  Vec bw(n);
  for (int i = 0; i < n; ++i) {
    double w = 1.0;
    for (int j = 0; j < n; ++j)
      if (j != i) w *= r.nodes[i] - r.nodes[j];
    bw[i] = 1.0 / w;
  }
  double mx = 0.0;
  for (double v : bw) mx = std::max(mx, std::abs(v));
  for (double& v : bw) v /= mx;
  return bw;
}

// diff_matrix: quadrature.hpp:128-144.  D(j,i) = psi_i'(x_j); diagonal by the
// negative-sum trick so D 1 = 0 exactly.
inline Mat diff_matrix(const Rule& r) {
  const int n = r.n;
  const Vec bw = barycentric_weights(r);
  Mat D(n, n);
  for (int j = 0; j < n; ++j) {
    double diag = 0.0;
    for (int i = 0; i < n; ++i) {
      if (i == j) continue;
      D(j, i) = (bw[i] / bw[j]) / (r.nodes[j] - r.nodes[i]);
      diag -= D(j, i);
    }
    D(j, j) = diag;
  }
  return D;
}

// eval_interpolant: quadrature.hpp:147-165
inline double eval_interpolant(const Rule& r, const Vec& coeffs, double tau) {
  if (!(tau >= -1.0 && tau <= 1.0))
    throw std::invalid_argument("eval_interpolant: tau outside [-1,1]");
  const Vec bw = barycentric_weights(r);
  for (int j = 0; j < r.n; ++j)
    if (tau == r.nodes[j]) return coeffs[j];
  double num = 0.0, den = 0.0;
  for (int j = 0; j < r.n; ++j) {
    const double t = bw[j] / (tau - r.nodes[j]);
    num += t * coeffs[j];
    den += t;
  }
  return num / den;
}

// --------------------------------------------------------------------------
// Dense LU with partial pivoting (stand-in for Eigen::PartialPivLU, which is
// third-party, version unpinned; used at operators.hpp:59-60, lodg.hpp:25,
// newton.hpp:61).  Row-major, in place.
// --------------------------------------------------------------------------
struct LU {
  int n = 0;
  Mat lu;
  std::vector<int> piv;
  bool singular = false;
};

inline LU lu_factor(const Mat& A) {
  LU f;
  f.n = A.rows;
  f.lu = A;
  f.piv.resize(f.n);
  const int n = f.n;
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::abs(f.lu(k, k));
    for (int i = k + 1; i < n; ++i)
      if (std::abs(f.lu(i, k)) > best) {
        best = std::abs(f.lu(i, k));
        p = i;
      }
    f.piv[k] = p;
    if (p != k)
      for (int j = 0; j < n; ++j) std::swap(f.lu(k, j), f.lu(p, j));
    const double pivot = f.lu(k, k);
    if (pivot == 0.0) {
      f.singular = true;
      continue;
    }
    for (int i = k + 1; i < n; ++i) {
      const double l = f.lu(i, k) / pivot;
      f.lu(i, k) = l;
      if (l == 0.0) continue;
      for (int j = k + 1; j < n; ++j) f.lu(i, j) -= l * f.lu(k, j);
    }
  }
  return f;
}

inline Vec lu_solve(const LU& f, Vec b) {
  const int n = f.n;
  for (int k = 0; k < n; ++k)
    if (f.piv[k] != k) std::swap(b[k], b[f.piv[k]]);
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    for (int j = 0; j < i; ++j) s -= f.lu(i, j) * b[j];
    b[i] = s;
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int j = i + 1; j < n; ++j) s -= f.lu(i, j) * b[j];
    b[i] = s / f.lu(i, i);
  }
  return b;
}

inline Mat matmul(const Mat& A, const Mat& B) {
  Mat C(A.rows, B.cols);
  for (int i = 0; i < A.rows; ++i)
    for (int k = 0; k < A.cols; ++k)
      for (int j = 0; j < B.cols; ++j) C(i, j) += A(i, k) * B(k, j);
  return C;
}

inline Mat inverse(const Mat& A) {
  const LU f = lu_factor(A);
  Mat inv(A.rows, A.cols);
  for (int c = 0; c < A.cols; ++c) {
    Vec e(A.rows, 0.0);
    e[c] = 1.0;
    const Vec x = lu_solve(f, e);
    for (int r = 0; r < A.rows; ++r) inv(r, c) = x[r];
  }
  return inv;
}

// checked_inverse: lodg.hpp:23-29 (a-posteriori defect <= 1e-10).
inline Mat checked_inverse(const Mat& A, const std::string& ctx) {
  const Mat inv = inverse(A);
  const Mat P = matmul(A, inv);
  double defect = 0.0;
  for (int i = 0; i < A.rows; ++i)
    for (int j = 0; j < A.cols; ++j)
      defect = std::max(defect, std::abs(P(i, j) - (i == j ? 1.0 : 0.0)));
  if (!(defect <= 1e-10)) throw std::runtime_error(ctx + ": singular matrix");
  return inv;
}

// --------------------------------------------------------------------------
// Temporal SBP operators and Butcher tableaus -- operators.hpp:16-112
// --------------------------------------------------------------------------
struct Sbp {
  int n = 0;
  Vec w;   // M = diag(w)
  Mat D;   // nodal differentiation matrix
  Vec tau; // LGL nodes
};

// sbp_operators: operators.hpp:33-44
inline Sbp sbp_operators(int n) {
  if (n < 2) throw std::invalid_argument("sbp_operators: need n >= 2");
  const Rule r = lgl_rule(n);
  Sbp s;
  s.n = n;
  s.w = r.weights;
  s.D = diff_matrix(r);
  s.tau = r.nodes;
  return s;
}

// sbp_defect: operators.hpp:47-50, max |MD + (MD)^T - B|
inline double sbp_defect(const Sbp& s) {
  const int n = s.n;
  double d = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const double mdij = s.w[i] * s.D(i, j);
      const double mdji = s.w[j] * s.D(j, i);
      double b = 0.0;
      if (i == j && i == 0) b = -1.0;
      if (i == j && i == n - 1) b = 1.0;
      d = std::max(d, std::abs(mdij + mdji - b));
    }
  return d;
}

struct Tableau {
  int s = 0;
  Mat A;
  Vec b, c;
};

// to_butcher: operators.hpp:55-72.  A = (D + M^{-1} e1 e1^T)^{-1}/2.
inline Tableau to_butcher(const Sbp& ops) {
  const int n = ops.n;
  Mat K = ops.D;
  K(0, 0) += 1.0 / ops.w[0];
  const Mat Kinv = inverse(K);
  const Mat P = matmul(K, Kinv);
  double defect = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      defect = std::max(defect, std::abs(P(i, j) - (i == j ? 1.0 : 0.0)));
  if (!(defect <= 1e-10))
    throw std::runtime_error("to_butcher: singular operator");
  Tableau t;
  t.s = n;
  t.A = Mat(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) t.A(i, j) = Kinv(i, j) / 2.0;
  t.b.resize(n);
  t.c.resize(n);
  const Rule r = lgl_rule(n);
  for (int i = 0; i < n; ++i) {
    t.b[i] = ops.w[i] / 2.0;
    t.c[i] = (r.nodes[i] + 1.0) / 2.0;
  }
  return t;
}

// lobatto_tableau: operators.hpp:76-112 (closed forms, s in {2,3,4}).
inline Tableau lobatto_tableau(int s) {
  Tableau t;
  t.s = s;
  t.A = Mat(s, s);
  t.b.resize(s);
  t.c.resize(s);
  const double r5 = std::sqrt(5.0);
  auto setA = [&](std::initializer_list<double> v) {
    int k = 0;
    for (double x : v) t.A.a[k++] = x;
  };
  switch (s) {
    case 2:
      setA({0.5, -0.5, 0.5, 0.5});
      t.b = {0.5, 0.5};
      t.c = {0.0, 1.0};
      break;
    case 3:
      setA({1.0 / 6, -1.0 / 3, 1.0 / 6, 1.0 / 6, 5.0 / 12, -1.0 / 12, 1.0 / 6,
            2.0 / 3, 1.0 / 6});
      t.b = {1.0 / 6, 2.0 / 3, 1.0 / 6};
      t.c = {0.0, 0.5, 1.0};
      break;
    case 4:
      setA({1.0 / 12, -r5 / 12, r5 / 12, -1.0 / 12,
            1.0 / 12, 0.25, (10.0 - 7 * r5) / 60, r5 / 60,
            1.0 / 12, (10.0 + 7 * r5) / 60, 0.25, -r5 / 60,
            1.0 / 12, 5.0 / 12, 5.0 / 12, 1.0 / 12});
      t.b = {1.0 / 12, 5.0 / 12, 5.0 / 12, 1.0 / 12};
      t.c = {0.0, 0.5 - r5 / 10, 0.5 + r5 / 10, 1.0};
      break;
    default:
      throw std::invalid_argument("lobatto_tableau: s in {2,3,4}");
  }
  return t;
}

// --------------------------------------------------------------------------
// Mesh / DG space -- mesh.hpp:14-165, EXTENDED to d = 3.
// cell = (cz*ny + cy)*nx + cx, node = (iz*n + iy)*n + ix, r = 1.
// --------------------------------------------------------------------------
struct Space {
  int d = 1;
  int p = 1;           // spatial degree, n = p+1 nodes per axis
  int cells[3] = {1, 1, 1};
  double lower[3] = {0, 0, 0};
  double upper[3] = {1, 1, 1};
  double h[3] = {1, 1, 1};
  Rule rule;
  Mat D;

  int n1() const { return p + 1; }
  int n_cells() const { return cells[0] * cells[1] * cells[2]; }
  int npc() const {
    int k = 1;
    for (int a = 0; a < d; ++a) k *= n1();
    return k;
  }
  int64_t dof() const { return int64_t(n_cells()) * npc(); }
  int cell_index(int cx, int cy, int cz) const {
    return (cz * cells[1] + cy) * cells[0] + cx;
  }
  void cell_multi(int cell, int ci[3]) const {
    ci[0] = cell % cells[0];
    ci[1] = (cell / cells[0]) % cells[1];
    ci[2] = cell / (cells[0] * cells[1]);
  }
  // mesh.hpp:30-34 (periodic neighbour)
  int neighbor(int cell, int axis, int dir) const {
    int ci[3];
    cell_multi(cell, ci);
    ci[axis] = (ci[axis] + dir + cells[axis]) % cells[axis];
    return cell_index(ci[0], ci[1], ci[2]);
  }
  int node_index(int ix, int iy, int iz) const {
    return (iz * n1() + iy) * n1() + ix;
  }
  void node_multi(int node, int ni[3]) const {
    ni[0] = node % n1();
    ni[1] = d >= 2 ? (node / n1()) % n1() : 0;
    ni[2] = d >= 3 ? node / (n1() * n1()) : 0;
  }
  int64_t coeff(int cell, int node) const { return int64_t(cell) * npc() + node; }
  // node_coord: mesh.hpp:82-90
  void node_coord(int cell, int node, double x[3]) const {
    int ci[3], ni[3];
    cell_multi(cell, ci);
    node_multi(node, ni);
    for (int a = 0; a < 3; ++a) x[a] = 0.0;
    for (int a = 0; a < d; ++a)
      x[a] = lower[a] + (ci[a] + 0.5 * (1.0 + rule.nodes[ni[a]])) * h[a];
  }
};

// uniform_mesh + dg_space: mesh.hpp:37-55, 93-110 (d in {1,2} in the
// reference; d = 3 is an extension).  spacing = (upper-lower)/cells.
inline Space make_space(int d, int p, const int* cells, const double* lower,
                        const double* upper) {
  if (d < 1 || d > 3) throw std::invalid_argument("make_space: d in {1,2,3}");
  if (p < 1) throw std::invalid_argument("make_space: p >= 1");
  Space s;
  s.d = d;
  s.p = p;
  for (int a = 0; a < d; ++a) {
    if (!(upper[a] > lower[a]))
      throw std::invalid_argument("uniform_mesh: need upper > lower");
    if (cells[a] < 1) throw std::invalid_argument("uniform_mesh: cells >= 1");
    s.cells[a] = cells[a];
    s.lower[a] = lower[a];
    s.upper[a] = upper[a];
    s.h[a] = (upper[a] - lower[a]) / double(cells[a]);
  }
  s.rule = lgl_rule(p + 1);
  s.D = diff_matrix(s.rule);
  return s;
}

// global_mass: mesh.hpp:125-141.  vol_scale = prod(h)/2^d times tensor weights.
inline Vec global_mass(const Space& s) {
  Vec m(size_t(s.dof()));
  double hprod = 1.0;
  for (int a = 0; a < s.d; ++a) hprod *= s.h[a];
  const double vol_scale = hprod / std::pow(2.0, s.d);
  const auto& w = s.rule.weights;
  for (int cell = 0; cell < s.n_cells(); ++cell)
    for (int node = 0; node < s.npc(); ++node) {
      int ni[3];
      s.node_multi(node, ni);
      double wn = w[ni[0]];
      if (s.d >= 2) wn *= w[ni[1]];
      if (s.d >= 3) wn *= w[ni[2]];
      m[size_t(s.coeff(cell, node))] = vol_scale * wn;
    }
  return m;
}

// interpolate_scalar: mesh.hpp:145-165
inline Vec interpolate(const Space& s,
                       const std::function<double(const double*)>& f) {
  Vec u(size_t(s.dof()));
  for (int cell = 0; cell < s.n_cells(); ++cell)
    for (int node = 0; node < s.npc(); ++node) {
      double x[3];
      s.node_coord(cell, node, x);
      u[size_t(s.coeff(cell, node))] = f(x);
    }
  return u;
}

// --------------------------------------------------------------------------
// Spatial operator F = M^{-1} L_h for constant-velocity linear advection
// (advection_model models.hpp:40-66, llf_flux spatial.hpp:20-25,
// SpatialOperator::rhs spatial.hpp:107-266 with has_diffusion = false).
// The d = 3 branch is the tensor extension of the 2-D branch (140-155).
// --------------------------------------------------------------------------
struct Advection {
  Space s;
  double b[3] = {0, 0, 0};
  Vec mass;
};

inline Advection make_advection(const Space& s, const double* b) {
  Advection a;
  a.s = s;
  for (int k = 0; k < s.d; ++k) a.b[k] = b[k];
  a.mass = global_mass(s);
  return a;
}

// llf_flux for scalar advection with unit normal e_axis:
// 0.5*((F_c(uL)+F_c(uR)) n) + 0.5*lambda*(uL-uR), F_c(u) = u b^T,
// lambda = |b . n| (models.hpp:55-58).
inline double llf_advection(double uL, double uR, double b_axis) {
  const double lambda = std::abs(b_axis);
  return 0.5 * (uL * b_axis + uR * b_axis) + 0.5 * lambda * (uL - uR);
}

inline void advection_rhs(const Advection& op, const double* u, double* F) {
  const Space& s = op.s;
  const int n1 = s.n1();
  const int p = s.p;
  const Mat& D = s.D;
  const Vec& w = s.rule.weights;
  const int64_t dof = s.dof();
  std::vector<double> Lh(size_t(dof), 0.0);
  const int npc = s.npc();

  // Element integrals F_c : grad(psi) by collocation (spatial.hpp:117-156).
#pragma omp parallel
  {
  std::vector<double> flux(size_t(npc) * 3);
#pragma omp for schedule(static)
  for (int cell = 0; cell < s.n_cells(); ++cell) {
    for (int node = 0; node < npc; ++node) {
      const double un = u[s.coeff(cell, node)];
      for (int a = 0; a < s.d; ++a) flux[size_t(node) * 3 + a] = un * op.b[a];
    }
    if (s.d == 1) {
      const double hx = s.h[0];
      for (int i = 0; i < n1; ++i) {
        double val = w[i] * (hx / 2.0) * 0.0;  // source S = 0
        for (int k = 0; k < n1; ++k) val += w[k] * D(k, i) * flux[size_t(k) * 3 + 0];
        Lh[s.coeff(cell, i)] += val;
      }
    } else if (s.d == 2) {
      const double hx = s.h[0], hy = s.h[1];
      for (int ix = 0; ix < n1; ++ix)
        for (int iy = 0; iy < n1; ++iy) {
          double val = w[ix] * w[iy] * (hx * hy / 4.0) * 0.0;
          for (int k = 0; k < n1; ++k) {
            val += w[iy] * (hy / 2.0) * w[k] * D(k, ix) *
                   flux[size_t(s.node_index(k, iy, 0)) * 3 + 0];
            val += w[ix] * (hx / 2.0) * w[k] * D(k, iy) *
                   flux[size_t(s.node_index(ix, k, 0)) * 3 + 1];
          }
          Lh[s.coeff(cell, s.node_index(ix, iy, 0))] += val;
        }
    } else {  // EXTENSION: d = 3 tensor form of spatial.hpp:140-155
      const double hx = s.h[0], hy = s.h[1], hz = s.h[2];
      for (int ix = 0; ix < n1; ++ix)
        for (int iy = 0; iy < n1; ++iy)
          for (int iz = 0; iz < n1; ++iz) {
            double val = w[ix] * w[iy] * w[iz] * (hx * hy * hz / 8.0) * 0.0;
            for (int k = 0; k < n1; ++k) {
              val += w[iy] * (hy / 2.0) * w[iz] * (hz / 2.0) * w[k] * D(k, ix) *
                     flux[size_t(s.node_index(k, iy, iz)) * 3 + 0];
              val += w[ix] * (hx / 2.0) * w[iz] * (hz / 2.0) * w[k] * D(k, iy) *
                     flux[size_t(s.node_index(ix, k, iz)) * 3 + 1];
              val += w[ix] * (hx / 2.0) * w[iy] * (hy / 2.0) * w[k] * D(k, iz) *
                     flux[size_t(s.node_index(ix, iy, k)) * 3 + 2];
            }
            Lh[s.coeff(cell, s.node_index(ix, iy, iz))] += val;
          }
    }
  }
  }  // omp parallel

  // Facet integrals, facet-major (spatial.hpp:158-208): for each axis and
  // each cell's upper face, H at (L node i_a = p, R node i_a = 0);
  // L_L -= H wf, L_R += H wf, wf = prod of transverse w h/2 (1-D: 1).
  for (int axis = 0; axis < s.d; ++axis) {
    const int t1 = s.d >= 2 ? (axis == 0 ? 1 : 0) : -1;
    const int t2 = s.d >= 3 ? (axis == 2 ? 1 : 2) : -1;
    const int nq1 = t1 >= 0 ? n1 : 1;
    const int nq2 = t2 >= 0 ? n1 : 1;
    // Within one axis every face writes distinct (cell, node) slots (p >= 1),
    // so the facet loop is race-free and bitwise deterministic under OpenMP.
#pragma omp parallel for schedule(static) collapse(2)
    for (int cz = 0; cz < s.cells[2]; ++cz)
      for (int cy = 0; cy < s.cells[1]; ++cy)
        for (int cx = 0; cx < s.cells[0]; ++cx) {
          const int L = s.cell_index(cx, cy, cz);
          const int R = s.neighbor(L, axis, +1);
          for (int q2 = 0; q2 < nq2; ++q2)
            for (int q1 = 0; q1 < nq1; ++q1) {
              int iL[3] = {0, 0, 0}, iR[3] = {0, 0, 0};
              if (t1 >= 0) iL[t1] = iR[t1] = q1;
              if (t2 >= 0) iL[t2] = iR[t2] = q2;
              iL[axis] = p;
              iR[axis] = 0;
              const int nodeL = s.node_index(iL[0], iL[1], iL[2]);
              const int nodeR = s.node_index(iR[0], iR[1], iR[2]);
              double wf = 1.0;
              if (t1 >= 0) wf = s.rule.weights[q1] * s.h[t1] / 2.0;
              if (t2 >= 0) wf = wf * (s.rule.weights[q2] * s.h[t2] / 2.0);
              const double uL = u[s.coeff(L, nodeL)];
              const double uR = u[s.coeff(R, nodeR)];
              const double H = llf_advection(uL, uR, op.b[axis]);
              Lh[s.coeff(L, nodeL)] -= H * wf;
              Lh[s.coeff(R, nodeR)] += H * wf;
            }
        }
  }
  // F = L ./ m  (spatial.hpp:265)
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < dof; ++i) F[i] = Lh[size_t(i)] / op.mass[size_t(i)];
}

// --------------------------------------------------------------------------
// EXTENSION (not in the reference; "parity unpinned"): 1-D inviscid Burgers,
// f = u^2/2, entropy-conservative two-point flux f#(a,b) = (a^2+ab+b^2)/6,
// strong-form flux differencing with an LLF interface flux
// (lambda = max|u|) and SAT lifting.
// --------------------------------------------------------------------------
struct Burgers {
  Space s;
};

inline double burgers_f(double u) { return 0.5 * u * u; }
inline double burgers_ec(double a, double b) { return (a * a + a * b + b * b) / 6.0; }
inline double burgers_llf(double uL, double uR) {
  const double lambda = std::max(std::abs(uL), std::abs(uR));
  return 0.5 * (burgers_f(uL) + burgers_f(uR)) + 0.5 * lambda * (uL - uR);
}

inline void burgers_rhs(const Burgers& op, const double* u, double* F) {
  const Space& s = op.s;
  if (s.d != 1) throw std::invalid_argument("burgers: d = 1 only");
  const int n1 = s.n1();
  const int K = s.cells[0];
  const double sc = 2.0 / s.h[0];
  const auto& w = s.rule.weights;
  for (int c = 0; c < K; ++c) {
    const double* uc = u + int64_t(c) * n1;
    const double uLnb = u[int64_t((c + K - 1) % K) * n1 + (n1 - 1)];
    const double uRnb = u[int64_t((c + 1) % K) * n1 + 0];
    for (int i = 0; i < n1; ++i) {
      double vol = 0.0;
      for (int k = 0; k < n1; ++k) vol += 2.0 * s.D(i, k) * burgers_ec(uc[i], uc[k]);
      double val = -sc * vol;
      if (i == n1 - 1) val -= sc * (burgers_llf(uc[n1 - 1], uRnb) - burgers_f(uc[n1 - 1])) / w[n1 - 1];
      if (i == 0) val += sc * (burgers_llf(uLnb, uc[0]) - burgers_f(uc[0])) / w[0];
      F[int64_t(c) * n1 + i] = val;
    }
  }
}

// Exact directional derivative of burgers_rhs at u in direction v (the LLF
// lambda = max(|uL|,|uR|) is differentiated branch-wise; ties take uL).
inline void burgers_jvp(const Burgers& op, const double* u, const double* v,
                        double* Jv) {
  const Space& s = op.s;
  const int n1 = s.n1();
  const int K = s.cells[0];
  const double sc = 2.0 / s.h[0];
  const auto& w = s.rule.weights;
  auto dllf = [](double uL, double uR, double vL, double vR) {
    const double aL = std::abs(uL), aR = std::abs(uR);
    double lambda, dlambda;
    if (aL >= aR) {
      lambda = aL;
      dlambda = (uL >= 0 ? 1.0 : -1.0) * vL;
    } else {
      lambda = aR;
      dlambda = (uR >= 0 ? 1.0 : -1.0) * vR;
    }
    return 0.5 * (uL * vL + uR * vR) + 0.5 * dlambda * (uL - uR) +
           0.5 * lambda * (vL - vR);
  };
  for (int c = 0; c < K; ++c) {
    const double* uc = u + int64_t(c) * n1;
    const double* vc = v + int64_t(c) * n1;
    const int64_t iLn = int64_t((c + K - 1) % K) * n1 + (n1 - 1);
    const int64_t iRn = int64_t((c + 1) % K) * n1;
    for (int i = 0; i < n1; ++i) {
      double vol = 0.0;
      for (int k = 0; k < n1; ++k)
        vol += 2.0 * s.D(i, k) *
               ((2.0 * uc[i] + uc[k]) * vc[i] + (uc[i] + 2.0 * uc[k]) * vc[k]) / 6.0;
      double val = -sc * vol;
      if (i == n1 - 1)
        val -= sc * (dllf(uc[n1 - 1], u[iRn], vc[n1 - 1], v[iRn]) - uc[n1 - 1] * vc[n1 - 1]) / w[n1 - 1];
      if (i == 0)
        val += sc * (dllf(u[iLn], uc[0], v[iLn], vc[0]) - uc[0] * vc[0]) / w[0];
      Jv[int64_t(c) * n1 + i] = val;
    }
  }
}

// --------------------------------------------------------------------------
// General flux models with r components on d in {1, 2} (models.hpp:23-192)
// and SpatialOperator::rhs with interior-penalty diffusion
// (spatial.hpp:20-52, 107-266), restated in the reference's loop order.
//   kind 0: advdiff_model(d, b, eps) -- b constant or rotating_field()
//           (models.hpp:40-84); eps = 0 is plain advection_model
//   kind 1: euler_model(gamma), r = 4, d = 2 (models.hpp:118-159)
// --------------------------------------------------------------------------
// AdmissibilityError: models.hpp:15-20
struct AdmissibilityError : std::runtime_error {
  Vec state;
  AdmissibilityError(const std::string& what, Vec s)
      : std::runtime_error(what), state(std::move(s)) {}
};

struct GenModel {
  int kind = 0;    // 0 advdiff, 1 euler
  int r = 1;
  int d = 1;
  int field = 0;   // 0 constant b, 1 rotating_field (models.hpp:73-80)
  double b[3] = {0, 0, 0};
  double eps = 0.0;
  double gamma = 1.4;

  bool has_diffusion() const { return kind == 0 && eps > 0; }
  bool linear() const { return kind == 0; }
  void velocity(const double* x, double* bv) const {
    if (field == 1) {
      bv[0] = -4.0 * (x[1] - 0.5);
      bv[1] = 4.0 * (x[0] - 0.5);
    } else {
      for (int a = 0; a < d; ++a) bv[a] = b[a];
    }
  }
  // euler_pressure / require_admissible: models.hpp:100-113
  double pressure(const double* u) const {
    const double rho = u[0];
    const double kinetic = (u[1] * u[1] + u[2] * u[2]) / (2.0 * rho);
    return (gamma - 1.0) * (u[3] - kinetic);
  }
  void require_admissible(const double* u) const {
    if (!(u[0] > 0.0) || !(pressure(u) > 0.0))
      throw AdmissibilityError("euler_model: nonphysical state", Vec(u, u + 4));
  }
  // F_c(u, x): r x d row-major, f[comp*d + a]  (models.hpp:46-48, 126-141)
  void Fc(const double* u, const double* x, double* f) const {
    if (kind == 0) {
      double bv[3];
      velocity(x, bv);
      for (int a = 0; a < d; ++a) f[a] = u[0] * bv[a];
      return;
    }
    require_admissible(u);
    const double rho = u[0];
    const double v[2] = {u[1] / rho, u[2] / rho};
    const double P = pressure(u);
    const double e = u[3];
    for (int a = 0; a < 2; ++a) {
      f[0 * 2 + a] = rho * v[a];
      for (int i = 0; i < 2; ++i) f[(1 + i) * 2 + a] = rho * v[i] * v[a] + (i == a ? P : 0.0);
      f[3 * 2 + a] = (e + P) * v[a];
    }
  }
  // F_v(u, grad, x) = eps grad (models.hpp:70-72); zero for Euler
  void Fv(const double* grad, double* f) const {
    for (int k = 0; k < r * d; ++k) f[k] = kind == 0 ? eps * grad[k] : 0.0;
  }
  // max_wave_speed: models.hpp:55-58 (|b(x).n|), 145-156 (max |v.n| + c)
  double max_wave_speed(const double* uL, const double* uR, const double* n,
                        const double* x) const {
    if (kind == 0) {
      double bv[3];
      velocity(x, bv);
      double dot = 0.0;
      for (int a = 0; a < d; ++a) dot += bv[a] * n[a];
      return std::abs(dot);
    }
    double lambda = 0.0;
    for (const double* u : {uL, uR}) {
      require_admissible(u);
      const double rho = u[0];
      const double v[2] = {u[1] / rho, u[2] / rho};
      const double c = std::sqrt(gamma * pressure(u) / rho);
      lambda = std::max(lambda, std::abs(v[0] * n[0] + v[1] * n[1]) + c);
    }
    return lambda;
  }
};

struct GenOperator {
  Space s;       // geometry (r = 1 indexing); coefficients carry r components
  GenModel m;
  double eta = 1.0;
  Vec mass;      // per coefficient (replicated across components)
  int64_t dof() const { return s.dof() * m.r; }
  int64_t coeff(int cell, int node, int comp) const {
    return (int64_t(cell) * s.npc() + node) * m.r + comp;
  }
  // 2-D node_index(ix, iy) = iy*(p+1) + ix; 1-D: ix (mesh.hpp:70-72)
  int node2(int ix, int iy) const { return s.d == 1 ? ix : iy * s.n1() + ix; }
};

// assemble_semidiscrete: spatial.hpp:352-373 (eta default 10 p^2)
inline GenOperator make_gen_operator(const Space& s, const GenModel& m, double eta) {
  if (s.d > 2) throw std::invalid_argument("general models: d in {1, 2}");
  if (m.d != s.d) throw std::invalid_argument("assemble_semidiscrete: dimension mismatch");
  if (m.kind == 1 && (m.r != 4 || s.d != 2))
    throw std::invalid_argument("euler_model: r = 4, d = 2");
  if (m.kind == 0 && m.r != 1) throw std::invalid_argument("advdiff_model: r = 1");
  if (m.kind == 0 && m.eps < 0) throw std::invalid_argument("advdiff_model: need eps >= 0");
  if (m.kind == 1 && !(m.gamma > 1.0)) throw std::invalid_argument("euler_model: gamma > 1");
  GenOperator op;
  op.s = s;
  op.m = m;
  op.eta = eta > 0 ? eta : 10.0 * s.p * s.p;
  const Vec m1 = global_mass(s);
  op.mass.resize(size_t(op.dof()));
  for (int64_t k = 0; k < s.dof(); ++k)
    for (int c = 0; c < m.r; ++c) op.mass[size_t(k * m.r + c)] = m1[size_t(k)];
  return op;
}

// SpatialOperator::rhs: spatial.hpp:107-266
inline void gen_rhs(const GenOperator& op, const double* u, double* F) {
  const Space& s = op.s;
  const GenModel& m = op.m;
  const int n1 = s.n1(), p = s.p, r = m.r, d = s.d, npc = s.npc();
  const Mat& D = s.D;
  const Vec& w = s.rule.weights;
  const int64_t dof = op.dof();
  std::vector<double> Lh(size_t(dof), 0.0);
  const bool diff = m.has_diffusion();
  const size_t R1 = static_cast<size_t>(r), RD = static_cast<size_t>(r) * d;
  std::vector<double> loc(static_cast<size_t>(npc) * R1), grads(static_cast<size_t>(npc) * RD),
      flux(static_cast<size_t>(npc) * RD), fv(RD);
  // element integrals (F_c - F_v) : grad(psi), S = 0 (spatial.hpp:117-156)
  for (int cell = 0; cell < s.n_cells(); ++cell) {
    for (int node = 0; node < npc; ++node)
      for (int c = 0; c < r; ++c) loc[size_t(node) * r + c] = u[op.coeff(cell, node, c)];
    if (diff) {  // local_grad: spatial.hpp:72-99
      std::fill(grads.begin(), grads.end(), 0.0);
      const double sx = 2.0 / s.h[0];
      if (d == 1) {
        for (int i = 0; i < n1; ++i)
          for (int k = 0; k < n1; ++k)
            for (int c = 0; c < r; ++c)
              grads[(size_t(i) * r + c) * d + 0] += sx * D(i, k) * loc[size_t(k) * r + c];
      } else {
        const double sy = 2.0 / s.h[1];
        for (int ix = 0; ix < n1; ++ix)
          for (int iy = 0; iy < n1; ++iy) {
            const int g = op.node2(ix, iy);
            for (int k = 0; k < n1; ++k)
              for (int c = 0; c < r; ++c) {
                grads[(size_t(g) * r + c) * d + 0] +=
                    sx * D(ix, k) * loc[size_t(op.node2(k, iy)) * r + c];
                grads[(size_t(g) * r + c) * d + 1] +=
                    sy * D(iy, k) * loc[size_t(op.node2(ix, k)) * r + c];
              }
          }
      }
    }
    for (int node = 0; node < npc; ++node) {
      double x[3];
      s.node_coord(cell, node, x);
      m.Fc(&loc[size_t(node) * r], x, &flux[size_t(node) * r * d]);
      if (diff) {
        m.Fv(&grads[size_t(node) * r * d], fv.data());
        for (int k = 0; k < r * d; ++k) flux[size_t(node) * r * d + k] -= fv[size_t(k)];
      }
    }
    if (d == 1) {
      const double h = s.h[0];
      for (int i = 0; i < n1; ++i)
        for (int c = 0; c < r; ++c) {
          double val = w[i] * (h / 2.0) * 0.0;
          for (int k = 0; k < n1; ++k) val += w[k] * D(k, i) * flux[(size_t(k) * r + c) * d + 0];
          Lh[op.coeff(cell, i, c)] += val;
        }
    } else {
      const double hx = s.h[0], hy = s.h[1];
      for (int ix = 0; ix < n1; ++ix)
        for (int iy = 0; iy < n1; ++iy)
          for (int c = 0; c < r; ++c) {
            double val = w[ix] * w[iy] * (hx * hy / 4.0) * 0.0;
            for (int k = 0; k < n1; ++k) {
              val += w[iy] * (hy / 2.0) * w[k] * D(k, ix) *
                     flux[(size_t(op.node2(k, iy)) * r + c) * d + 0];
              val += w[ix] * (hx / 2.0) * w[k] * D(k, iy) *
                     flux[(size_t(op.node2(ix, k)) * r + c) * d + 1];
            }
            Lh[op.coeff(cell, op.node2(ix, iy), c)] += val;
          }
    }
  }
  // facet integrals, facet-major (spatial.hpp:158-261)
  std::vector<double> uL(R1), uR(R1), FL(RD), FR(RD), H(R1), gL(RD), gR(RD), uavg(R1), jt(RD),
      fvL(RD), fvR(RD), fj(RD), jump(R1), avg(R1);
  for (int axis = 0; axis < d; ++axis) {
    const int nx = s.cells[0];
    const int ny = d == 2 ? s.cells[1] : 1;
    const double h_n = s.h[axis];
    const double h_e = d == 2 ? s.h[axis] : s.h[0];
    double nrm[2] = {0.0, 0.0};
    nrm[axis] = 1.0;
    for (int cy = 0; cy < ny; ++cy)
      for (int cx = 0; cx < nx; ++cx) {
        const int L = s.cell_index(cx, cy, 0);
        const int R = s.neighbor(L, axis, +1);
        const int n_trans = d == 2 ? n1 : 1;
        for (int q = 0; q < n_trans; ++q) {
          const int nodeL = d == 1 ? p : (axis == 0 ? op.node2(p, q) : op.node2(q, p));
          const int nodeR = d == 1 ? 0 : (axis == 0 ? op.node2(0, q) : op.node2(q, 0));
          double x[3] = {0.0, 0.0, 0.0};
          {
            int ci[3];
            s.cell_multi(L, ci);
            x[axis] = s.lower[axis] + (ci[axis] + 1) * s.h[axis];
            if (d == 2) {
              const int tangent = 1 - axis;
              x[tangent] = s.lower[tangent] +
                           (ci[tangent] + 0.5 * (1.0 + s.rule.nodes[q])) * s.h[tangent];
            }
          }
          const double wf = d == 2 ? s.rule.weights[q] * s.h[1 - axis] / 2.0 : 1.0;
          for (int c = 0; c < r; ++c) {
            uL[size_t(c)] = u[op.coeff(L, nodeL, c)];
            uR[size_t(c)] = u[op.coeff(R, nodeR, c)];
          }
          // llf_flux: spatial.hpp:20-25
          const double lambda = m.max_wave_speed(uL.data(), uR.data(), nrm, x);
          m.Fc(uL.data(), x, FL.data());
          m.Fc(uR.data(), x, FR.data());
          for (int c = 0; c < r; ++c) {
            double fn = 0.0;
            for (int a = 0; a < d; ++a)
              fn += (FL[size_t(c) * d + a] + FR[size_t(c) * d + a]) * nrm[a];
            H[size_t(c)] = 0.5 * fn + 0.5 * lambda * (uL[size_t(c)] - uR[size_t(c)]);
          }
          for (int c = 0; c < r; ++c) {
            Lh[op.coeff(L, nodeL, c)] -= H[size_t(c)] * wf;
            Lh[op.coeff(R, nodeR, c)] += H[size_t(c)] * wf;
          }
          if (!diff) continue;
          // gradient traces (spatial.hpp:213-240)
          std::fill(gL.begin(), gL.end(), 0.0);
          std::fill(gR.begin(), gR.end(), 0.0);
          const double sn = 2.0 / h_n;
          for (int k = 0; k < n1; ++k) {
            const int lkn = d == 1 ? k : (axis == 0 ? op.node2(k, q) : op.node2(q, k));
            for (int c = 0; c < r; ++c) {
              gL[size_t(c) * d + axis] += sn * D(n1 - 1, k) * u[op.coeff(L, lkn, c)];
              gR[size_t(c) * d + axis] += sn * D(0, k) * u[op.coeff(R, lkn, c)];
            }
          }
          if (d == 2) {
            const int tangent = 1 - axis;
            const double st = 2.0 / s.h[tangent];
            for (int k = 0; k < n1; ++k) {
              const int ltk = axis == 0 ? op.node2(p, k) : op.node2(k, p);
              const int rtk = axis == 0 ? op.node2(0, k) : op.node2(k, 0);
              for (int c = 0; c < r; ++c) {
                gL[size_t(c) * d + tangent] += st * D(q, k) * u[op.coeff(L, ltk, c)];
                gR[size_t(c) * d + tangent] += st * D(q, k) * u[op.coeff(R, rtk, c)];
              }
            }
          }
          // interior_penalty_surface: spatial.hpp:35-52
          for (int c = 0; c < r; ++c) {
            uavg[size_t(c)] = 0.5 * (uL[size_t(c)] + uR[size_t(c)]);
            for (int a = 0; a < d; ++a) jt[size_t(c) * d + a] = (uL[size_t(c)] - uR[size_t(c)]) * nrm[a];
          }
          m.Fv(jt.data(), fj.data());
          m.Fv(gL.data(), fvL.data());
          m.Fv(gR.data(), fvR.data());
          for (int c = 0; c < r; ++c) {
            double jf = 0.0, af = 0.0;
            for (int a = 0; a < d; ++a) {
              jf += fj[size_t(c) * d + a] * nrm[a];
              af += (fvL[size_t(c) * d + a] + fvR[size_t(c) * d + a]) * nrm[a];
            }
            jump[size_t(c)] = jf;
            avg[size_t(c)] = 0.5 * af;
          }
          for (int c = 0; c < r; ++c) {
            const double sym = -0.5 * jump[size_t(c)];
            const double tL = -avg[size_t(c)] + (op.eta / h_e) * jump[size_t(c)];
            const double tR = avg[size_t(c)] - (op.eta / h_e) * jump[size_t(c)];
            Lh[op.coeff(L, nodeL, c)] -= tL * wf;
            Lh[op.coeff(R, nodeR, c)] -= tR * wf;
            // symmetry term along the normal line (spatial.hpp:248-259)
            for (int i = 0; i < n1; ++i) {
              const int lin = d == 1 ? i : (axis == 0 ? op.node2(i, q) : op.node2(q, i));
              Lh[op.coeff(L, lin, c)] -= sym * D(n1 - 1, i) * sn * wf;
              Lh[op.coeff(R, lin, c)] -= sym * D(0, i) * sn * wf;
            }
          }
        }
      }
  }
  for (int64_t i = 0; i < dof; ++i) F[i] = Lh[size_t(i)] / op.mass[size_t(i)];
}

// --------------------------------------------------------------------------
// Semidiscrete system seam (system.hpp:16-23): rhs(t, u) plus a flag for
// linearity (spatial_jacobian's exact branch, spatial.hpp:290-298).
// --------------------------------------------------------------------------
struct System {
  int64_t dof = 0;
  bool linear = true;
  std::function<void(double, const double*, double*)> rhs;
  // Spatial Jacobian action J_F(t,u) v.  For linear models it is the exact
  // "probe from the zero state" difference rhs(v) - rhs(0) (spatial.hpp:290).
  std::function<void(double, const double*, const double*, double*)> jac;
};

inline System advection_system(const Advection& op) {
  System sys;
  sys.dof = op.s.dof();
  sys.linear = true;
  auto opp = std::make_shared<Advection>(op);
  sys.rhs = [opp](double, const double* u, double* F) { advection_rhs(*opp, u, F); };
  // The zero-state probe rhs(0) is computed once and cached, as the
  // reference caches the Jacobian of linear models (spatial.hpp:375-383).
  auto base = std::make_shared<Vec>();
  sys.jac = [opp, base](double, const double*, const double* v, double* Jv) {
    const int64_t n = opp->s.dof();
    if (base->empty()) {
      Vec zero(static_cast<size_t>(n), 0.0);
      base->resize(static_cast<size_t>(n));
      advection_rhs(*opp, zero.data(), base->data());
    }
    advection_rhs(*opp, v, Jv);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) Jv[i] -= (*base)[size_t(i)];
  };
  return sys;
}

inline System burgers_system(const Burgers& op) {
  System sys;
  sys.dof = op.s.dof();
  sys.linear = false;
  auto opp = std::make_shared<Burgers>(op);
  sys.rhs = [opp](double, const double* u, double* F) { burgers_rhs(*opp, u, F); };
  sys.jac = [opp](double, const double* u, const double* v, double* Jv) {
    burgers_jvp(*opp, u, v, Jv);
  };
  return sys;
}

// advdiff: linear, J v = rhs(v) - rhs(0) (spatial.hpp:290-298, cached base);
// euler: the reference assembles a coloured central-difference Jacobian
// (spatial.hpp:299-320, step sqrt(eps)(1+|u_j|)); its action is restated as
// the directional central difference with step 1e-7 (1 + ||u||_inf)/||v||_inf.
inline System gen_system(const GenOperator& op) {
  System sys;
  sys.dof = op.dof();
  sys.linear = op.m.linear();
  auto opp = std::make_shared<GenOperator>(op);
  sys.rhs = [opp](double, const double* u, double* F) { gen_rhs(*opp, u, F); };
  if (sys.linear) {
    auto base = std::make_shared<Vec>();
    sys.jac = [opp, base](double, const double*, const double* v, double* Jv) {
      const int64_t n = opp->dof();
      if (base->empty()) {
        Vec zero(static_cast<size_t>(n), 0.0);
        base->resize(static_cast<size_t>(n));
        gen_rhs(*opp, zero.data(), base->data());
      }
      gen_rhs(*opp, v, Jv);
      for (int64_t i = 0; i < n; ++i) Jv[i] -= (*base)[size_t(i)];
    };
  } else {
    sys.jac = [opp](double, const double* u, const double* v, double* Jv) {
      const int64_t n = opp->dof();
      double un = 0.0, vn = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        un = std::max(un, std::abs(u[i]));
        vn = std::max(vn, std::abs(v[i]));
      }
      if (vn == 0.0) {
        for (int64_t i = 0; i < n; ++i) Jv[i] = 0.0;
        return;
      }
      const double h = 1e-7 * (1.0 + un) / vn;
      Vec up(u, u + n), um(u, u + n), Fp(static_cast<size_t>(n)), Fm(static_cast<size_t>(n));
      for (int64_t i = 0; i < n; ++i) {
        up[size_t(i)] += h * v[i];
        um[size_t(i)] -= h * v[i];
      }
      gen_rhs(*opp, up.data(), Fp.data());
      gen_rhs(*opp, um.data(), Fm.data());
      for (int64_t i = 0; i < n; ++i) Jv[i] = (Fp[size_t(i)] - Fm[size_t(i)]) / (2.0 * h);
    };
  }
  return sys;
}

// test_equation_system: system.hpp:26-44 -- scalar u' = -u, u(0) = 4.
inline System test_equation_system() {
  System sys;
  sys.dof = 1;
  sys.linear = true;
  sys.rhs = [](double, const double* u, double* F) { F[0] = -u[0]; };
  sys.jac = [](double, const double*, const double* v, double* Jv) { Jv[0] = -v[0]; };
  return sys;
}

// zero_system: test_stdg.cpp:30-38 -- F == 0 (fake backend used by the pins).
inline System zero_system() {
  System sys;
  sys.dof = 1;
  sys.linear = true;
  sys.rhs = [](double, const double*, double* F) { F[0] = 0.0; };
  sys.jac = [](double, const double*, const double*, double* Jv) { Jv[0] = 0.0; };
  return sys;
}

// --------------------------------------------------------------------------
// STDG slab -- stdg.hpp:21-143
// --------------------------------------------------------------------------
// st_node_times: stdg.hpp:33-39
inline Vec st_node_times(const Sbp& ops, double t_n, double dt) {
  Vec t(ops.n);
  for (int i = 0; i < ops.n; ++i) t[i] = t_n + 0.5 * dt * (1.0 + ops.tau[i]);
  return t;
}

// st_residual: stdg.hpp:56-76
// res_i = (B U*)_i - sum_j D(j,i) M(j,j) U_j - (dt/2) M(i,i) F(t_i, U_i)
inline void st_residual(const System& sys, const Sbp& ops, double t_n, double dt,
                        const double* u_n, const double* U, double* res) {
  const int n = ops.n;
  const int64_t dof = sys.dof;
  const Vec times = st_node_times(ops, t_n, dt);
  for (int64_t k = 0; k < n * dof; ++k) res[k] = 0.0;
  for (int64_t k = 0; k < dof; ++k) res[k] -= u_n[k];
  for (int64_t k = 0; k < dof; ++k) res[(n - 1) * dof + k] += U[(n - 1) * dof + k];
  Vec F(static_cast<size_t>(dof));
  for (int i = 0; i < n; ++i) {
    double* block = res + i * dof;
    for (int j = 0; j < n; ++j) {
      const double c = ops.D(j, i) * ops.w[j];
      const double* Uj = U + j * dof;
#pragma omp parallel for schedule(static)
      for (int64_t k = 0; k < dof; ++k) block[k] -= c * Uj[k];
    }
    sys.rhs(times[i], U + i * dof, F.data());
    const double c = 0.5 * dt * ops.w[i];
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < dof; ++k) block[k] -= c * F[size_t(k)];
  }
}

// st_jacobian action: stdg.hpp:79-110 applied to v (the reference assembles
// (e_n e_n^T - D^T M) (x) I - (dt/2)(M (x) I) blockdiag(J_i)).
inline void st_jacobian_apply(const System& sys, const Sbp& ops, double t_n,
                              double dt, const double* U, const double* v,
                              double* Jv) {
  const int n = ops.n;
  const int64_t dof = sys.dof;
  const Vec times = st_node_times(ops, t_n, dt);
  for (int64_t k = 0; k < n * dof; ++k) Jv[k] = 0.0;
  Vec JF(static_cast<size_t>(dof));
  for (int i = 0; i < n; ++i) {
    double* block = Jv + i * dof;
    for (int j = 0; j < n; ++j) {
      double value = -ops.D(j, i) * ops.w[j];
      if (i == n - 1 && j == n - 1) value += 1.0;
      if (value == 0.0) continue;
      const double* vj = v + j * dof;
      for (int64_t k = 0; k < dof; ++k) block[k] += value * vj[k];
    }
    sys.jac(times[i], U + i * dof, v + i * dof, JF.data());
    const double scale = -0.5 * dt * ops.w[i];
    for (int64_t k = 0; k < dof; ++k) block[k] += scale * JF[size_t(k)];
  }
}

// --------------------------------------------------------------------------
// LoDG stage residual -- lodg.hpp:104-122
// --------------------------------------------------------------------------
enum class JacForm { a_form = 0, a_inv_form = 1 };

inline void stage_residual(const System& sys, const Tableau& tab, double t,
                           double dt, const double* u, const double* U,
                           JacForm form, double* R) {
  const int s = tab.s;
  const int64_t dof = sys.dof;
  std::vector<double> F(size_t(s) * dof);
  for (int j = 0; j < s; ++j)
    sys.rhs(t + tab.c[j] * dt, U + j * dof, F.data() + j * dof);
  Mat Ainv;
  if (form == JacForm::a_inv_form) Ainv = checked_inverse(tab.A, "rk_step");
  for (int i = 0; i < s; ++i) {
    double* block = R + i * dof;
    if (form == JacForm::a_form) {
      for (int64_t k = 0; k < dof; ++k) block[k] = U[i * dof + k] - u[k];
      for (int j = 0; j < s; ++j) {
        const double c = dt * tab.A(i, j);
        for (int64_t k = 0; k < dof; ++k) block[k] -= c * F[size_t(j * dof + k)];
      }
    } else {
      for (int64_t k = 0; k < dof; ++k) block[k] = -F[size_t(i * dof + k)];
      for (int j = 0; j < s; ++j) {
        const double c = Ainv(i, j) / dt;
        for (int64_t k = 0; k < dof; ++k) block[k] += c * (U[j * dof + k] - u[k]);
      }
    }
  }
}

// stage_jacobian action: lodg.hpp:43-85 applied to v.
inline void stage_jacobian_apply(const System& sys, const Tableau& tab, double t,
                                 double dt, const double* U, JacForm form,
                                 const double* v, double* Jv) {
  const int s = tab.s;
  const int64_t dof = sys.dof;
  for (int64_t k = 0; k < s * dof; ++k) Jv[k] = 0.0;
  Vec JF(static_cast<size_t>(dof));
  if (form == JacForm::a_form) {
    for (int j = 0; j < s; ++j) {
      sys.jac(t + tab.c[j] * dt, U + j * dof, v + j * dof, JF.data());
      for (int i = 0; i < s; ++i) {
        const double c = -dt * tab.A(i, j);
        for (int64_t k = 0; k < dof; ++k) Jv[i * dof + k] += c * JF[size_t(k)];
      }
    }
    for (int64_t k = 0; k < s * dof; ++k) Jv[k] += v[k];
  } else {
    const Mat Ainv = checked_inverse(tab.A, "stage_jacobian");
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j) {
        const double c = Ainv(i, j) / dt;
        if (c == 0.0) continue;
        for (int64_t k = 0; k < dof; ++k) Jv[i * dof + k] += c * v[j * dof + k];
      }
    for (int i = 0; i < s; ++i) {
      sys.jac(t + tab.c[i] * dt, U + i * dof, v + i * dof, JF.data());
      for (int64_t k = 0; k < dof; ++k) Jv[i * dof + k] -= JF[size_t(k)];
    }
  }
}

// --------------------------------------------------------------------------
// Linear solvers and Newton -- newton.hpp:28-130
// --------------------------------------------------------------------------
enum class LinearMethod { auto_select = 0, dense_lu = 1, gmres = 3 };

struct NewtonConfig {
  double abs_tol = 1e-12;
  double rel_tol = 1e-12;
  int max_iter = 50;
  LinearMethod linear = LinearMethod::auto_select;
  int gmres_restart = 30;
  double gmres_tol = 1e-12;
  int gmres_max_it = 1000;
};

struct NonconvergenceError : std::runtime_error {
  Vec last_iterate;
  std::vector<double> residual_history;
  NonconvergenceError(const std::string& what, Vec u, std::vector<double> h)
      : std::runtime_error(what), last_iterate(std::move(u)), residual_history(std::move(h)) {}
};

using LinOp = std::function<void(const double*, double*)>;

struct GmresStats {
  int iterations = 0;
  double rel_residual = 0.0;
  bool converged = false;
};

inline double dot(const double* a, const double* b, int64_t n) {
  double s = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : s)
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

// Restarted GMRES(m), right-unpreconditioned, modified Gram-Schmidt Arnoldi
// with Givens rotations; stop when ||b - A x||_2 <= tol ||b||_2 (the
// tolerance semantics of Eigen::IterativeSolverBase used at newton.hpp:68-77).
inline GmresStats gmres(const LinOp& A, const double* b, double* x, int64_t n,
                        int restart, double tol, int max_it) {
  GmresStats st;
  const double bnorm = std::sqrt(dot(b, b, n));
  if (bnorm == 0.0) {
    for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
    st.converged = true;
    return st;
  }
  const int m = restart;
  std::vector<Vec> V(size_t(m + 1), Vec(static_cast<size_t>(n)));
  Mat H(m + 1, m);
  Vec cs(m), sn(m), g(m + 1);
  Vec r(static_cast<size_t>(n)), w(static_cast<size_t>(n));
  int total = 0;
  while (true) {
    A(x, r.data());
    for (int64_t i = 0; i < n; ++i) r[size_t(i)] = b[i] - r[size_t(i)];
    double beta = std::sqrt(dot(r.data(), r.data(), n));
    st.rel_residual = beta / bnorm;
    if (st.rel_residual <= tol) {
      st.converged = true;
      break;
    }
    if (total >= max_it) break;
    for (int64_t i = 0; i < n; ++i) V[0][size_t(i)] = r[size_t(i)] / beta;
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int k = 0;
    for (; k < m && total < max_it; ++k) {
      ++total;
      A(V[k].data(), w.data());
      for (int j = 0; j <= k; ++j) {
        const double hjk = dot(w.data(), V[j].data(), n);
        H(j, k) = hjk;
        double* wp = w.data();
        const double* vp = V[j].data();
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) wp[i] -= hjk * vp[i];
      }
      const double hn = std::sqrt(dot(w.data(), w.data(), n));
      H(k + 1, k) = hn;
      if (hn != 0.0) {
        double* vp = V[k + 1].data();
        const double* wp = w.data();
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) vp[i] = wp[i] / hn;
      }
      for (int j = 0; j < k; ++j) {
        const double t0 = cs[j] * H(j, k) + sn[j] * H(j + 1, k);
        H(j + 1, k) = -sn[j] * H(j, k) + cs[j] * H(j + 1, k);
        H(j, k) = t0;
      }
      const double den = std::hypot(H(k, k), H(k + 1, k));
      cs[k] = den == 0.0 ? 1.0 : H(k, k) / den;
      sn[k] = den == 0.0 ? 0.0 : H(k + 1, k) / den;
      H(k, k) = den;
      H(k + 1, k) = 0.0;
      g[k + 1] = -sn[k] * g[k];
      g[k] = cs[k] * g[k];
      if (std::abs(g[k + 1]) / bnorm <= tol || hn == 0.0) {
        ++k;
        break;
      }
    }
    // back substitution, update x
    Vec y(static_cast<size_t>(k));
    for (int i = k - 1; i >= 0; --i) {
      double s = g[i];
      for (int j = i + 1; j < k; ++j) s -= H(i, j) * y[size_t(j)];
      y[size_t(i)] = s / H(i, i);
    }
    for (int j = 0; j < k; ++j) {
      const double yj = y[size_t(j)];
      const double* vp = V[j].data();
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) x[i] += yj * vp[i];
    }
  }
  st.iterations = total;
  return st;
}

// Dense Jacobian by columns of a matrix-free action (small problems only).
inline Mat assemble_dense(const LinOp& A, int64_t n) {
  if (n > 6000) throw std::invalid_argument("assemble_dense: too large");
  Mat M(static_cast<int>(n), static_cast<int>(n));
  Vec e(size_t(n), 0.0), col(static_cast<size_t>(n));
  for (int64_t c = 0; c < n; ++c) {
    e[size_t(c)] = 1.0;
    A(e.data(), col.data());
    e[size_t(c)] = 0.0;
    for (int64_t r = 0; r < n; ++r) M(int(r), int(c)) = col[size_t(r)];
  }
  return M;
}

// linear_solve: newton.hpp:51-86 (dense LU with the a-posteriori defect gate
// ||Ax-b||_inf <= 1e-10 (1+||b||_inf); GMRES returns before the gate).
inline Vec linear_solve(const LinOp& A, const Vec& b, const NewtonConfig& cfg,
                        GmresStats* stats = nullptr) {
  const int64_t n = int64_t(b.size());
  LinearMethod method = cfg.linear;
  if (method == LinearMethod::auto_select)
    method = n < 600 ? LinearMethod::dense_lu : LinearMethod::gmres;
  Vec x(size_t(n), 0.0);
  if (method == LinearMethod::dense_lu) {
    const Mat M = assemble_dense(A, n);
    const LU f = lu_factor(M);
    x = lu_solve(f, b);
    Vec Ax(static_cast<size_t>(n));
    A(x.data(), Ax.data());
    double defect = 0.0, bmax = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      defect = std::max(defect, std::abs(Ax[size_t(i)] - b[size_t(i)]));
      bmax = std::max(bmax, std::abs(b[size_t(i)]));
    }
    if (!(defect <= 1e-10 * (1.0 + bmax)))
      throw std::runtime_error("linear_solve: direct solve defect exceeds gate");
    return x;
  }
  GmresStats st = gmres(A, b.data(), x.data(), n, cfg.gmres_restart, cfg.gmres_tol,
                        cfg.gmres_max_it);
  if (stats) *stats = st;
  if (!st.converged) throw std::runtime_error("linear_solve: GMRES did not converge");
  return x;
}

struct NewtonResult {
  Vec u;
  int iterations = 0;
  double final_residual = 0.0;
  std::vector<double> residual_history;
  int linear_iterations = 0;
};

inline double max_abs(const Vec& v) {
  double m = 0.0;
  for (double x : v) m = std::max(m, std::abs(x));
  return m;
}

// newton_solve: newton.hpp:102-130.  Full steps; stop when ||res||_inf <=
// abs_tol or <= rel_tol ||res0||_inf.
inline NewtonResult newton_solve(
    const std::function<void(const double*, double*)>& residual,
    const std::function<LinOp(const double*)>& jacobian, const Vec& u0,
    const NewtonConfig& cfg) {
  NewtonResult res;
  res.u = u0;
  const int64_t n = int64_t(u0.size());
  Vec r(static_cast<size_t>(n));
  residual(res.u.data(), r.data());
  double norm = max_abs(r);
  const double norm0 = norm;
  res.residual_history.push_back(norm);
  auto converged = [&](double x) { return x <= cfg.abs_tol || x <= cfg.rel_tol * norm0; };
  while (!converged(norm)) {
    if (res.iterations >= cfg.max_iter)
      throw NonconvergenceError("newton_solve: no convergence", res.u, res.residual_history);
    const LinOp J = jacobian(res.u.data());
    Vec mr(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) mr[size_t(i)] = -r[size_t(i)];
    GmresStats st;
    const Vec du = linear_solve(J, mr, cfg, &st);
    res.linear_iterations += st.iterations;
    for (int64_t i = 0; i < n; ++i) res.u[size_t(i)] += du[size_t(i)];
    ++res.iterations;
    residual(res.u.data(), r.data());
    norm = max_abs(r);
    res.residual_history.push_back(norm);
  }
  res.final_residual = norm;
  return res;
}

// stdg_step: stdg.hpp:120-143 (guess 1 (x) u_n, u_next = last block).
struct StepResult {
  Vec U;
  Vec u_next;
  int newton_iterations = 0;
  int linear_iterations = 0;
};

inline StepResult stdg_step(const System& sys, const Sbp& ops, double t_n,
                            const Vec& u_n, double dt, const NewtonConfig& cfg) {
  if (!(dt > 0)) throw std::invalid_argument("stdg_step: dt > 0 required");
  const int n = ops.n;
  const int64_t dof = sys.dof;
  Vec U0(static_cast<size_t>(n * dof));
  for (int i = 0; i < n; ++i)
    for (int64_t k = 0; k < dof; ++k) U0[size_t(i * dof + k)] = u_n[size_t(k)];
  auto residual = [&](const double* U, double* R) {
    st_residual(sys, ops, t_n, dt, u_n.data(), U, R);
  };
  auto jacobian = [&](const double* U) -> LinOp {
    Vec Ucopy(U, U + n * dof);
    return [&sys, &ops, t_n, dt, Ucopy](const double* v, double* Jv) {
      st_jacobian_apply(sys, ops, t_n, dt, Ucopy.data(), v, Jv);
    };
  };
  NewtonResult nr = newton_solve(residual, jacobian, U0, cfg);
  StepResult r;
  r.u_next.assign(nr.u.begin() + (n - 1) * dof, nr.u.end());
  r.U = std::move(nr.u);
  r.newton_iterations = nr.iterations;
  r.linear_iterations = nr.linear_iterations;
  return r;
}

// rk_step: lodg.hpp:89-149 (Newton on the stage system from 1 (x) u, then
// u_next = u + dt sum_j b_j F(t_j, U_j)).
struct RkResult {
  Vec U;  // stages, stage-major
  Vec u_next;
  int newton_iterations = 0;
  int linear_iterations = 0;
};

inline RkResult rk_step(const System& sys, const Tableau& tab, double t,
                        const Vec& u, double dt, const NewtonConfig& cfg,
                        JacForm form) {
  if (!(dt > 0)) throw std::invalid_argument("rk_step: dt > 0 required");
  const int s = tab.s;
  const int64_t dof = sys.dof;
  Vec U0(static_cast<size_t>(s * dof));
  for (int i = 0; i < s; ++i)
    for (int64_t k = 0; k < dof; ++k) U0[size_t(i * dof + k)] = u[size_t(k)];
  auto residual = [&](const double* U, double* R) {
    stage_residual(sys, tab, t, dt, u.data(), U, form, R);
  };
  auto jacobian = [&](const double* U) -> LinOp {
    Vec Ucopy(U, U + s * dof);
    return [&sys, &tab, t, dt, form, Ucopy](const double* v, double* Jv) {
      stage_jacobian_apply(sys, tab, t, dt, Ucopy.data(), form, v, Jv);
    };
  };
  NewtonResult nr = newton_solve(residual, jacobian, U0, cfg);
  RkResult r;
  r.u_next = u;
  Vec F(static_cast<size_t>(dof));
  for (int j = 0; j < s; ++j) {
    sys.rhs(t + tab.c[j] * dt, nr.u.data() + j * dof, F.data());
    const double c = dt * tab.b[j];
    for (int64_t k = 0; k < dof; ++k) r.u_next[size_t(k)] += c * F[size_t(k)];
  }
  r.U = std::move(nr.u);
  r.newton_iterations = nr.iterations;
  r.linear_iterations = nr.linear_iterations;
  return r;
}

}  // namespace stdg_oracle
