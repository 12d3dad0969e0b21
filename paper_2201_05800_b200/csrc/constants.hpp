// Operator constants of the product library, computed on the host in fp64.
//
// The GPU must use D, w and the Lobatto IIIC tableau produced by exactly the
// reference's construction (SURVEY.md §7 "Bit-faithful semantics"); recomputing
// them on the device would round differently.  This follows
//   lgl_rule        quadrature.hpp:66-105
//   lagrange_basis  quadrature.hpp:107-124
//   diff_matrix     quadrature.hpp:128-144
//   lobatto_tableau operators.hpp:76-112
// and tests/test_abi.py (test_constants_bitwise_equal_to_oracle) checks it is
// bitwise equal to the oracle's.
#pragma once

#include <cmath>
#include <stdexcept>
#include <vector>

namespace stg {

struct LglRule {
  int n = 0;
  std::vector<double> x, w;
};

inline void legendre_pair(int m, double x, double& pm, double& pm1) {
  pm = 1.0;
  pm1 = 0.0;
  for (int k = 0; k < m; ++k) {
    const double next = ((2 * k + 1) * x * pm - double(k) * pm1) / double(k + 1);
    pm1 = pm;
    pm = next;
  }
}

inline LglRule lgl(int n) {
  if (n < 2) throw std::invalid_argument("lgl_rule: need n >= 2 nodes");
  LglRule r;
  r.n = n;
  r.x.assign(n, 0.0);
  r.w.assign(n, 0.0);
  r.x[0] = -1.0;
  r.x[n - 1] = 1.0;
  const int m = n - 1;
  const double pi = 3.14159265358979323846;
  for (int i = 1; i < n - 1; ++i) {
    double x = -std::cos(pi * double(i) / double(m));
    for (int it = 0; it < 100; ++it) {  // Newton on P'_m (quadrature.hpp:79-88)
      double pm, pm1;
      legendre_pair(m, x, pm, pm1);
      const double x2m1 = x * x - 1.0;
      const double dp = double(m) * (x * pm - pm1) / x2m1;
      const double ddp = (2.0 * x * dp - double(m * (m + 1)) * pm) / (-x2m1);
      const double dx = dp / ddp;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    r.x[i] = x;
  }
  for (int i = 0; i < n; ++i) {  // exact symmetry (quadrature.hpp:90-99)
    const double sym = (r.x[i] - r.x[n - 1 - i]) / 2.0;
    if (2 * i < n - 1) {
      r.x[i] = sym;
      r.x[n - 1 - i] = -sym;
    } else if (2 * i == n - 1) {
      r.x[i] = 0.0;
    }
  }
  for (int i = 0; i < n; ++i) {
    double pm, pm1;
    legendre_pair(m, r.x[i], pm, pm1);
    r.w[i] = 2.0 / (double(n) * double(m) * pm * pm);
  }
  return r;
}

// D[j*n + i] = psi_i'(x_j), negative-sum diagonal.
inline std::vector<double> diff_matrix(const LglRule& r) {
  const int n = r.n;
  std::vector<double> bw(n);
  for (int i = 0; i < n; ++i) {
    double w = 1.0;
    for (int j = 0; j < n; ++j)
      if (j != i) w *= r.x[i] - r.x[j];
    bw[i] = 1.0 / w;
  }
  double mx = 0.0;
  for (double v : bw) mx = std::max(mx, std::abs(v));
  for (double& v : bw) v /= mx;
  std::vector<double> D(size_t(n) * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double diag = 0.0;
    for (int i = 0; i < n; ++i) {
      if (i == j) continue;
      D[size_t(j) * n + i] = (bw[i] / bw[j]) / (r.x[j] - r.x[i]);
      diag -= D[size_t(j) * n + i];
    }
    D[size_t(j) * n + j] = diag;
  }
  return D;
}

struct Tableau {
  int s = 0;
  std::vector<double> A, b, c;  // A row-major s x s
};

// lobatto_tableau: operators.hpp:76-112 closed forms for s in {2,3,4}; larger
// s via to_butcher (operators.hpp:55-72).
inline Tableau lobatto(int s);

// Small dense inverse with partial pivoting (stand-in for PartialPivLU at
// operators.hpp:59-60 and lodg.hpp:23-29); throws if the a-posteriori defect
// exceeds 1e-10.
inline std::vector<double> inverse(const std::vector<double>& A, int n) {
  std::vector<double> M = A, inv(size_t(n) * n, 0.0);
  for (int i = 0; i < n; ++i) inv[size_t(i) * n + i] = 1.0;
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(M[size_t(i) * n + k]) > std::abs(M[size_t(p) * n + k])) p = i;
    if (M[size_t(p) * n + k] == 0.0) throw std::runtime_error("inverse: singular matrix");
    if (p != k)
      for (int j = 0; j < n; ++j) {
        std::swap(M[size_t(k) * n + j], M[size_t(p) * n + j]);
        std::swap(inv[size_t(k) * n + j], inv[size_t(p) * n + j]);
      }
    const double piv = M[size_t(k) * n + k];
    for (int i = 0; i < n; ++i) {
      if (i == k) continue;
      const double l = M[size_t(i) * n + k] / piv;
      if (l == 0.0) continue;
      for (int j = 0; j < n; ++j) {
        M[size_t(i) * n + j] -= l * M[size_t(k) * n + j];
        inv[size_t(i) * n + j] -= l * inv[size_t(k) * n + j];
      }
    }
  }
  for (int k = 0; k < n; ++k) {
    const double piv = M[size_t(k) * n + k];
    for (int j = 0; j < n; ++j) inv[size_t(k) * n + j] /= piv;
  }
  double defect = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int k = 0; k < n; ++k) s += A[size_t(i) * n + k] * inv[size_t(k) * n + j];
      defect = std::max(defect, std::abs(s - (i == j ? 1.0 : 0.0)));
    }
  if (!(defect <= 1e-10)) throw std::runtime_error("inverse: singular matrix");
  return inv;
}

inline Tableau lobatto(int s) {
  Tableau t;
  t.s = s;
  const double r5 = std::sqrt(5.0);
  switch (s) {
    case 2:
      t.A = {0.5, -0.5, 0.5, 0.5};
      t.b = {0.5, 0.5};
      t.c = {0.0, 1.0};
      return t;
    case 3:
      t.A = {1.0 / 6, -1.0 / 3, 1.0 / 6, 1.0 / 6, 5.0 / 12, -1.0 / 12, 1.0 / 6, 2.0 / 3, 1.0 / 6};
      t.b = {1.0 / 6, 2.0 / 3, 1.0 / 6};
      t.c = {0.0, 0.5, 1.0};
      return t;
    case 4:
      t.A = {1.0 / 12, -r5 / 12, r5 / 12, -1.0 / 12,
             1.0 / 12, 0.25, (10.0 - 7 * r5) / 60, r5 / 60,
             1.0 / 12, (10.0 + 7 * r5) / 60, 0.25, -r5 / 60,
             1.0 / 12, 5.0 / 12, 5.0 / 12, 1.0 / 12};
      t.b = {1.0 / 12, 5.0 / 12, 5.0 / 12, 1.0 / 12};
      t.c = {0.0, 0.5 - r5 / 10, 0.5 + r5 / 10, 1.0};
      return t;
    default: {
      // to_butcher (operators.hpp:55-72): A = (D + M^{-1} e1 e1^T)^{-1} / 2
      if (s < 2) throw std::invalid_argument("lobatto_tableau: s >= 2");
      const LglRule r = lgl(s);
      std::vector<double> K = diff_matrix(r);
      K[0] += 1.0 / r.w[0];
      const std::vector<double> Kinv = inverse(K, s);
      t.A.resize(size_t(s) * s);
      for (size_t i = 0; i < t.A.size(); ++i) t.A[i] = Kinv[i] / 2.0;
      t.b.resize(s);
      t.c.resize(s);
      for (int i = 0; i < s; ++i) {
        t.b[i] = r.w[i] / 2.0;
        t.c[i] = (r.x[i] + 1.0) / 2.0;
      }
      return t;
    }
  }
}

}  // namespace stg
