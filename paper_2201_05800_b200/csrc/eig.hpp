// Small dense complex eigen-decomposition (host, fp64) for the fast-
// diagonalisation element-block preconditioner: M = P diag(lam) P^-1 for a real
// n x n matrix (n <= 8) with distinct eigenvalues.  No LAPACK in this image:
//   characteristic polynomial  Faddeev-LeVerrier recursion
//   eigenvalues                Aberth-Ehrlich simultaneous iteration
//   eigenvectors               two steps of inverse iteration with complex LU
// Complex-conjugate pairs are returned adjacently, (lam, conj(lam)), with
// eigenvector columns that are exact conjugates of each other; callers verify
// the reconstruction and fall back when it is not accurate.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <vector>

namespace stg {

using cplx = std::complex<double>;

// x = A^{-1} b for a small complex matrix (partial pivoting); returns false if singular
inline bool csolve(std::vector<cplx> A, std::vector<cplx>& b, int n) {
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(A[size_t(i) * n + k]) > std::abs(A[size_t(p) * n + k])) p = i;
    if (std::abs(A[size_t(p) * n + k]) == 0.0) return false;
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(A[size_t(k) * n + j], A[size_t(p) * n + j]);
      std::swap(b[size_t(k)], b[size_t(p)]);
    }
    for (int i = k + 1; i < n; ++i) {
      const cplx l = A[size_t(i) * n + k] / A[size_t(k) * n + k];
      for (int j = k; j < n; ++j) A[size_t(i) * n + j] -= l * A[size_t(k) * n + j];
      b[size_t(i)] -= l * b[size_t(k)];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    cplx s = b[size_t(i)];
    for (int j = i + 1; j < n; ++j) s -= A[size_t(i) * n + j] * b[size_t(j)];
    b[size_t(i)] = s / A[size_t(i) * n + i];
  }
  return true;
}

inline bool cinverse(const std::vector<cplx>& A, std::vector<cplx>& inv, int n) {
  inv.assign(size_t(n) * n, 0.0);
  for (int c = 0; c < n; ++c) {
    std::vector<cplx> e(size_t(n), 0.0);
    e[size_t(c)] = 1.0;
    if (!csolve(A, e, n)) return false;
    for (int r = 0; r < n; ++r) inv[size_t(r) * n + c] = e[size_t(r)];
  }
  return true;
}

// M (row-major, real n x n) = P diag(lam) Pinv.  Returns false if the
// eigenvalues are not distinct or the reconstruction error exceeds tol.
inline bool eig_real(const std::vector<double>& M, int n, std::vector<cplx>& lam,
                     std::vector<cplx>& P, std::vector<cplx>& Pinv, double tol = 1e-11) {
  // Faddeev-LeVerrier: det(x I - M) = x^n + c[1] x^{n-1} + ... + c[n]
  std::vector<double> c(size_t(n) + 1, 0.0), Mk(size_t(n) * n, 0.0), AM(size_t(n) * n);
  c[0] = 1.0;
  for (int k = 1; k <= n; ++k) {
    // Mk = M * (M_{k-1} + c_{k-1} I), starting from M_0 = 0
    std::vector<double> B = Mk;
    for (int i = 0; i < n; ++i) B[size_t(i) * n + i] += c[size_t(k - 1)];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int q = 0; q < n; ++q) s += M[size_t(i) * n + q] * B[size_t(q) * n + j];
        AM[size_t(i) * n + j] = s;
      }
    double tr = 0.0;
    for (int i = 0; i < n; ++i) tr += AM[size_t(i) * n + i];
    c[size_t(k)] = -tr / k;
    Mk = AM;
  }
  auto poly = [&](cplx x, cplx& dp) {
    cplx p = 1.0;
    dp = 0.0;
    for (int k = 1; k <= n; ++k) {
      dp = dp * x + p;
      p = p * x + c[size_t(k)];
    }
    return p;
  };
  // Aberth-Ehrlich from points on a circle of radius ~ max |coefficient|^(1/k)
  double rad = 0.0;
  for (int k = 1; k <= n; ++k) rad = std::max(rad, std::pow(std::abs(c[size_t(k)]), 1.0 / k));
  rad = std::max(rad, 1e-300);
  lam.assign(size_t(n), 0.0);
  for (int i = 0; i < n; ++i)
    lam[size_t(i)] = std::polar(rad, 2.0 * M_PI * (i + 0.25) / n + 0.4);
  for (int it = 0; it < 500; ++it) {
    double worst = 0.0;
    for (int i = 0; i < n; ++i) {
      cplx dp;
      const cplx p = poly(lam[size_t(i)], dp);
      const cplx ratio = p / dp;
      cplx s = 0.0;
      for (int j = 0; j < n; ++j)
        if (j != i) s += 1.0 / (lam[size_t(i)] - lam[size_t(j)]);
      const cplx step = ratio / (1.0 - ratio * s);
      lam[size_t(i)] -= step;
      worst = std::max(worst, std::abs(step) / std::max(1.0, std::abs(lam[size_t(i)])));
    }
    if (worst < 1e-15) break;
  }
  // polish each root with Newton on the polynomial
  for (int i = 0; i < n; ++i)
    for (int it = 0; it < 3; ++it) {
      cplx dp;
      const cplx p = poly(lam[size_t(i)], dp);
      if (std::abs(dp) > 0.0) lam[size_t(i)] -= p / dp;
    }
  // pair conjugates: (lam, conj(lam)) with Im(lam) > 0 first; real roots stay single
  std::vector<cplx> sorted;
  std::vector<bool> used(size_t(n), false);
  const double scale = std::max(1.0, rad);
  for (int i = 0; i < n; ++i) {
    if (used[size_t(i)]) continue;
    used[size_t(i)] = true;
    if (std::abs(lam[size_t(i)].imag()) <= 1e-12 * scale) {
      sorted.push_back(cplx(lam[size_t(i)].real(), 0.0));
      continue;
    }
    int best = -1;
    double bd = 1e300;
    for (int j = 0; j < n; ++j)
      if (!used[size_t(j)]) {
        const double dd = std::abs(lam[size_t(j)] - std::conj(lam[size_t(i)]));
        if (dd < bd) {
          bd = dd;
          best = j;
        }
      }
    if (best < 0) return false;
    used[size_t(best)] = true;
    cplx a = 0.5 * (lam[size_t(i)] + std::conj(lam[size_t(best)]));
    if (a.imag() < 0) a = std::conj(a);
    sorted.push_back(a);
    sorted.push_back(std::conj(a));
  }
  lam = sorted;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      if (std::abs(lam[size_t(i)] - lam[size_t(j)]) < 1e-9 * scale) return false;  // repeated
  // eigenvectors by inverse iteration
  P.assign(size_t(n) * n, 0.0);
  for (int i = 0; i < n; ++i) {
    if (i > 0 && lam[size_t(i)].imag() < 0 && lam[size_t(i)] == std::conj(lam[size_t(i - 1)])) {
      for (int r = 0; r < n; ++r) P[size_t(r) * n + i] = std::conj(P[size_t(r) * n + i - 1]);
      continue;
    }
    const cplx shift = lam[size_t(i)] * (1.0 + 1e-13) + 1e-14 * scale;
    std::vector<cplx> A(size_t(n) * n);
    for (int r = 0; r < n; ++r)
      for (int q = 0; q < n; ++q)
        A[size_t(r) * n + q] = M[size_t(r) * n + q] - (r == q ? shift : cplx(0.0));
    std::vector<cplx> v(static_cast<size_t>(n));
    for (int r = 0; r < n; ++r) v[size_t(r)] = cplx(1.0 + 0.1 * r, 0.3 - 0.05 * r);
    for (int it = 0; it < 3; ++it) {
      if (!csolve(A, v, n)) return false;
      double nrm = 0.0;
      for (const cplx& z : v) nrm += std::norm(z);
      nrm = std::sqrt(nrm);
      for (cplx& z : v) z /= nrm;
    }
    for (int r = 0; r < n; ++r) P[size_t(r) * n + i] = v[size_t(r)];
  }
  if (!cinverse(P, Pinv, n)) return false;
  // verify M = P diag(lam) Pinv
  double err = 0.0, mx = 0.0;
  for (int r = 0; r < n; ++r)
    for (int q = 0; q < n; ++q) {
      cplx s = 0.0;
      for (int k = 0; k < n; ++k) s += P[size_t(r) * n + k] * lam[size_t(k)] * Pinv[size_t(k) * n + q];
      err = std::max(err, std::abs(s - M[size_t(r) * n + q]));
      mx = std::max(mx, std::abs(M[size_t(r) * n + q]));
    }
  return err <= tol * std::max(mx, 1e-300);
}

}  // namespace stg
