// Device helpers shared by the Krylov kernels (kernels_vec.cu) and the fused
// Arnoldi-update + preconditioner kernel (kernels_fdm.cu): deterministic
// last-block reductions and the on-device Givens step of GMRES.
#pragma once

#include "kernels.hpp"

namespace stg {
namespace {

// max that propagates NaN (fmax drops it): a NaN residual must not read as
// converged (the reference's inf-norm of a NaN vector is NaN)
__device__ __forceinline__ double nan_max(double a, double b) { return (b > a || b != b) ? b : a; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
// Last-block completion: every block publishes its partials, bumps the
// counter, and the block that arrives last finishes the reduction -- in the
// fixed block order, so the result does not depend on arrival order -- and
// resets the counter for the next launch.  Saves one launch per reduction.
__device__ __forceinline__ bool is_last_block(unsigned* counter) {
  __shared__ unsigned last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1 ? 1u : 0u;
  __syncthreads();
  return last != 0u;
}

__device__ __forceinline__ void block_finish_sum(const double* part, int nblocks, int cnt,
                                                 double* out, unsigned* counter) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < cnt; j += nw) {
    // eight independent accumulators: the partial loads of a lane are in
    // flight together (one L2 round trip per 8 instead of per load -- with
    // ~1k blocks the serial version was several microseconds per launch);
    // the summation order is a fixed function of nblocks (deterministic)
    double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int b = lane;
    for (; b + 7 * 32 < nblocks; b += 8 * 32) {
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] += __ldcg(part + (size_t)(b + q * 32) * cnt + j);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (b + q * 32 < nblocks) a[q] += __ldcg(part + (size_t)(b + q * 32) * cnt + j);
    double s = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    s = warp_sum(s);
    if (lane == 0) out[j] = s;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// Arnoldi step k's Givens update (thread 0 of the update pass's last block;
// n2 = ||S_{k+1}||^2 just reduced, sc = the scale this pass applied).  The
// same arithmetic as the host loop it replaces: H(j,k) = c_k c_j d_j with
// c_j = 1/||S_j||, h_{k+1,k} = c_k ||S_{k+1}|| / scale, then the previous
// rotations, a new rotation, and the residual estimate |g_{k+1}|.
constexpr int kGivensLocal = 64;  // restart lengths up to this decide convergence before a 2nd pass
// out[j] = y_j c_j, y = R^-1 g over the first kk columns (one thread; the
// same arithmetic as k_gmres_backsub)
__device__ __forceinline__ void givens_backsub(const GmresDev* G, int kk, double* out) {
  const int m = G->m;
  double y[kInlineBacksub];
  for (int i = kk - 1; i >= 0; --i) {
    double acc = G->g[i];
    for (int j = i + 1; j < kk; ++j) acc -= G->H[i * m + j] * y[j];
    y[i] = acc / G->H[i * m + i];
  }
  for (int j = 0; j < kk; ++j) out[j] = y[j] * G->cn[j];
}

__device__ __noinline__ void gmres_givens(const GivensArgs& a, const double* d, double sc,
                                          const double* hn2, double n2) {
  GmresDev* G = a.G;
  const int m = G->m, k = a.k, kk = k + 1;
  const double* d1 = a.d1;
  const double ckk = G->cn[k];
  double* Hc = G->H;  // column k: Hc[i * m + k]
  double hn;
  if (a.pass == 0) {
    const double ww = d1[kk];
    double hh = 0.0;
    for (int j = 0; j <= k; ++j) hh += d1[j] * d1[j] / hn2[j];
    if (!(ww - hh > G->reorth_tol * ww) || !(n2 > 0.0)) {
      // heavy cancellation.  A nearly exact preconditioner makes A P^-1 v_k
      // almost a combination of the basis, so the step that converges is
      // exactly the one that cancels: decide convergence first, with the
      // exact norm n2 this pass has reduced (accurate to ~eps * ||w|| / ||S||
      // relative; the single pass's orthogonality loss only matters for
      // later steps, and there are none).  Converged: commit the step.
      // Otherwise the host enqueues a second pass for this step.
      if (n2 > 0.0 && ww > 0.0 && k < kGivensLocal) {
        double col[kGivensLocal + 1];
        for (int j = 0; j <= k; ++j) col[j] = ckk * G->cn[j] * d1[j];
        for (int j = 0; j < k; ++j) {
          const double a0 = col[j], a1 = col[j + 1];
          col[j] = G->cs[j] * a0 + G->sn[j] * a1;
          col[j + 1] = -G->sn[j] * a0 + G->cs[j] * a1;
        }
        const double hnt = ckk * sqrt(n2) / sc;
        const double dent = hypot(col[k], hnt);
        const double snt = dent == 0.0 ? 0.0 : hnt / dent;
        if (fabs(snt * G->g[k]) <= G->tol_abs) {
          for (int j = 0; j <= k; ++j) Hc[j * m + k] = col[j];
          const double ct = dent == 0.0 ? 1.0 : col[k] / dent;
          G->cn[kk] = 1.0 / sqrt(n2);
          G->cs[k] = ct;
          G->sn[k] = snt;
          Hc[k * m + k] = dent;
          Hc[kk * m + k] = 0.0;
          const double gk = G->g[k];
          G->g[kk] = -snt * gk;
          G->g[k] = ct * gk;
          G->est = fabs(G->g[kk]);
          G->k_done = kk;
          G->status = 1;
          if (a.ysol && kk <= kInlineBacksub) givens_backsub(G, kk, a.ysol);
          reinterpret_cast<volatile int*>(a.host)[k] = 1;
          __threadfence_system();
          return;
        }
      }
      G->status = 3;
      reinterpret_cast<volatile int*>(a.host)[k] = 3;
      __threadfence_system();
      return;
    }
    for (int j = 0; j <= k; ++j) Hc[j * m + k] = ckk * G->cn[j] * d1[j];
    hn = ckk * sqrt(n2) / sc;
    if (!(ww > 0.0)) hn = 0.0;  // exact breakdown: A P^-1 v_k = 0
  } else {
    const double sc1 = *a.sc1;
    for (int j = 0; j <= k; ++j) Hc[j * m + k] = ckk * G->cn[j] * (d1[j] + d[j] / sc1);
    hn = ckk * sqrt(n2) / (sc1 * sc);
    if (!(d1[kk] > 0.0)) hn = 0.0;
  }
  G->cn[kk] = n2 > 0.0 ? 1.0 / sqrt(n2) : 0.0;
  for (int j = 0; j < k; ++j) {
    const double a0 = Hc[j * m + k], a1 = Hc[(j + 1) * m + k];
    Hc[j * m + k] = G->cs[j] * a0 + G->sn[j] * a1;
    Hc[(j + 1) * m + k] = -G->sn[j] * a0 + G->cs[j] * a1;
  }
  const double hk = Hc[k * m + k];
  const double den = hypot(hk, hn);
  const double c = den == 0.0 ? 1.0 : hk / den;
  const double sn = den == 0.0 ? 0.0 : hn / den;
  G->cs[k] = c;
  G->sn[k] = sn;
  Hc[k * m + k] = den;
  Hc[kk * m + k] = 0.0;
  const double gk = G->g[k];
  G->g[kk] = -sn * gk;
  G->g[k] = c * gk;
  const double est = fabs(G->g[kk]);
  G->est = est;
  G->k_done = kk;
  const int st = est <= G->tol_abs ? 1 : ((hn == 0.0 || !isfinite(hn)) ? 2 : 0);
  G->status = st;
  if (st == 1 && a.ysol && kk <= kInlineBacksub) givens_backsub(G, kk, a.ysol);
  reinterpret_cast<volatile int*>(a.host)[k] = st;
  __threadfence_system();
}

}  // namespace
}  // namespace stg
