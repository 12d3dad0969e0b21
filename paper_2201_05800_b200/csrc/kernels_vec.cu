// HBM-bound Krylov vector kernels (GMRES inner products, norms, axpys) with
// deterministic reductions: the grid size is a fixed function of n, every
// block reduces its slice in a fixed order, and the last block to finish (the
// only atomic is its completion counter) sums the block partials in block
// order.  Results are bitwise reproducible run to run.
//
// These replace the vector work inside Eigen::GMRES (newton.hpp:68-77): the
// Arnoldi step is one multi-dot pass ([V^T w, <w,w>]) and one fused
// project + Pythagorean-normalise + norm pass (stg.cpp, gmres).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>

#include "kernels.hpp"
#include "krylov.cuh"

namespace stg {
namespace {

constexpr int kBlock = 256;
constexpr int kMaxGrid = 148 * 8;

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nan_max(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

__global__ void k_fill(double* x, double v, long long n) {
  pdl_entry();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = v;
}
__global__ void k_copy(double* __restrict__ y, const double* __restrict__ x, long long n) {
  pdl_entry();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = x[i];
}
__global__ void k_axpby(double* y, double a, const double* x, double b, long long n) {
  pdl_entry();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], b * y[i]);
}
// one Neumann step of the polynomial preconditioner: y = z + x - q (x may be y)
__global__ void k_poly_step(double* y, const double* __restrict__ z, const double* x,
                            const double* __restrict__ q, long long n, Skip skip) {
  pdl_entry();
  if (skip_now(skip)) return;
  const long long n2 = n >> 1;
  const double2* z2 = reinterpret_cast<const double2*>(z);
  const double2* x2 = reinterpret_cast<const double2*>(x);
  const double2* q2 = reinterpret_cast<const double2*>(q);
  double2* y2 = reinterpret_cast<double2*>(y);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2;
       i += (long long)gridDim.x * blockDim.x) {
    const double2 a = z2[i], b = x2[i], c = q2[i];
    y2[i] = make_double2(a.x + b.x - c.x, a.y + b.y - c.y);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) y[n - 1] = z[n - 1] + x[n - 1] - q[n - 1];
}
__global__ void k_axpy(double* y, double a, const double* x, long long n) {
  pdl_entry();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}
__global__ void k_broadcast(double* __restrict__ U, const double* __restrict__ u, int nb,
                            long long n) {
  pdl_entry();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = u[i];
    for (int j = 0; j < nb; ++j) U[j * n + i] = v;
  }
}
__global__ void k_scale_invsqrt(double* y, const double* x, const double* nrm2, long long n,
                                double sign, int vec2) {
  pdl_entry();
  const double s = sign / sqrt(nrm2[0]);
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (vec2) {  // 16-byte accesses (both vectors 16-byte aligned)
    const double2* x2 = reinterpret_cast<const double2*>(x);
    double2* y2 = reinterpret_cast<double2*>(y);
    for (long long i = i0; i < n / 2; i += stride) {
      const double2 v = __ldcs(x2 + i);
      __stcs(y2 + i, make_double2(v.x * s, v.y * s));
    }
    if (i0 == 0 && (n & 1)) y[n - 1] = x[n - 1] * s;
  } else {
    for (long long i = i0; i < n; i += stride) y[i] = x[i] * s;
  }
}

// ---- multi-vector kernels: thread-per-chunk.  Each thread owns W
// consecutive elements (W = 2: one 16-byte load per vector) in a grid-stride
// loop and walks the basis vectors in groups of 8, so a thread keeps up to 9
// independent loads in flight and every element of every vector is loaded
// exactly once per pass.  Block partials are reduced warp-wise in a fixed
// order; the grid depends only on n, so sums are reproducible.
constexpr int kGroup = 8;
constexpr int kVecBlock = 256;

template <int W>
struct VecT;
template <>
struct VecT<1> {
  using T = double;
  __device__ static T ld(const double* p, long long i) { return __ldcs(p + i); }
  __device__ static void st(double* p, long long i, T v) { __stcs(p + i, v); }
  __device__ static double dot(T a, T b, double acc) { return fma(a, b, acc); }
  __device__ static T axpy(double a, T x, T y) { return fma(a, x, y); }
  __device__ static T scale(T x, double s) { return x * s; }
  __device__ static T zero() { return 0.0; }
};
template <>
struct VecT<2> {
  using T = double2;
  __device__ static T ld(const double* p, long long i) {
    return __ldcs(reinterpret_cast<const double2*>(p) + i);
  }
  __device__ static void st(double* p, long long i, T v) {
    __stcs(reinterpret_cast<double2*>(p) + i, v);
  }
  __device__ static double dot(T a, T b, double acc) { return fma(a.x, b.x, fma(a.y, b.y, acc)); }
  __device__ static T axpy(double a, T x, T y) { return make_double2(fma(a, x.x, y.x), fma(a, x.y, y.y)); }
  __device__ static T scale(T x, double s) { return make_double2(x.x * s, x.y * s); }
  __device__ static T zero() { return make_double2(0.0, 0.0); }
};

// Block-reduce acc[0..cnt) (cnt <= KMAX + 1) into part[blockIdx.x*cnt + j];
// the last block sums the partials into out[0..cnt).
template <int NACC>
__device__ __forceinline__ bool reduce_out(const double (&acc)[NACC], int cnt, double* part,
                                           double* out, unsigned* counter) {
  __shared__ double red[kVecBlock / 32][NACC];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NACC; ++j) {
    if (j < cnt) {
      const double s = warp_sum(acc[j]);
      if (lane == 0) red[wp][j] = s;
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < cnt; j += kVecBlock) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < kVecBlock / 32; ++q) s += red[q][j];
    part[(size_t)blockIdx.x * cnt + j] = s;
  }
  if (!is_last_block(counter)) return false;
  block_finish_sum(part, gridDim.x, cnt, out, counter);
  return true;
}

// out[j] = <V_j, w>, j < k <= KMAX
template <int KMAX, int W>
__global__ void __launch_bounds__(kVecBlock) k_multidot(const double* __restrict__ V,
                                                        long long ldv, int k,
                                                        const double* __restrict__ w,
                                                        long long nw, double* part,
                                                        double* out, unsigned* counter,
                                                        Skip skip) {
  pdl_entry();
  if (skip_now(skip)) return;
  using O = VecT<W>;
  const int kk = KMAX <= kGroup ? KMAX : k;  // KMAX <= 8: instantiated for k == KMAX
  // the last "basis vector" is often w itself (<w,w> in the Arnoldi pass, or
  // a plain norm): use the loaded x instead of reading w twice
  const int self = (V + (long long)(kk - 1) * ldv == w) ? kk - 1 : -1;
  double acc[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) acc[j] = 0.0;
  for (long long i = blockIdx.x * (long long)kVecBlock + threadIdx.x; i < nw;
       i += (long long)gridDim.x * kVecBlock) {
    const typename O::T x = O::ld(w, i);
#pragma unroll
    for (int g = 0; g < KMAX; g += kGroup) {
      if (g < kk) {
        typename O::T v[kGroup];
#pragma unroll
        for (int q = 0; q < kGroup; ++q)
          v[q] = (g + q < KMAX && g + q < kk)
                     ? (g + q == self ? x : O::ld(V + (g + q) * ldv, i))
                     : O::zero();
#pragma unroll
        for (int q = 0; q < kGroup; ++q)
          if (g + q < KMAX) acc[g + q] = O::dot(v[q], x, acc[g + q]);
      }
    }
  }
  reduce_out(acc, kk, part, out, counter);
}

// w = (accumulate ? w : 0) + sign * sum_{j<k} h_j V_j, times s = 1 or the
// Pythagorean scale from scale_src; out[0] = <w_new, w_new> (part may be
// null: no reduction).
template <int KMAX, int W>
__global__ void __launch_bounds__(kVecBlock) k_update(double* __restrict__ w,
                                                      const double* __restrict__ V,
                                                      long long ldv, int k,
                                                      const double* __restrict__ h, long long nw,
                                                      double sign, int accumulate, double* part,
                                                      const double* __restrict__ scale_src,
                                                      double* scale_out, double* out,
                                                      unsigned* counter,
                                                      const double* __restrict__ hn2, Skip skip,
                                                      GivensArgs gv,
                                                      const double* __restrict__ bsrc,
                                                      long long bper) {
  pdl_entry();
  if (skip_now(skip)) return;
  using O = VecT<W>;
  const int kk = KMAX <= kGroup ? KMAX : k;  // KMAX <= 8: instantiated for k == KMAX
  __shared__ double hs[KMAX];
  __shared__ double sc;
  // hn2 (optional) = ||V_j||^2: the basis vectors are stored unnormalised
  // (exact norms tracked instead of a rescaling pass), so the projection
  // coefficient of <V_j, w> is <V_j, w> / ||V_j||^2
  for (int j = threadIdx.x; j < KMAX; j += kVecBlock)
    hs[j] = j < k ? sign * (hn2 ? h[j] / hn2[j] : h[j]) : 0.0;
  if (threadIdx.x == 0) {
    // scale_src = [h_0..h_{k-1}, <w,w>]: normalise by the Pythagorean norm
    // sqrt(<w,w> - sum h_j^2 / ||V_j||^2) of the projected vector (fallback: ||w||)
    double s = 1.0;
    if (scale_src) {
      const double ww = scale_src[k];
      double hh = 0.0;
      for (int j = 0; j < k; ++j)
        hh = fma(scale_src[j], hn2 ? scale_src[j] / hn2[j] : scale_src[j], hh);
      const double est = ww - hh;
      s = est > 1e-28 * ww ? 1.0 / sqrt(est) : (ww > 0.0 ? 1.0 / sqrt(ww) : 1.0);
      if (scale_out && blockIdx.x == 0) scale_out[0] = s;
    }
    sc = s;
  }
  __syncthreads();
  const double s = sc;
  double hr[KMAX];  // registers: a generic store to w could alias hs
#pragma unroll
  for (int j = 0; j < KMAX; ++j) hr[j] = hs[j];
  double acc[1] = {0.0};
  for (long long i = blockIdx.x * (long long)kVecBlock + threadIdx.x; i < nw;
       i += (long long)gridDim.x * kVecBlock) {
    // accumulate 2: the old w is bsrc repeated with period bper (the lazy
    // initial guess 1 (x) u_n, never written out)
    // accumulate 3: as 1, but the result is only reduced, not stored (the
    // step is expected to converge: its new basis vector is never read)
    typename O::T x = (accumulate & 1)  ? O::ld(w, i)
                      : accumulate == 2 ? O::ld(bsrc, i % bper)
                                        : O::zero();
#pragma unroll
    for (int g = 0; g < KMAX; g += kGroup) {
      if (g < kk) {
        typename O::T v[kGroup];
#pragma unroll
        for (int q = 0; q < kGroup; ++q)
          v[q] = (g + q < KMAX && g + q < kk) ? O::ld(V + (g + q) * ldv, i) : O::zero();
#pragma unroll
        for (int q = 0; q < kGroup; ++q)
          if (g + q < KMAX) x = O::axpy(hr[g + q], v[q], x);
      }
    }
    x = O::scale(x, s);
    if (accumulate != 3) O::st(w, i, x);
    acc[0] = O::dot(x, x, acc[0]);
  }
  if (part == nullptr) return;
  if (reduce_out(acc, 1, part, out, counter) && gv.G && threadIdx.x == 0)
    gmres_givens(gv, scale_src, s, hn2, out[0]);
}

__global__ void k_gmres_init(GmresDev* G, int m, const double* bb, double beta, double tol,
                             double reorth_tol, double* hn2_0, int* host, double s0_sign) {
  pdl_entry();
  double tol_abs = tol;
  if (bb) {  // first cycle from x = 0: ||r|| = ||b|| is only known here
    beta = sqrt(*bb);
    G->bnorm = beta;
    tol_abs = tol * beta;
  }
  G->m = m;
  G->status = 0;
  // b = 0: nothing to do (4).  A NaN / infinite ||r|| is a failure (5), not
  // "b = 0": the reference's Eigen GMRES does not converge on it and
  // linear_solve throws (newton.hpp:74-76).  Every step slot reads the status.
  const int st0 = beta == 0.0 ? 4 : (!(beta > 0.0) || isinf(beta) ? 5 : 0);
  if (st0 != 0) {
    G->status = st0;
    for (int j = 0; j <= m; ++j) reinterpret_cast<volatile int*>(host)[j] = st0;
    __threadfence_system();
  }
  G->k_done = 0;
  G->est = beta;
  G->tol_abs = tol_abs;
  G->reorth_tol = reorth_tol;
  G->g[0] = beta;
  for (int j = 1; j <= m; ++j) G->g[j] = 0.0;
  G->cn[0] = 1.0;
  if (hn2_0) *hn2_0 = 1.0;  // ||S_0||^2 = 1 (S_0 = r / ||r||)
  if (s0_sign != 0.0 && beta > 0.0) {  // S_0 = b unnormalised; the sign rides on g_0
    G->g[0] = s0_sign * beta;
    G->cn[0] = 1.0 / beta;
    if (hn2_0) *hn2_0 = beta * beta;
  }
}

__device__ __forceinline__ double fd_step(const double* vv, const double* uu, double c) {
  const double e = uu ? c * sqrt(1.0 + sqrt(*uu)) : c;
  return *vv > 0.0 ? e / sqrt(*vv) : 1.0;
}
__global__ void k_fd_pm(double* __restrict__ Up, double* __restrict__ Um,
                        const double* __restrict__ U, const double* __restrict__ v, long long n,
                        const double* vv, const double* uu, double c, Skip skip) {
  pdl_entry();
  if (skip_now(skip)) return;
  const double e = fd_step(vv, uu, c);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double u = U[i], d = e * v[i];
    Up[i] = u + d;
    Um[i] = u - d;
  }
}
__global__ void k_fd_diff(double* __restrict__ Jv, const double* __restrict__ Fm, long long n,
                          const double* vv, const double* uu, double c, Skip skip) {
  pdl_entry();
  if (skip_now(skip)) return;
  const double h = 0.5 / fd_step(vv, uu, c);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    Jv[i] = (Jv[i] - Fm[i]) * h;
}

// y = R^-1 g over the first k Givens-reduced Hessenberg columns, scaled by
// the basis norms (out[j] = y_j c_j: x += sum out_j S_j), k <= 60.  The
// block stages R's upper triangle, g and c in shared memory (independent
// loads), then one thread substitutes from there.
__global__ void __launch_bounds__(128) k_gmres_backsub(const GmresDev* G, int k, double* out) {
  pdl_entry();
  __shared__ double Rs[kGmresMaxRestart * kGmresMaxRestart];
  __shared__ double gs[kGmresMaxRestart], cs[kGmresMaxRestart], y[kGmresMaxRestart];
  const int m = G->m;
  for (int q = threadIdx.x; q < k * k; q += blockDim.x) {
    const int i = q / k, j = q - i * k;
    if (j >= i) Rs[q] = G->H[i * m + j];
  }
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    gs[j] = G->g[j];
    cs[j] = G->cn[j];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int i = k - 1; i >= 0; --i) {
    double acc = gs[i];
    for (int j = i + 1; j < k; ++j) acc -= Rs[i * k + j] * y[j];
    y[i] = acc / Rs[i * k + i];
  }
  for (int j = 0; j < k; ++j) out[j] = y[j] * cs[j];
}

__global__ void __launch_bounds__(kBlock) k_maxabs(const double* __restrict__ x, long long n,
                                                   double* part, double* out,
                                                   unsigned* counter) {
  pdl_entry();
  __shared__ double red[kBlock / 32];
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    m = nan_max(m, fabs(x[i]));
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < kBlock / 32; ++w) r = nan_max(r, red[w]);
    part[blockIdx.x] = r;
  }
  if (is_last_block(counter) && threadIdx.x < 32) {
    double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // 8 loads in flight per lane
    int b = threadIdx.x;
    for (; b + 7 * 32 < (int)gridDim.x; b += 8 * 32) {
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = nan_max(a[q], __ldcg(part + b + q * 32));
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (b + q * 32 < (int)gridDim.x) a[q] = nan_max(a[q], __ldcg(part + b + q * 32));
    double r = nan_max(nan_max(nan_max(a[0], a[1]), nan_max(a[2], a[3])),
                       nan_max(nan_max(a[4], a[5]), nan_max(a[6], a[7])));
    r = warp_max(r);
    if (threadIdx.x == 0) {
      out[0] = r;
      *counter = 0u;
    }
  }
}

int grid_for(long long n) {
  long long g = (n + kBlock - 1) / kBlock;
  if (g < 1) g = 1;
  if (g > kMaxGrid) g = kMaxGrid;
  return int(g);
}

}  // namespace

// The completion counter lives right after the partial-sum area (see
// kPartialDoubles in kernels.hpp); it is zero between launches.
unsigned* counter_of(double* partial) {
  return reinterpret_cast<unsigned*>(partial + kPartialDoubles);
}

int reduce_grid(long long n) { return grid_for(n); }

// Vector kernels use PDL only below 4 Mi elements: there the launch latency
// it hides is a large share of the kernel; on the 64 MiB c4 vectors it
// measured slower (c4 solve 2.09 -> 2.20 ms, c3 8.2 -> 7.9 ms with it on)
int vec_pdl(long long n) { return n < (4LL << 20) ? kPdlVec : 0; }

bool pdl_enabled(int cls) {
  static const int mask = [] {
    if (std::getenv("STG_NO_PDL")) return 0;
    const char* e = std::getenv("STG_PDL_MASK");
    return e ? std::atoi(e) : kPdlSlab | kPdlFdm | kPdlVec | kPdlPrecond;
  }();
  return (mask & cls) != 0;
}

void vec_fill(double* x, double v, long long n, cudaStream_t s) {
  launch_ex(vec_pdl(n), k_fill, grid_for(n), kBlock, 0, s, x, v, n);
}
void vec_copy(double* y, const double* x, long long n, cudaStream_t s) {
  launch_ex(vec_pdl(n), k_copy, grid_for(n), kBlock, 0, s, y, x, n);
}
void vec_axpy(double* y, double a, const double* x, long long n, cudaStream_t s) {
  launch_ex(vec_pdl(n), k_axpy, grid_for(n), kBlock, 0, s, y, a, x, n);
}
void vec_axpby(double* y, double a, const double* x, double b, long long n, cudaStream_t s) {
  launch_ex(vec_pdl(n), k_axpby, grid_for(n), kBlock, 0, s, y, a, x, b, n);
}
void vec_poly_step(double* y, const double* z, const double* x, const double* q, long long n,
                   cudaStream_t s, Skip skip) {
  launch_ex(vec_pdl(n), k_poly_step, grid_for(n / 2 + 1), kBlock, 0, s, y, z, x, q, n, skip);
}
void vec_broadcast(double* U, const double* u, int nb, long long n, cudaStream_t s) {
  launch_ex(vec_pdl(n), k_broadcast, grid_for(n), kBlock, 0, s, U, u, nb, n);
}
void vec_scale_invsqrt(double* y, const double* x, const double* nrm2, long long n,
                       cudaStream_t s, double sign) {
  const int v2 = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
  launch_ex(vec_pdl(n), k_scale_invsqrt, grid_for(v2 ? n / 2 + 1 : n), kBlock, 0, s, y, x, nrm2,
            n, sign, v2);
}

namespace {

// Grid: enough blocks to fill every SM to the kernel's occupancy (so the
// loads in flight cover HBM latency at small k), fewer for short vectors.
// A fixed function of (n, kernel): reductions stay reproducible.  One cache
// per instantiation; at most kPartialDoubles / 80 blocks.
template <int KM, int WW, bool UPD>
int multi_grid(long long n) {
  static int cap_dev[kMaxDevices];
  const int dev = device_slot();
  int& cap = cap_dev[dev];
  if (cap == 0) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (UPD)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_update<KM, WW>, kVecBlock, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_multidot<KM, WW>, kVecBlock, 0);
    cap = std::max(1, std::min(per_sm * sms, int(kPartialDoubles / 80)));
  }
  long long g = (n / WW + kVecBlock - 1) / kVecBlock;
  return int(std::max(1LL, std::min(g, (long long)cap)));
}


bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// W = 2 (16-byte accesses) when n, ldv and every base pointer allow it
int vec_width(long long n, long long ldv, const void* a, const void* b) {
  return (n % 2 == 0 && ldv % 2 == 0 && aligned16(a) && aligned16(b)) ? 2 : 1;
}

// k <= 8: exact-k instantiations (no predicated lanes in the loop); above:
// runtime k up to KMAX = 16, 32, 64
#define STG_KSWITCH(k, CALL)                                 \
  switch (k) {                                               \
    case 1: { constexpr int KM = 1; CALL; } break;           \
    case 2: { constexpr int KM = 2; CALL; } break;           \
    case 3: { constexpr int KM = 3; CALL; } break;           \
    case 4: { constexpr int KM = 4; CALL; } break;           \
    case 5: { constexpr int KM = 5; CALL; } break;           \
    case 6: { constexpr int KM = 6; CALL; } break;           \
    case 7: { constexpr int KM = 7; CALL; } break;           \
    case 8: { constexpr int KM = 8; CALL; } break;           \
    default:                                                 \
      if ((k) <= 16) { constexpr int KM = 16; CALL; }        \
      else if ((k) <= 32) { constexpr int KM = 32; CALL; }   \
      else { constexpr int KM = 64; CALL; }                  \
  }

#define STG_DISPATCH_K(k, W, CALL)                                                \
  do {                                                                            \
    if ((k) < 1 || (k) > 64) throw std::invalid_argument("multi-vector kernels: 1 <= k <= 64"); \
    if ((W) == 2) {                                                               \
      constexpr int WW = 2;                                                       \
      STG_KSWITCH(k, CALL)                                                        \
    } else {                                                                      \
      constexpr int WW = 1;                                                       \
      STG_KSWITCH(k, CALL)                                                        \
    }                                                                             \
  } while (0)

}  // namespace

void vec_multidot(const double* V, long long ldv, int k, const double* w, long long n,
                  double* partial, double* out, cudaStream_t s, Skip skip) {
  const int W = vec_width(n, ldv, V, w);
  unsigned* c = counter_of(partial);
  STG_DISPATCH_K(k, W, (launch_ex(vec_pdl(n), k_multidot<KM, WW>, multi_grid<KM, WW, false>(n), kVecBlock,
                                              0, s, V, ldv, k, w, n / WW, partial, out, c,
                                                      skip)));
}

void vec_fd_pm(double* Up, double* Um, const double* U, const double* v, long long n,
               const double* vv, const double* uu, double c, cudaStream_t s, Skip skip) {
  launch_ex(vec_pdl(n), k_fd_pm, grid_for(n), kBlock, 0, s, Up, Um, U, v, n, vv, uu, c, skip);
}
void vec_fd_diff(double* Jv, const double* Fm, long long n, const double* vv, const double* uu,
                 double c, cudaStream_t s, Skip skip) {
  launch_ex(vec_pdl(n), k_fd_diff, grid_for(n), kBlock, 0, s, Jv, Fm, n, vv, uu, c, skip);
}

void gmres_backsub(const GmresDev* G, int k, double* out, cudaStream_t s) {
  launch_ex(kPdlVec, k_gmres_backsub, 1, 128, 0, s, G, k, out);
}

void gmres_init(GmresDev* G, int m, const double* bb, double beta, double tol, double reorth_tol,
                double* hn2_0, int* host, cudaStream_t s, double s0_sign) {
  launch_ex(kPdlVec, k_gmres_init, 1, 1, 0, s, G, m, bb, beta, tol, reorth_tol, hn2_0, host,
            s0_sign);
}

void vec_update_dot(double* w, const double* V, long long ldv, int k, const double* h,
                    long long n, int want_dots, double* partial, double* out2, cudaStream_t s,
                    const double* scale_src, double* scale_out, const double* hn2, Skip skip,
                    GivensArgs gv, bool norm_only) {
  const int W = vec_width(n, ldv, V, w);
  unsigned* c = counter_of(partial);
  STG_DISPATCH_K(k, W, (launch_ex(vec_pdl(n), k_update<KM, WW>, multi_grid<KM, WW, true>(n), kVecBlock, 0, s, 
                           w, V, ldv, k, h, n / WW, -1.0, norm_only ? 3 : 1, partial, scale_src, scale_out,
                           out2 + k, c, hn2, skip, gv, nullptr, 1LL)));
  if (want_dots) vec_multidot(V, ldv, k, w, n, partial, out2, s, skip);  // <V_j, w_new>
}

void vec_combine(double* x, const double* V, long long ldv, int k, const double* y, long long n,
                 cudaStream_t s, bool accumulate, const double* bsrc, long long bper) {
  if (k == 0) {
    if (bsrc) vec_broadcast(x, bsrc, int(n / bper), bper, s);
    else if (!accumulate) vec_fill(x, 0.0, n, s);
    return;
  }
  int W = vec_width(n, ldv, V, x);
  if (bsrc && (bper % 2 != 0 || !aligned16(bsrc))) W = 1;
  const int mode = bsrc ? 2 : (accumulate ? 1 : 0);
  STG_DISPATCH_K(k, W, (launch_ex(vec_pdl(n), k_update<KM, WW>, multi_grid<KM, WW, true>(n), kVecBlock, 0, s, 
                           x, V, ldv, k, y, n / WW, 1.0, mode, nullptr, nullptr,
                           nullptr, nullptr, nullptr, nullptr, Skip{}, GivensArgs{}, bsrc,
                           bper / WW)));
}

void vec_maxabs(const double* x, long long n, double* partial, double* out, cudaStream_t s) {
  const int g = grid_for(n);
  launch_ex(vec_pdl(n), k_maxabs, g, kBlock, 0, s, x, n, partial, out, counter_of(partial));
}

void vec_dot(const double* x, const double* y, long long n, double* partial, double* out,
             cudaStream_t s, Skip skip) {
  vec_multidot(x, 0, 1, y, n, partial, out, s, skip);
}

}  // namespace stg
