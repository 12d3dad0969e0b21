// HBM-bound Krylov vector kernels (GMRES inner products, norms, axpys) with
// deterministic reductions: the grid size is a fixed function of n, every
// block reduces its slice in a fixed order, and a single block finishes the
// reduction in a fixed order.  No atomics, so results are bitwise
// reproducible run to run.
//
// These replace the vector work inside Eigen::GMRES (newton.hpp:68-77) with a
// classical Gram-Schmidt Arnoldi whose passes are fused: one multi-dot pass,
// one "update + re-dot" pass (CGS2), one "update + norm" pass.
#include "kernels.hpp"

namespace stg {
namespace {

constexpr int kBlock = 256;
constexpr int kMaxGrid = 148 * 8;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
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
    double s = 0.0;
    for (int b = lane; b < nblocks; b += 32) s += __ldcg(part + (size_t)b * cnt + j);
    s = warp_sum(s);
    if (lane == 0) out[j] = s;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

__global__ void k_fill(double* x, double v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = v;
}
__global__ void k_copy(double* __restrict__ y, const double* __restrict__ x, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = x[i];
}
__global__ void k_axpby(double* y, double a, const double* x, double b, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], b * y[i]);
}
__global__ void k_axpy(double* y, double a, const double* x, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}
__global__ void k_broadcast(double* __restrict__ U, const double* __restrict__ u, int nb,
                            long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = u[i];
    for (int j = 0; j < nb; ++j) U[j * n + i] = v;
  }
}
__global__ void k_scale_invsqrt(double* y, const double* x, const double* nrm2, long long n) {
  const double s = 1.0 / sqrt(nrm2[0]);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = x[i] * s;
}

// ---- multi-vector kernels: block = 8 warps x 32 lanes.  Warp g owns basis
// vectors j = g, g+8, g+16, ... (MPW of them); per iteration the block covers
// kU = 8 slots of 32 consecutive elements (lane l of slot u owns element
// base + 32u + l), so every thread keeps MPW*kU independent loads in flight.
// Every V_j entry is loaded once per pass and kept in a register for the
// second half of a fused pass; the cross-warp sum of slot u is done by warp u
// (balanced), in a fixed order.
constexpr int kWarps = 8;
constexpr int kMultiBlock = 32 * kWarps;
constexpr int kU = 8;
constexpr int kTile = 32 * kU;

int multi_grid(long long n) {
  long long g = (n + kTile - 1) / kTile;
  if (g < 1) g = 1;
  if (g > 148 * 4) g = 148 * 4;
  return int(g);
}

// part[b*k + j] = block partial of <V_j, w>
template <int MPW>
__global__ void __launch_bounds__(kMultiBlock) k_multidot(const double* __restrict__ V,
                                                          long long ldv, int k,
                                                          const double* __restrict__ w,
                                                          long long n, double* part,
                                                          double* out, unsigned* counter) {
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  double acc[MPW];
#pragma unroll
  for (int m = 0; m < MPW; ++m) acc[m] = 0.0;
  for (long long base = (long long)blockIdx.x * kTile; base < n;
       base += (long long)gridDim.x * kTile) {
    double wv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long i = base + 32 * u + lane;
      wv[u] = i < n ? w[i] : 0.0;
    }
#pragma unroll
    for (int m = 0; m < MPW; ++m) {
      const int j = g + kWarps * m;
      if (j < k) {
        const double* Vj = V + j * ldv;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const long long i = base + 32 * u + lane;
          if (i < n) acc[m] = fma(Vj[i], wv[u], acc[m]);
        }
      }
    }
  }
#pragma unroll
  for (int m = 0; m < MPW; ++m) {
    const int j = g + kWarps * m;
    const double s = warp_sum(acc[m]);
    if (lane == 0 && j < k) part[(size_t)blockIdx.x * k + j] = s;
  }
  if (is_last_block(counter)) block_finish_sum(part, gridDim.x, k, out, counter);
}

// w += sign * sum_j h_j V_j; optionally dots <V_j, w_new>; always <w_new, w_new>.
// part[b*(k+1) + j], j < k dots (0 if !dots), j = k norm^2 (part may be null).
template <int MPW>
__global__ void __launch_bounds__(kMultiBlock) k_update(double* __restrict__ w,
                                                        const double* __restrict__ V,
                                                        long long ldv, int k,
                                                        const double* __restrict__ h,
                                                        long long n, int dots, double sign,
                                                        double* part,
                                                        const double* __restrict__ scale_src,
                                                        double* scale_out, double* out,
                                                        unsigned* counter) {
  __shared__ double red[kWarps][kU][32];
  __shared__ double wnew[kU][32];
  __shared__ double hs[kWarps * MPW];
  __shared__ double sc;
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  for (int j = threadIdx.x; j < kWarps * MPW; j += blockDim.x) hs[j] = j < k ? h[j] : 0.0;
  if (threadIdx.x == 0) {
    // scale_src = [h_0..h_{k-1}, <w,w>]: normalise by the Pythagorean norm
    // sqrt(<w,w> - sum h_j^2) of the projected vector (fallback: ||w||)
    double s = 1.0;
    if (scale_src) {
      const double ww = scale_src[k];
      double hh = 0.0;
      for (int j = 0; j < k; ++j) hh = fma(scale_src[j], scale_src[j], hh);
      const double est = ww - hh;
      s = est > 1e-28 * ww ? 1.0 / sqrt(est) : (ww > 0.0 ? 1.0 / sqrt(ww) : 1.0);
      if (scale_out && blockIdx.x == 0) scale_out[0] = s;
    }
    sc = s;
  }
  __syncthreads();
  const double s = sc;
  double acc[MPW];
#pragma unroll
  for (int m = 0; m < MPW; ++m) acc[m] = 0.0;
  double nrm = 0.0;
  for (long long base = (long long)blockIdx.x * kTile; base < n;
       base += (long long)gridDim.x * kTile) {
    double v[MPW][kU];
    double p[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) p[u] = 0.0;
#pragma unroll
    for (int m = 0; m < MPW; ++m) {
      const int j = g + kWarps * m;
      const double hj = hs[j];
      const double* Vj = V + j * ldv;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const long long i = base + 32 * u + lane;
        v[m][u] = (j < k && i < n) ? Vj[i] : 0.0;
        p[u] = fma(hj, v[m][u], p[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) red[g][u][lane] = p[u];
    __syncthreads();
    {
      // warp g finishes slot u = g
      const long long i = base + 32 * g + lane;
      double sum = 0.0;
#pragma unroll
      for (int q = 0; q < kWarps; ++q) sum += red[q][g][lane];
      double wi = 0.0;
      if (i < n) {
        wi = fma(sign, sum, w[i]) * s;
        w[i] = wi;
      }
      wnew[g][lane] = wi;
      nrm = fma(wi, wi, nrm);
    }
    __syncthreads();
    if (dots) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const double wi = wnew[u][lane];
#pragma unroll
        for (int m = 0; m < MPW; ++m) acc[m] = fma(v[m][u], wi, acc[m]);
      }
    }
  }
  if (part == nullptr) return;
  __shared__ double nr[kWarps];
#pragma unroll
  for (int m = 0; m < MPW; ++m) {
    const int j = g + kWarps * m;
    const double s = warp_sum(acc[m]);
    if (lane == 0 && j < k) part[(size_t)blockIdx.x * (k + 1) + j] = dots ? s : 0.0;
  }
  const double sn = warp_sum(nrm);
  if (lane == 0) nr[g] = sn;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < kWarps; ++q) t += nr[q];
    part[(size_t)blockIdx.x * (k + 1) + k] = t;
  }
  if (is_last_block(counter)) block_finish_sum(part, gridDim.x, k + 1, out, counter);
}

__global__ void __launch_bounds__(kBlock) k_maxabs(const double* __restrict__ x, long long n,
                                                   double* part, double* out,
                                                   unsigned* counter) {
  __shared__ double red[kBlock / 32];
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    m = fmax(m, fabs(x[i]));
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < kBlock / 32; ++w) r = fmax(r, red[w]);
    part[blockIdx.x] = r;
  }
  if (is_last_block(counter) && threadIdx.x < 32) {
    double r = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) r = fmax(r, __ldcg(part + b));
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

int reduce_grid(long long n) { return grid_for(n); }

void vec_fill(double* x, double v, long long n, cudaStream_t s) {
  k_fill<<<grid_for(n), kBlock, 0, s>>>(x, v, n);
}
void vec_copy(double* y, const double* x, long long n, cudaStream_t s) {
  k_copy<<<grid_for(n), kBlock, 0, s>>>(y, x, n);
}
void vec_axpy(double* y, double a, const double* x, long long n, cudaStream_t s) {
  k_axpy<<<grid_for(n), kBlock, 0, s>>>(y, a, x, n);
}
void vec_axpby(double* y, double a, const double* x, double b, long long n, cudaStream_t s) {
  k_axpby<<<grid_for(n), kBlock, 0, s>>>(y, a, x, b, n);
}
void vec_broadcast(double* U, const double* u, int nb, long long n, cudaStream_t s) {
  k_broadcast<<<grid_for(n), kBlock, 0, s>>>(U, u, nb, n);
}
void vec_scale_invsqrt(double* y, const double* x, const double* nrm2, long long n,
                       cudaStream_t s) {
  k_scale_invsqrt<<<grid_for(n), kBlock, 0, s>>>(y, x, nrm2, n);
}

#define STG_DISPATCH_MPW(k, CALL)        \
  if ((k) <= 8) {                        \
    constexpr int MPW = 1;               \
    CALL;                                \
  } else if ((k) <= 16) {                \
    constexpr int MPW = 2;               \
    CALL;                                \
  } else if ((k) <= 32) {                \
    constexpr int MPW = 4;               \
    CALL;                                \
  } else {                               \
    constexpr int MPW = 8;               \
    CALL;                                \
  }

// The completion counter lives right after the partial-sum area (see
// kPartialDoubles in kernels.hpp); it is zero between launches.
unsigned* counter_of(double* partial) {
  return reinterpret_cast<unsigned*>(partial + kPartialDoubles);
}

void vec_multidot(const double* V, long long ldv, int k, const double* w, long long n,
                  double* partial, double* out, cudaStream_t s) {
  const int g = multi_grid(n);
  unsigned* c = counter_of(partial);
  STG_DISPATCH_MPW(k, (k_multidot<MPW><<<g, kMultiBlock, 0, s>>>(V, ldv, k, w, n, partial, out,
                                                                 c)));
}

void vec_update_dot(double* w, const double* V, long long ldv, int k, const double* h,
                    long long n, int want_dots, double* partial, double* out2, cudaStream_t s,
                    const double* scale_src, double* scale_out) {
  const int g = multi_grid(n);
  unsigned* c = counter_of(partial);
  STG_DISPATCH_MPW(k, (k_update<MPW><<<g, kMultiBlock, 0, s>>>(w, V, ldv, k, h, n, want_dots,
                                                               -1.0, partial, scale_src,
                                                               scale_out, out2, c)));
}

void vec_combine(double* x, const double* V, long long ldv, int k, const double* y, long long n,
                 cudaStream_t s) {
  const int g = multi_grid(n);
  STG_DISPATCH_MPW(k, (k_update<MPW><<<g, kMultiBlock, 0, s>>>(x, V, ldv, k, y, n, 0, 1.0,
                                                               nullptr, nullptr, nullptr, nullptr,
                                                               nullptr)));
}

void vec_maxabs(const double* x, long long n, double* partial, double* out, cudaStream_t s) {
  const int g = grid_for(n);
  k_maxabs<<<g, kBlock, 0, s>>>(x, n, partial, out, counter_of(partial));
}

void vec_dot(const double* x, const double* y, long long n, double* partial, double* out,
             cudaStream_t s) {
  vec_multidot(x, 0, 1, y, n, partial, out, s);
}

}  // namespace stg
