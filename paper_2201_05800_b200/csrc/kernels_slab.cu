// Fused space-time DG-SEM slab-operator kernels (sm_100a, fp64).
//
// One launch computes, for every element and every output temporal block,
//   R_r = sum_j T(r,j) X_j + sum_j S(r,j) G_j + c_r W
// with G_j the DG-SEM spatial operator of block j (see kernels.hpp for how the
// reference callers st_residual / st_jacobian / rk_step map onto T, S, c).
// The spatial operator restates SpatialOperator::rhs (spatial.hpp:107-266)
// for constant-velocity advection: the weak-form volume term by sum
// factorisation (spatial.hpp:117-156), LLF faces (spatial.hpp:20-25,
// 158-208) gathered from neighbour traces (no atomics; every element
// recomputes its own face fluxes, which is bitwise deterministic), and the
// mass division (spatial.hpp:265) folded into the coefficients.
//
// Kernels:
//   slab1d_kernel<N1>        d = 1: one thread per element, all temporal nodes
//                            in registers; advection and Burgers (EXTENSION).
//   slab_generic_kernel<D,N1> d = 2, 3: one thread per spatial node with the
//                            element staged in shared memory.
//   slab3d_n4_tma<...>       d = 3, N = 3, n_tau = 4 (the c4/c5 target): one
//                            TMA tensor load (128B-swizzled) of an 8-element
//                            x-pencil, two register-tiled phases (x/y, then
//                            z/t) exchanging partial results through shared
//                            memory.
#include <cuda.h>

#include <cstdlib>
#include <type_traits>

#include "kernels.hpp"
#include "krylov.cuh"

namespace stg {
namespace {

constexpr int kThreads1d = 128;

__device__ __forceinline__ int wrap_m(int c, int n) { return c == 0 ? n - 1 : c - 1; }
__device__ __forceinline__ int wrap_p(int c, int n) { return c == n - 1 ? 0 : c + 1; }

// ---------------------------------------------------------------------------
// Spatial operators on one line of N1 nodes (1-D element)
// ---------------------------------------------------------------------------
template <int N1>
__device__ __forceinline__ void advection_line(const SpatialCoef& sp, const double* x, double xl,
                                               double xr, double* G) {
#pragma unroll
  for (int i = 0; i < N1; ++i) {
    double g = 0.0;
#pragma unroll
    for (int k = 0; k < N1; ++k) g = fma(sp.V[0][i][k], x[k], g);
    G[i] = g;
  }
  G[0] = fma(sp.cL[0], xl, G[0]);
  G[N1 - 1] = fma(sp.cR[0], xr, G[N1 - 1]);
}

// Burgers (EXTENSION, not in the reference): flux differencing with the
// entropy-conservative two-point flux f#(a,b) = (a^2+ab+b^2)/6, LLF
// interface flux with lambda = max(|uL|,|uR|), SAT lifting.
__device__ __forceinline__ double bf(double u) { return 0.5 * u * u; }
__device__ __forceinline__ double bllf(double uL, double uR) {
  const double lam = fmax(fabs(uL), fabs(uR));
  return 0.5 * (bf(uL) + bf(uR)) + 0.5 * lam * (uL - uR);
}
__device__ __forceinline__ double dbllf(double uL, double uR, double vL, double vR) {
  const double aL = fabs(uL), aR = fabs(uR);
  double lam, dlam;
  if (aL >= aR) {
    lam = aL;
    dlam = (uL >= 0.0 ? 1.0 : -1.0) * vL;
  } else {
    lam = aR;
    dlam = (uR >= 0.0 ? 1.0 : -1.0) * vR;
  }
  return 0.5 * (uL * vL + uR * vR) + 0.5 * dlam * (uL - uR) + 0.5 * lam * (vL - vR);
}

template <int N1>
__device__ __forceinline__ void burgers_line(const SpatialCoef& sp, const double* u, double ul,
                                             double ur, double* G) {
  // sum_k 2 D(i,k) f#(u_i,u_k), f#(a,b) = (a^2+ab+b^2)/6, with the 2/6 = 1/3
  // factored out of the sum: no division per pair
#pragma unroll
  for (int i = 0; i < N1; ++i) {
    double vol = 0.0;
#pragma unroll
    for (int k = 0; k < N1; ++k) vol = fma(sp.Dm[i][k], fma(u[i], u[i] + u[k], u[k] * u[k]), vol);
    G[i] = -sp.sc * vol * (1.0 / 3.0);
  }
  G[N1 - 1] -= sp.sc * (bllf(u[N1 - 1], ur) - bf(u[N1 - 1])) * sp.inv_wN;
  G[0] += sp.sc * (bllf(ul, u[0]) - bf(u[0])) * sp.inv_w0;
}

template <int N1>
__device__ __forceinline__ void burgers_jvp_line(const SpatialCoef& sp, const double* u, double ul,
                                                 double ur, const double* v, double vl, double vr,
                                                 double* G) {
#pragma unroll
  for (int i = 0; i < N1; ++i) {
    double vol = 0.0;
#pragma unroll
    for (int k = 0; k < N1; ++k)
      vol = fma(sp.Dm[i][k], (2.0 * u[i] + u[k]) * v[i] + (u[i] + 2.0 * u[k]) * v[k], vol);
    G[i] = -sp.sc * vol * (1.0 / 3.0);
  }
  G[N1 - 1] -= sp.sc * (dbllf(u[N1 - 1], ur, v[N1 - 1], vr) - u[N1 - 1] * v[N1 - 1]) * sp.inv_wN;
  G[0] += sp.sc * (dbllf(ul, u[0], vl, v[0]) - u[0] * v[0]) * sp.inv_w0;
}

// ---------------------------------------------------------------------------
// d = 1: one thread per element
// ---------------------------------------------------------------------------
template <int N1>
__global__ void __launch_bounds__(kThreads1d) slab1d_kernel(const SlabArgs a) {
  pdl_entry();
  if (skip_now(a.skip)) return;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int K = a.g.nx;
  if (c >= K) return;
  const long long ns = a.g.n_sdof;
  const int cl = wrap_m(c, K), cr = wrap_p(c, K);
  const long long oc = (long long)c * N1, ol = (long long)cl * N1 + (N1 - 1),
                  orr = (long long)cr * N1;
  double x[kMaxT][N1];
  double G[kMaxT][N1];
#pragma unroll
  for (int j = 0; j < kMaxT; ++j) {
    if (j < a.n_in) {
      const double* Xj = a.X + j * ns;
#pragma unroll
      for (int i = 0; i < N1; ++i) x[j][i] = Xj[oc + i];
      const double xl = Xj[ol], xr = Xj[orr];
      if (a.model == int(Model::advection)) {
        advection_line<N1>(a.sp, x[j], xl, xr, G[j]);
      } else if (!a.jvp) {
        burgers_line<N1>(a.sp, x[j], xl, xr, G[j]);
      } else {
        const double* Uj = a.U + j * ns;
        double u[N1];
#pragma unroll
        for (int i = 0; i < N1; ++i) u[i] = Uj[oc + i];
        burgers_jvp_line<N1>(a.sp, u, Uj[ol], Uj[orr], x[j], xl, xr, G[j]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < N1; ++i) x[j][i] = G[j][i] = 0.0;
    }
  }
  double w[N1];
#pragma unroll
  for (int i = 0; i < N1; ++i) w[i] = a.has_w ? a.W[oc + i] : 0.0;
#pragma unroll
  for (int r = 0; r < kMaxT; ++r) {
    if (r >= a.n_out) break;
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      double acc = a.mx.c[r] * w[i];
#pragma unroll
      for (int j = 0; j < kMaxT; ++j) {
        if (j < a.n_in) {
          acc = fma(a.mx.T[r][j], x[j][i], acc);
          acc = fma(a.mx.S[r][j], G[j][i], acc);
        }
      }
      a.R[r * ns + oc + i] = acc;
    }
  }
}

// ---------------------------------------------------------------------------
// d = 1, large meshes (c3): one lane per (element, temporal block).  The
// NT lanes of an element compute their block's F(X_j) (or Burgers' exact
// J_F(U_j) X_j) and exchange X_j, G_j by shuffles for the temporal mix; lane
// j writes output block j.  32 / NT elements per warp: 4x the threads of
// slab1d_kernel and short per-lane chains.
// ---------------------------------------------------------------------------
// CTA + grid reduction of the fused residual norms (RED kernels): max via
// atomic max on the bit patterns of non-negative doubles, the sum of squares
// via per-CTA partials added in fixed order by the last CTA
__device__ __forceinline__ void block_reduce_r(const SlabArgs& a, double rmax, double rss) {
  __shared__ double red_m[32], red_s[32];
  const int tid = threadIdx.x, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    rmax = nan_max(rmax, __shfl_down_sync(0xffffffffu, rmax, o));
    rss += __shfl_down_sync(0xffffffffu, rss, o);
  }
  if ((tid & 31) == 0) {
    red_m[tid >> 5] = rmax;
    red_s[tid >> 5] = rss;
  }
  __syncthreads();
  if (tid == 0) {
    double m = 0.0, s2 = 0.0;
    for (int q = 0; q < nw; ++q) {
      m = nan_max(m, red_m[q]);
      s2 += red_s[q];
    }
    atomicMax(a.red_max, static_cast<unsigned long long>(__double_as_longlong(m)));
    a.red_part[blockIdx.x] = s2;
  }
  unsigned* counter = reinterpret_cast<unsigned*>(a.red_part + kPartialDoubles);
  if (is_last_block(counter)) block_finish_sum(a.red_part, gridDim.x, 1, a.red_ss, counter);
}

// RED: also max |R_i| and <R,R> (the Newton residual, see slab3d_n4_persist)
template <int N1, int NT, bool RED = false>
__global__ void __launch_bounds__(256) slab1d_lane_kernel(const SlabArgs a) {
  pdl_entry();
  if (skip_now(a.skip)) return;
  constexpr int EPW = 32 / NT;  // elements per warp
  const int lane = threadIdx.x & 31;
  const int e = lane / NT, j = lane - (lane / NT) * NT;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int K = a.g.nx;
  const long long c0 = warp * EPW + e;
  const bool act = e < EPW && c0 < K;
  const int c = act ? int(c0) : 0;
  const long long ns = a.g.n_sdof;
  const int cl = wrap_m(c, K), cr = wrap_p(c, K);
  const long long oc = (long long)c * N1, ol = (long long)cl * N1 + (N1 - 1),
                  orr = (long long)cr * N1;
  double x[N1], G[N1];
#pragma unroll
  for (int i = 0; i < N1; ++i) x[i] = G[i] = 0.0;
  if (act && j < a.n_in && a.fdv) {
    // fused central difference: x <- v, G <- [F(U + e v) - F(U - e v)] / 2e
    const double vv = *a.fd_vv;
    const double c = a.fd_uu ? a.fd_c * sqrt(1.0 + sqrt(*a.fd_uu)) : a.fd_c;
    const double e = vv > 0.0 ? c / sqrt(vv) : 1.0;
    const double* Uj = a.X + j * ns;
    const double* vj = a.fdv + j * ns;
    double up[N1], um[N1], Gp[N1], Gm[N1];
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      x[i] = vj[oc + i];
      up[i] = fma(e, x[i], Uj[oc + i]);
      um[i] = fma(-e, x[i], Uj[oc + i]);
    }
    const double vl = vj[ol], vr = vj[orr];
    burgers_line<N1>(a.sp, up, fma(e, vl, Uj[ol]), fma(e, vr, Uj[orr]), Gp);
    burgers_line<N1>(a.sp, um, fma(-e, vl, Uj[ol]), fma(-e, vr, Uj[orr]), Gm);
    const double inv = 0.5 / e;
#pragma unroll
    for (int i = 0; i < N1; ++i) G[i] = (Gp[i] - Gm[i]) * inv;
  } else if (act && j < a.n_in) {
    const double* Xj = a.X + j * ns;
#pragma unroll
    for (int i = 0; i < N1; ++i) x[i] = Xj[oc + i];
    const double xl = Xj[ol], xr = Xj[orr];
    if (a.model == int(Model::advection)) {
      advection_line<N1>(a.sp, x, xl, xr, G);
    } else if (!a.jvp) {
      burgers_line<N1>(a.sp, x, xl, xr, G);
    } else {
      const double* Uj = a.U + j * ns;
      double u[N1];
#pragma unroll
      for (int i = 0; i < N1; ++i) u[i] = Uj[oc + i];
      burgers_jvp_line<N1>(a.sp, u, Uj[ol], Uj[orr], x, xl, xr, G);
    }
  }
  const int base = e * NT;  // first lane of this element's group
  double acc[N1];
  const bool out_lane = act && j < a.n_out;
  const double cr_ = out_lane ? a.mx.c[j] : 0.0;
#pragma unroll
  for (int i = 0; i < N1; ++i) acc[i] = out_lane && a.has_w ? cr_ * a.W[oc + i] : 0.0;
#pragma unroll
  for (int jj = 0; jj < NT; ++jj) {
    const double tr = out_lane ? a.mx.T[j][jj] : 0.0, sr = out_lane ? a.mx.S[j][jj] : 0.0;
    const int src = base + jj < 32 ? base + jj : lane;
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      const double xv = __shfl_sync(0xffffffffu, x[i], src);
      const double gv = __shfl_sync(0xffffffffu, G[i], src);
      acc[i] = fma(tr, xv, acc[i]);
      acc[i] = fma(sr, gv, acc[i]);
    }
  }
  if (RED) {
    double rmax = 0.0, rss = 0.0;
    if (out_lane) {
#pragma unroll
      for (int i = 0; i < N1; ++i) {
        rmax = nan_max(rmax, fabs(acc[i]));
        rss = fma(acc[i], acc[i], rss);
      }
    }
    block_reduce_r(a, rmax, rss);
  }
  if (out_lane) {
    double* Rj = a.R + j * ns + oc;
    if (N1 % 2 == 0 && (reinterpret_cast<uintptr_t>(Rj) & 15) == 0) {
      // 16-byte stores: each lane's row is one or more whole 32-byte sectors
#pragma unroll
      for (int i = 0; i + 1 < N1; i += 2)
        *reinterpret_cast<double2*>(Rj + i) = make_double2(acc[i], acc[i + 1]);
    } else {
#pragma unroll
      for (int i = 0; i < N1; ++i) Rj[i] = acc[i];
    }
  }
}

// ---------------------------------------------------------------------------
// d = 2, 3 generic: one thread per spatial node, element in shared memory
// ---------------------------------------------------------------------------
template <int D, int N1>
struct GenericShape {
  static constexpr int NPC = D == 2 ? N1 * N1 : N1 * N1 * N1;
  static constexpr int E = NPC >= 128 ? 1 : (NPC >= 64 ? 2 : (NPC >= 32 ? 4 : 8));
  static constexpr int THREADS = E * NPC;
};

template <int D, int N1>
__global__ void __launch_bounds__(GenericShape<D, N1>::THREADS)
    slab_generic_kernel(const SlabArgs a) {
  pdl_entry();
  if (skip_now(a.skip)) return;
  using Sh = GenericShape<D, N1>;
  constexpr int NPC = Sh::NPC;
  constexpr int E = Sh::E;
  constexpr int S1 = N1, S2 = N1 * N1;  // node strides for y, z
  extern __shared__ double sm[];
  const int tid = threadIdx.x;
  const int e = tid / NPC, node = tid - e * NPC;
  const int cell = blockIdx.x * E + e;
  const bool active = cell < a.g.n_cells;
  const long long ns = a.g.n_sdof;
  const int nin = a.n_in;
  double* Xs = sm + (size_t)e * kMaxT * NPC;
  if (active) {
#pragma unroll
    for (int j = 0; j < kMaxT; ++j)
      if (j < nin) Xs[j * NPC + node] = a.X[j * ns + (long long)cell * NPC + node];
  }
  __syncthreads();
  if (!active) return;

  const int ix = node % N1;
  const int iy = (node / N1) % N1;
  const int iz = D == 3 ? node / S2 : 0;
  const int nx = a.g.nx, ny = a.g.ny, nz = a.g.nz;
  const int cx = cell % nx;
  const int cy = (cell / nx) % ny;
  const int cz = D == 3 ? cell / (nx * ny) : 0;
  // neighbour cells and the traces this node needs (face gather)
  const bool fxL = ix == 0 && a.sp.cL[0] != 0.0, fxR = ix == N1 - 1 && a.sp.cR[0] != 0.0;
  const bool fyL = iy == 0 && a.sp.cL[1] != 0.0, fyR = iy == N1 - 1 && a.sp.cR[1] != 0.0;
  const bool fzL = D == 3 && iz == 0 && a.sp.cL[2] != 0.0;
  const bool fzR = D == 3 && iz == N1 - 1 && a.sp.cR[2] != 0.0;
  const long long oxL = ((long long)(cell - cx + wrap_m(cx, nx))) * NPC + node + (N1 - 1);
  const long long oxR = ((long long)(cell - cx + wrap_p(cx, nx))) * NPC + node - (N1 - 1);
  const long long oyL = ((long long)(cell + (wrap_m(cy, ny) - cy) * nx)) * NPC + node + (N1 - 1) * S1;
  const long long oyR = ((long long)(cell + (wrap_p(cy, ny) - cy) * nx)) * NPC + node - (N1 - 1) * S1;
  const long long ozL = ((long long)(cell + (wrap_m(cz, nz) - cz) * nx * ny)) * NPC + node + (N1 - 1) * S2;
  const long long ozR = ((long long)(cell + (wrap_p(cz, nz) - cz) * nx * ny)) * NPC + node - (N1 - 1) * S2;

  double x[kMaxT], G[kMaxT];
#pragma unroll
  for (int j = 0; j < kMaxT; ++j) {
    x[j] = 0.0;
    G[j] = 0.0;
    if (j < nin) {
      const double* Xe = Xs + j * NPC;
      x[j] = Xe[node];
      double g = 0.0;
#pragma unroll
      for (int k = 0; k < N1; ++k) g = fma(a.sp.V[0][ix][k], Xe[node - ix + k], g);
#pragma unroll
      for (int k = 0; k < N1; ++k) g = fma(a.sp.V[1][iy][k], Xe[node + (k - iy) * S1], g);
      if (D == 3) {
#pragma unroll
        for (int k = 0; k < N1; ++k) g = fma(a.sp.V[2][iz][k], Xe[node + (k - iz) * S2], g);
      }
      const double* Xj = a.X + j * ns;
      if (fxL) g = fma(a.sp.cL[0], Xj[oxL], g);
      if (fxR) g = fma(a.sp.cR[0], Xj[oxR], g);
      if (fyL) g = fma(a.sp.cL[1], Xj[oyL], g);
      if (fyR) g = fma(a.sp.cR[1], Xj[oyR], g);
      if (fzL) g = fma(a.sp.cL[2], Xj[ozL], g);
      if (fzR) g = fma(a.sp.cR[2], Xj[ozR], g);
      G[j] = g;
    }
  }
  const long long o = (long long)cell * NPC + node;
  const double w = a.has_w ? a.W[o] : 0.0;
#pragma unroll
  for (int r = 0; r < kMaxT; ++r) {
    if (r >= a.n_out) break;
    double acc = a.mx.c[r] * w;
#pragma unroll
    for (int j = 0; j < kMaxT; ++j) {
      if (j < nin) {
        acc = fma(a.mx.T[r][j], x[j], acc);
        acc = fma(a.mx.S[r][j], G[j], acc);
      }
    }
    a.R[r * ns + o] = acc;
  }
}

// ---------------------------------------------------------------------------
// d = 2: E consecutive cells per CTA staged in shared memory, three balanced
// line-owner phases (every thread owns one line of N1 nodes per phase):
//   A: x-line at (t, y)  -> x derivative + x faces      -> G
//   B: y-line at (t, x)  -> y derivative + y faces      -> G (complete F)
//   C: t-line at (y, x)  -> temporal mixing + u_n term  -> R (coalesced STG)
// Shared-memory traffic is ~8 doubles per DOF and there are few registers
// per thread, so many CTAs stay resident to hide HBM latency.
// ---------------------------------------------------------------------------
template <int N1, int NT>
struct Shape2d {
  static constexpr int NPC = N1 * N1;
  static constexpr int LINES = (NT > N1 ? NT : N1) * N1;  // threads per cell
  static constexpr int E = LINES >= 32 ? 4 : 8;
  static constexpr int THREADS = E * LINES;
};

template <int N1, int NT>
__global__ void __launch_bounds__(Shape2d<N1, NT>::THREADS)
    slab2d_kernel(const SlabArgs a) {
  pdl_entry();
  if (skip_now(a.skip)) return;
  using Sh = Shape2d<N1, NT>;
  constexpr int NPC = Sh::NPC, E = Sh::E;
  __shared__ double Xs[NT][E][NPC];
  __shared__ double Gs[NT][E][NPC];
  const int tid = threadIdx.x;
  const int nx = a.g.nx, ny = a.g.ny;
  const long long ns = a.g.n_sdof;
  const int c0 = blockIdx.x * E;
  const int ncell = a.g.n_cells;

  // ---- coalesced staging of the tile: for each t, E*NPC contiguous doubles
  for (int q = tid; q < NT * E * NPC; q += Sh::THREADS) {
    const int t = q / (E * NPC), r = q - t * (E * NPC);
    const int e = r / NPC;
    Xs[t][e][r - e * NPC] = (c0 + e < ncell) ? a.X[t * ns + (long long)c0 * NPC + r] : 0.0;
  }

  // ---- identities and early global loads ---------------------------------
  const int e = tid / Sh::LINES, l = tid - (tid / Sh::LINES) * Sh::LINES;
  const int cell = c0 + e;
  const bool active = e < E && cell < ncell;
  const int cx = cell % nx, cy = (cell / nx) % ny;
  const bool nLx = a.sp.cL[0] != 0.0, nRx = a.sp.cR[0] != 0.0;
  const bool nLy = a.sp.cL[1] != 0.0, nRy = a.sp.cR[1] != 0.0;
  // phase A/B line index: t = l / N1, m = l % N1 (y for A, x for B)
  const bool lineAB = active && l < NT * N1;
  const int tL = l / N1, mL = l - (l / N1) * N1;
  double xl = 0.0, xr = 0.0, yl = 0.0, yr = 0.0;
  if (lineAB) {
    const double* Xt = a.X + tL * ns;
    const bool inL = e > 0 && cx > 0, inR = e < E - 1 && cx < nx - 1 && cell + 1 < ncell;
    if (nLx && !inL) xl = Xt[(long long)(cell - cx + (cx == 0 ? nx - 1 : cx - 1)) * NPC + mL * N1 + N1 - 1];
    if (nRx && !inR) xr = Xt[(long long)(cell - cx + (cx == nx - 1 ? 0 : cx + 1)) * NPC + mL * N1];
    if (nLy) yl = Xt[(long long)(cell + ((cy == 0 ? ny - 1 : cy - 1) - cy) * nx) * NPC + (N1 - 1) * N1 + mL];
    if (nRy) yr = Xt[(long long)(cell + ((cy == ny - 1 ? 0 : cy + 1) - cy) * nx) * NPC + mL];
  }
  // phase C: node (y, x) = (l / N1, l % N1)
  const bool lineC = active && l < NPC;
  double w = 0.0;
  if (lineC && a.has_w) w = a.W[(long long)cell * NPC + l];
  __syncthreads();

  // ---- phase A: x-line at (t = tL, y = mL) ---------------------------------
  if (lineAB) {
    const double* row = &Xs[tL][e][mL * N1];
    if (nLx && e > 0 && cx > 0) xl = Xs[tL][e - 1][mL * N1 + N1 - 1];
    if (nRx && e < E - 1 && cx < nx - 1 && cell + 1 < ncell) xr = Xs[tL][e + 1][mL * N1];
    double u[N1];
#pragma unroll
    for (int k = 0; k < N1; ++k) u[k] = row[k];
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      double g = 0.0;
#pragma unroll
      for (int k = 0; k < N1; ++k) g = fma(a.sp.V[0][i][k], u[k], g);
      if (i == 0) g = fma(a.sp.cL[0], xl, g);
      if (i == N1 - 1) g = fma(a.sp.cR[0], xr, g);
      Gs[tL][e][mL * N1 + i] = g;
    }
  }
  __syncthreads();
  // ---- phase B: y-line at (t = tL, x = mL) ---------------------------------
  if (lineAB) {
    double u[N1];
#pragma unroll
    for (int k = 0; k < N1; ++k) u[k] = Xs[tL][e][k * N1 + mL];
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      double g = Gs[tL][e][i * N1 + mL];
#pragma unroll
      for (int k = 0; k < N1; ++k) g = fma(a.sp.V[1][i][k], u[k], g);
      if (i == 0) g = fma(a.sp.cL[1], yl, g);
      if (i == N1 - 1) g = fma(a.sp.cR[1], yr, g);
      Gs[tL][e][i * N1 + mL] = g;
    }
  }
  __syncthreads();
  // ---- phase C: t-line at node l ---------------------------------------------
  if (lineC) {
    double x[NT], G[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      x[j] = Xs[j][e][l];
      G[j] = Gs[j][e][l];
    }
    double* Rp = a.R + (long long)cell * NPC + l;
#pragma unroll
    for (int r = 0; r < NT; ++r) {
      if (r >= a.n_out) break;
      double acc = a.mx.c[r] * w;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        acc = fma(a.mx.T[r][j], x[j], acc);
        acc = fma(a.mx.S[r][j], G[j], acc);
      }
      Rp[r * ns] = acc;
    }
  }
}

// PTX helpers for the mbarrier / bulk-async-copy pipelines.
namespace ptx {
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(phase)
      : "memory");
  return ok != 0;
}
// generic-proxy reads of a buffer before async-proxy (TMA / bulk) writes to it
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
}  // namespace ptx

// Persistent variant of slab2d_kernel: the E-cell tile of segment i+1 is
// bulk-copied (cp.async.bulk, one copy per temporal block) into the other
// stage of a 2-stage ring while segment i is computed, and each thread
// prefetches the next segment's neighbour traces and u_n into registers.
// Time planes are padded by 2 doubles (keeps 16-byte alignment for the bulk
// copies and breaks the 2-way bank conflicts between planes).
// Requires n_cells % E == 0.
template <int N1, int NT>
struct P2d {
  using Sh = Shape2d<N1, NT>;
  static constexpr int E = Sh::E, NPC = Sh::NPC;
  // plane pitch: +10 doubles for (N1, NT) = (5, 5) (c2) minimises shared-
  // memory wavefronts with the line-major thread mapping (bank simulation:
  // 735 vs 915 half-warp wavefronts per tile); +2 keeps 16-byte alignment
  static constexpr int PAD = (N1 == 5 && NT == 5) ? 10 : 2;
  static constexpr int PLANE = E * NPC + PAD;         // padded plane (doubles)
  static constexpr int STAGE = NT * PLANE;            // doubles per stage
  static constexpr int SMEM = (3 * STAGE) * 8 + 64;   // 2 X stages + G + barriers
};

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
      : "memory");
}

template <int N1, int NT>
__global__ void __launch_bounds__(Shape2d<N1, NT>::THREADS)
    slab2d_persist(const SlabArgs a) {
  pdl_entry();
  if (skip_now(a.skip)) return;
  using P = P2d<N1, NT>;
  using Sh = typename P::Sh;
  constexpr int NPC = P::NPC, E = P::E, PL = P::PLANE;
  extern __shared__ __align__(16) double sm2[];
  double* G = sm2 + 2 * P::STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm2 + 3 * P::STAGE);
  const uint32_t bar0 = ptx::smem_u32(bars), bar1 = ptx::smem_u32(bars + 1);
  const int tid = threadIdx.x;
  const int nx = a.g.nx, ny = a.g.ny;
  const long long ns = a.g.n_sdof;
  const int nseg = a.g.n_cells / E;
  const uint32_t tbytes = E * NPC * 8;
  const bool nLx = a.sp.cL[0] != 0.0, nRx = a.sp.cR[0] != 0.0;
  const bool nLy = a.sp.cL[1] != 0.0, nRy = a.sp.cR[1] != 0.0;

  if (tid == 0) {
    ptx::mbar_init(bar0, 1);
    ptx::mbar_init(bar1, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();

  const int e = tid / Sh::LINES, l = tid - (tid / Sh::LINES) * Sh::LINES;
  const bool lineAB = l < NT * N1;
  const bool lineC = l < NPC;
  const int tL = l % NT, mL = l / NT;  // line-major: consecutive lanes step in t

  auto issue = [&](int seg, int st) {
    const uint32_t bar = st ? bar1 : bar0;
    ptx::mbar_expect_tx(bar, NT * tbytes);
    const uint32_t dst = ptx::smem_u32(sm2 + st * P::STAGE);
    const double* src = a.X + (long long)seg * E * NPC;
    for (int t = 0; t < NT; ++t) bulk_g2s(dst + t * PL * 8, src + t * ns, tbytes, bar);
  };
  // neighbour traces (x halos from outside the tile, y faces) and u_n
  auto faces = [&](int seg, double& xl, double& xr, double& yl, double& yr, double& w) {
    const int cell = seg * E + e;
    const int cx = cell % nx, cy = (cell / nx) % ny;
    xl = xr = yl = yr = w = 0.0;
    if (lineAB) {
      const double* Xt = a.X + tL * ns;
      if (nLx && !(e > 0 && cx > 0))
        xl = Xt[(long long)(cell - cx + (cx == 0 ? nx - 1 : cx - 1)) * NPC + mL * N1 + N1 - 1];
      if (nRx && !(e < E - 1 && cx < nx - 1))
        xr = Xt[(long long)(cell - cx + (cx == nx - 1 ? 0 : cx + 1)) * NPC + mL * N1];
      if (nLy) yl = Xt[(long long)(cell + ((cy == 0 ? ny - 1 : cy - 1) - cy) * nx) * NPC + (N1 - 1) * N1 + mL];
      if (nRy) yr = Xt[(long long)(cell + ((cy == ny - 1 ? 0 : cy + 1) - cy) * nx) * NPC + mL];
    }
    if (lineC && a.has_w) w = a.W[(long long)cell * NPC + l];
  };

  int seg = blockIdx.x;
  if (tid == 0 && seg < nseg) issue(seg, 0);
  double xl, xr, yl, yr, w;
  if (seg < nseg) faces(seg, xl, xr, yl, yr, w);

  for (int it = 0; seg < nseg; ++it, seg += gridDim.x) {
    const int st = it & 1;
    const int nxt = seg + gridDim.x;
    if (tid == 0 && nxt < nseg) {
      ptx::fence_proxy_async_smem();
      issue(nxt, st ^ 1);
    }
    double nxl = 0, nxr = 0, nyl = 0, nyr = 0, nw = 0;
    if (nxt < nseg) faces(nxt, nxl, nxr, nyl, nyr, nw);
    while (!ptx::mbar_try_wait(st ? bar1 : bar0, (it >> 1) & 1)) {
    }
    const double* X = sm2 + st * P::STAGE;
    const int cell = seg * E + e;
    const int cx = cell % nx;

    // phase A: x-line at (t = tL, y = mL)
    if (lineAB) {
      const double* row = X + tL * PL + e * NPC + mL * N1;
      double hl = xl, hr = xr;
      if (nLx && e > 0 && cx > 0) hl = row[-NPC + N1 - 1];
      if (nRx && e < E - 1 && cx < nx - 1) hr = row[NPC];
      double u[N1];
#pragma unroll
      for (int k = 0; k < N1; ++k) u[k] = row[k];
      double* g = G + tL * PL + e * NPC + mL * N1;
#pragma unroll
      for (int i = 0; i < N1; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < N1; ++k) acc = fma(a.sp.V[0][i][k], u[k], acc);
        if (i == 0) acc = fma(a.sp.cL[0], hl, acc);
        if (i == N1 - 1) acc = fma(a.sp.cR[0], hr, acc);
        g[i] = acc;
      }
    }
    __syncthreads();
    // phase B: y-line at (t = tL, x = mL)
    if (lineAB) {
      const double* col = X + tL * PL + e * NPC + mL;
      double* g = G + tL * PL + e * NPC + mL;
      double u[N1];
#pragma unroll
      for (int k = 0; k < N1; ++k) u[k] = col[k * N1];
#pragma unroll
      for (int i = 0; i < N1; ++i) {
        double acc = g[i * N1];
#pragma unroll
        for (int k = 0; k < N1; ++k) acc = fma(a.sp.V[1][i][k], u[k], acc);
        if (i == 0) acc = fma(a.sp.cL[1], yl, acc);
        if (i == N1 - 1) acc = fma(a.sp.cR[1], yr, acc);
        g[i * N1] = acc;
      }
    }
    __syncthreads();
    // phase C: t-line at node l
    if (lineC) {
      double x[NT], Gv[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        x[j] = X[j * PL + e * NPC + l];
        Gv[j] = G[j * PL + e * NPC + l];
      }
      double* Rp = a.R + (long long)cell * NPC + l;
#pragma unroll
      for (int r = 0; r < NT; ++r) {
        if (r >= a.n_out) break;
        double acc = a.mx.c[r] * w;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          acc = fma(a.mx.T[r][j], x[j], acc);
          acc = fma(a.mx.S[r][j], Gv[j], acc);
        }
        Rp[r * ns] = acc;
      }
    }
    __syncthreads();  // stage st and G free for reuse
    xl = nxl;
    xr = nxr;
    yl = nyl;
    yr = nyr;
    w = nw;
  }
}

// ---------------------------------------------------------------------------
// d = 2, S diagonal (st_residual, J.v, A^-1-form stage residual): one thread
// per (cell, temporal node) PLANE.  With S diagonal, F(X_t) only enters row
// t of the mix, so the thread that owns plane t of a cell computes the whole
// output plane R_t = sum_j T(t,j) X_j + S(t,t) F(X_t) + c_t W in registers:
// the x and y derivatives on its n x n register tile, the temporal mix from
// the other planes of the staged tile, no intermediate buffer and no phase
// barrier.  E cells per segment; the tile (n_tau planes of E*n^2 doubles,
// plus u_n when present) arrives by bulk copy in a 2-stage ring; R is staged
// back into the consumed stage and written by bulk stores (full lines, no
// partial-sector write traffic).  Lanes are consecutive cells: a plane stride
// of n^2 = 25 doubles (odd) keeps the 64-bit shared accesses conflict-free.
// ---------------------------------------------------------------------------
template <int N1, int NT, int E>
struct Plane2d {
  static constexpr int NPC = N1 * N1;
  static constexpr int THREADS = E * NT;
  static constexpr int PLANE = E * NPC;                 // doubles per plane
  static constexpr int STAGE = (NT + 1) * PLANE;        // NT planes + u_n
  static constexpr int SMEM = (2 * STAGE + NT * PLANE) * 8 + 64;  // 2 stages + R staging
  static_assert(PLANE % 2 == 0, "16-byte aligned planes");
};

__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                   reinterpret_cast<uint64_t>(dst)),
               "r"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int N1, int NT, int E, int MINB>
__global__ void __launch_bounds__(Plane2d<N1, NT, E>::THREADS, MINB)
    slab2d_plane(const SlabArgs a) {
  pdl_entry();
  if (skip_now(a.skip)) return;
  using P = Plane2d<N1, NT, E>;
  constexpr int NPC = P::NPC, PL = P::PLANE;
  // plane j of segment cell c inside a staged tile
  auto tp = [](int j, int c) { return j * PL + c * NPC; };
  constexpr long long CS = NPC;  // global stride between cells
  extern __shared__ __align__(16) double sm2[];
  double* Rs = sm2 + 2 * P::STAGE;  // output staging (NT planes)
  uint64_t* bars = reinterpret_cast<uint64_t*>(Rs + NT * PL);
  const uint32_t bar0 = ptx::smem_u32(bars), bar1 = ptx::smem_u32(bars + 1);
  const int tid = threadIdx.x;
  const int e = tid % E, t = tid / E;
  const int nx = a.g.nx, ny = a.g.ny;
  const long long ns = a.g.n_sdof;
  const int nseg = a.g.n_cells / E;
  const uint32_t pbytes = PL * 8;
  const bool hw = a.has_w != 0;
  const uint32_t sbytes = (NT + (hw ? 1 : 0)) * pbytes;
  const bool nLx = a.sp.cL[0] != 0.0, nRx = a.sp.cR[0] != 0.0;
  const bool nLy = a.sp.cL[1] != 0.0, nRy = a.sp.cR[1] != 0.0;
  double Tr[NT];  // this thread's row of the mix
#pragma unroll
  for (int j = 0; j < NT; ++j) Tr[j] = a.mx.T[t][j];
  const double tt_ = a.mx.T[t][t], st_ = a.mx.S[t][t], ct_ = hw ? a.mx.c[t] : 0.0;

  if (tid == 0) {
    ptx::mbar_init(bar0, 1);
    ptx::mbar_init(bar1, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int seg, int stg) {
    const uint32_t bar = stg ? bar1 : bar0;
    ptx::mbar_expect_tx(bar, sbytes);
    const uint32_t dst = ptx::smem_u32(sm2 + stg * P::STAGE);
    const double* src = a.X + (long long)seg * PL;
    for (int j = 0; j < NT; ++j) bulk_g2s(dst + j * pbytes, src + j * ns, pbytes, bar);
    if (hw) bulk_g2s(dst + NT * pbytes, a.W + (long long)seg * PL, pbytes, bar);
  };
  // neighbour traces that are not in the tile (global / L2)
  auto faces = [&](int seg, double* xl, double* xr, double* yl, double* yr) {
    const int cell = seg * E + e;
    const int cx = cell % nx, cy = (cell / nx) % ny;
    const double* Xt = a.X + t * ns;
    if (nLx && !(e > 0 && cx > 0)) {
      const double* q = Xt + (long long)(cell - cx + (cx == 0 ? nx - 1 : cx - 1)) * CS + N1 - 1;
#pragma unroll
      for (int k = 0; k < N1; ++k) xl[k] = q[k * N1];
    }
    if (nRx && !(e < E - 1 && cx < nx - 1)) {
      const double* q = Xt + (long long)(cell - cx + (cx == nx - 1 ? 0 : cx + 1)) * CS;
#pragma unroll
      for (int k = 0; k < N1; ++k) xr[k] = q[k * N1];
    }
    if (nLy) {
      const double* q = Xt + (long long)(cell + ((cy == 0 ? ny - 1 : cy - 1) - cy) * nx) * CS +
                        (N1 - 1) * N1;
#pragma unroll
      for (int k = 0; k < N1; ++k) yl[k] = q[k];
    }
    if (nRy) {
      const double* q = Xt + (long long)(cell + ((cy == ny - 1 ? 0 : cy + 1) - cy) * nx) * CS;
#pragma unroll
      for (int k = 0; k < N1; ++k) yr[k] = q[k];
    }
  };

  int seg = blockIdx.x;
  if (tid == 0 && seg < nseg) issue(seg, 0);
  double xl[N1], xr[N1], yl[N1], yr[N1];
#pragma unroll
  for (int k = 0; k < N1; ++k) xl[k] = xr[k] = yl[k] = yr[k] = 0.0;
  if (seg < nseg) faces(seg, xl, xr, yl, yr);

  for (int it = 0; seg < nseg; ++it, seg += gridDim.x) {
    const int stg = it & 1;
    const int nxt = seg + gridDim.x;
    if (tid == 0 && nxt < nseg) {
      ptx::fence_proxy_async_smem();
      issue(nxt, stg ^ 1);
    }
    const double* X = sm2 + stg * P::STAGE;
    while (!ptx::mbar_try_wait(stg ? bar1 : bar0, (it >> 1) & 1)) {
    }
    const int cell = seg * E + e;
    const int cx = cell % nx;
    const double* own = X + tp(t, e);
    double u[NPC];
#pragma unroll
    for (int k = 0; k < NPC; ++k) u[k] = own[k];
    if (nLx && e > 0 && cx > 0) {
#pragma unroll
      for (int k = 0; k < N1; ++k) xl[k] = own[-CS + k * N1 + N1 - 1];
    }
    if (nRx && e < E - 1 && cx < nx - 1) {
#pragma unroll
      for (int k = 0; k < N1; ++k) xr[k] = own[CS + k * N1];
    }
    double r[NPC];
#pragma unroll
    for (int iy = 0; iy < N1; ++iy)
#pragma unroll
      for (int ix = 0; ix < N1; ++ix) {
        double g = 0.0;
#pragma unroll
        for (int k = 0; k < N1; ++k) g = fma(a.sp.V[0][ix][k], u[iy * N1 + k], g);
#pragma unroll
        for (int k = 0; k < N1; ++k) g = fma(a.sp.V[1][iy][k], u[k * N1 + ix], g);
        if (ix == 0) g = fma(a.sp.cL[0], xl[iy], g);
        if (ix == N1 - 1) g = fma(a.sp.cR[0], xr[iy], g);
        if (iy == 0) g = fma(a.sp.cL[1], yl[ix], g);
        if (iy == N1 - 1) g = fma(a.sp.cR[1], yr[ix], g);
        r[iy * N1 + ix] = fma(st_, g, tt_ * u[iy * N1 + ix]);
      }
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      if (j == t) continue;
      const double* pj = X + tp(j, e);
#pragma unroll
      for (int k = 0; k < NPC; ++k) r[k] = fma(Tr[j], pj[k], r[k]);
    }
    if (hw && ct_ != 0.0) {
      const double* pw = X + NT * PL + e * NPC;
#pragma unroll
      for (int k = 0; k < NPC; ++k) r[k] = fma(ct_, pw[k], r[k]);
    }
    // prefetch the next segment's out-of-tile traces
    if (nxt < nseg) faces(nxt, xl, xr, yl, yr);
    // the previous segment's bulk stores must have read Rs before it is rewritten
    if (tid == 0) bulk_wait_read0();
    __syncthreads();  // also: every thread has read stage stg (it is refilled next iteration)
    double* outp = Rs + tp(t, e);
#pragma unroll
    for (int k = 0; k < NPC; ++k) outp[k] = r[k];
    ptx::fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      for (int j = 0; j < NT; ++j)
        bulk_s2g(a.R + j * ns + (long long)seg * PL, ptx::smem_u32(Rs + j * PL), pbytes);
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait0();
}

// ---------------------------------------------------------------------------
// slab2d_plane3: the plane kernel with a 3-stage ring.  R is written back
// into the consumed stage and leaves by bulk stores from there (no separate
// output staging), and u_n rides in a 2-slot ring of its own, so a stage is
// the n_tau planes: 3 x 32 KB + 2 x 6.4 KB at c2, 2 CTAs per SM.  The load
// for segment it+2 is issued after the compute of segment it (by then the
// store of it-1, which last used that stage, has long read it).
// ---------------------------------------------------------------------------
template <int N1, int NT, int E>
struct Plane3 {
  static constexpr int NPC = N1 * N1;
  static constexpr int THREADS = E * NT;
  static constexpr int PLANE = E * NPC;
  static constexpr int STAGE = NT * PLANE;
  static constexpr int SMEM = (3 * STAGE + 2 * PLANE) * 8 + 64;
};

// RED: also max |R| and <R,R> (the Newton residual norm and the next GMRES's
// <b,b>), as in slab3d_n4_persist
template <int N1, int NT, int E, bool RED = false>
__global__ void __launch_bounds__(Plane3<N1, NT, E>::THREADS, 2)
    slab2d_plane3(const SlabArgs a) {
  pdl_entry();
  if (skip_now(a.skip)) return;
  using P = Plane3<N1, NT, E>;
  constexpr int NPC = P::NPC, PL = P::PLANE;
  auto tp = [](int j, int c) { return j * PL + c * NPC; };
  constexpr long long CS = NPC;
  extern __shared__ __align__(16) double sm3[];
  double* Ws = sm3 + 3 * P::STAGE;  // u_n ring, 2 slots
  uint64_t* bars = reinterpret_cast<uint64_t*>(Ws + 2 * PL);
  const int tid = threadIdx.x;
  const int e = tid % E, t = tid / E;
  const int nx = a.g.nx, ny = a.g.ny;
  const long long ns = a.g.n_sdof;
  const long long xs = a.x_bcast ? 0 : ns;  // temporal stride of X (x_bcast: one block)
  const int nseg = a.g.n_cells / E;
  const uint32_t pbytes = PL * 8;
  const bool nLx = a.sp.cL[0] != 0.0, nRx = a.sp.cR[0] != 0.0;
  const bool nLy = a.sp.cL[1] != 0.0, nRy = a.sp.cR[1] != 0.0;
  double Tr[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) Tr[j] = a.mx.T[t][j];
  const double tt_ = a.mx.T[t][t], st_ = a.mx.S[t][t];
  const bool hw = a.has_w != 0;
  const double ct_ = hw ? a.mx.c[t] : 0.0;

  if (tid == 0) {
    for (int q = 0; q < 3; ++q) ptx::mbar_init(ptx::smem_u32(bars + q), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  // segment sg into X stage stg and u_n slot wsl, on the stage's barrier
  auto issue = [&](int sg, int stg, int wsl) {
    const uint32_t bar = ptx::smem_u32(bars + stg);
    ptx::mbar_expect_tx(bar, (NT + (hw ? 1 : 0)) * pbytes);
    const uint32_t dst = ptx::smem_u32(sm3 + stg * P::STAGE);
    const double* src = a.X + (long long)sg * PL;
    for (int j = 0; j < NT; ++j) bulk_g2s(dst + j * pbytes, src + j * xs, pbytes, bar);
    if (hw) bulk_g2s(ptx::smem_u32(Ws + wsl * PL), a.W + (long long)sg * PL, pbytes, bar);
  };
  auto faces = [&](int sg, double* xl, double* xr, double* yl, double* yr) {
    const int cell = sg * E + e;
    const int cx = cell % nx, cy = (cell / nx) % ny;
    const double* Xt = a.X + t * xs;
    if (nLx && !(e > 0 && cx > 0)) {
      const double* q = Xt + (long long)(cell - cx + (cx == 0 ? nx - 1 : cx - 1)) * CS + N1 - 1;
#pragma unroll
      for (int k = 0; k < N1; ++k) xl[k] = q[k * N1];
    }
    if (nRx && !(e < E - 1 && cx < nx - 1)) {
      const double* q = Xt + (long long)(cell - cx + (cx == nx - 1 ? 0 : cx + 1)) * CS;
#pragma unroll
      for (int k = 0; k < N1; ++k) xr[k] = q[k * N1];
    }
    if (nLy) {
      const double* q = Xt + (long long)(cell + ((cy == 0 ? ny - 1 : cy - 1) - cy) * nx) * CS +
                        (N1 - 1) * N1;
#pragma unroll
      for (int k = 0; k < N1; ++k) yl[k] = q[k];
    }
    if (nRy) {
      const double* q = Xt + (long long)(cell + ((cy == ny - 1 ? 0 : cy + 1) - cy) * nx) * CS;
#pragma unroll
      for (int k = 0; k < N1; ++k) yr[k] = q[k];
    }
  };

  int seg = blockIdx.x;
  double rmax = 0.0, rss = 0.0;  // RED
  if (tid == 0) {
    if (seg < nseg) issue(seg, 0, 0);
    if (seg + (int)gridDim.x < nseg) issue(seg + gridDim.x, 1, 1);
  }
  double xl[N1], xr[N1], yl[N1], yr[N1];
#pragma unroll
  for (int k = 0; k < N1; ++k) xl[k] = xr[k] = yl[k] = yr[k] = 0.0;
  if (seg < nseg) faces(seg, xl, xr, yl, yr);

  for (int it = 0; seg < nseg; ++it, seg += gridDim.x) {
    const int stg = it % 3;
    const int nxt = seg + gridDim.x;
    double* X = sm3 + stg * P::STAGE;
    while (!ptx::mbar_try_wait(ptx::smem_u32(bars + stg), (it / 3) & 1)) {
    }
    const int cell = seg * E + e;
    const int cx = cell % nx;
    const double* own = X + tp(t, e);
    double u[NPC];
#pragma unroll
    for (int k = 0; k < NPC; ++k) u[k] = own[k];
    if (nLx && e > 0 && cx > 0) {
#pragma unroll
      for (int k = 0; k < N1; ++k) xl[k] = own[-CS + k * N1 + N1 - 1];
    }
    if (nRx && e < E - 1 && cx < nx - 1) {
#pragma unroll
      for (int k = 0; k < N1; ++k) xr[k] = own[CS + k * N1];
    }
    double r[NPC];
#pragma unroll
    for (int iy = 0; iy < N1; ++iy)
#pragma unroll
      for (int ix = 0; ix < N1; ++ix) {
        double g = 0.0;
#pragma unroll
        for (int k = 0; k < N1; ++k) g = fma(a.sp.V[0][ix][k], u[iy * N1 + k], g);
#pragma unroll
        for (int k = 0; k < N1; ++k) g = fma(a.sp.V[1][iy][k], u[k * N1 + ix], g);
        if (ix == 0) g = fma(a.sp.cL[0], xl[iy], g);
        if (ix == N1 - 1) g = fma(a.sp.cR[0], xr[iy], g);
        if (iy == 0) g = fma(a.sp.cL[1], yl[ix], g);
        if (iy == N1 - 1) g = fma(a.sp.cR[1], yr[ix], g);
        r[iy * N1 + ix] = fma(st_, g, tt_ * u[iy * N1 + ix]);
      }
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      if (j == t) continue;
      const double* pj = X + tp(j, e);
#pragma unroll
      for (int k = 0; k < NPC; ++k) r[k] = fma(Tr[j], pj[k], r[k]);
    }
    if (hw && ct_ != 0.0) {
      const double* pw = Ws + (it & 1) * PL + e * NPC;
#pragma unroll
      for (int k = 0; k < NPC; ++k) r[k] = fma(ct_, pw[k], r[k]);
    }
    // next segment's out-of-tile traces
    if (nxt < nseg) faces(nxt, xl, xr, yl, yr);
    __syncthreads();  // every thread has read stage stg and u_n slot it & 1
    if (tid == 0 && nxt + (int)gridDim.x < nseg) {
      // stage (it+2)%3 last held segment it-1, stored at the end of the
      // previous iteration: its bulk store must have read it; u_n slot it&1
      // was read by this iteration (barrier above)
      bulk_wait_read0();
      ptx::fence_proxy_async_smem();
      issue(nxt + gridDim.x, (it + 2) % 3, it & 1);
    }
    double* outp = X + tp(t, e);
#pragma unroll
    for (int k = 0; k < NPC; ++k) {
      outp[k] = r[k];
      if (RED) {
        rmax = nan_max(rmax, fabs(r[k]));
        rss = fma(r[k], r[k], rss);
      }
    }
    ptx::fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      for (int j = 0; j < NT; ++j)
        bulk_s2g(a.R + j * ns + (long long)seg * PL, ptx::smem_u32(X + j * PL), pbytes);
      bulk_commit();
    }
  }
  if (RED) block_reduce_r(a, rmax, rss);
  if (tid == 0) bulk_wait0();
}

// ---------------------------------------------------------------------------
// d = 3, N = 3, n_tau = 4: TMA-staged, register-tiled two-phase kernel
// ---------------------------------------------------------------------------
namespace fast {
constexpr int E = 8;                    // elements per CTA (an x-pencil segment)
constexpr int THREADS = 16 * E;         // 16 threads per element per phase
constexpr int ROWS = 4 * E * 4;         // rows (t, e, z), 16 doubles = 128 B each
constexpr int TILE_DOUBLES = ROWS * 16;
constexpr unsigned TILE_BYTES = TILE_DOUBLES * 8u;  // 16 KiB
constexpr int SMEM_BYTES = 2 * TILE_BYTES + 1024 + 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 128B swizzle (CU_TENSOR_MAP_SWIZZLE_128B): the 16-byte chunk c of row r
// lives at chunk c ^ (r & 7).  q = double index (0..15) within the row.
__device__ __forceinline__ int swz(int row, int q) {
  return row * 16 + ((((q >> 1) ^ (row & 7)) << 1) | (q & 1));
}
__device__ __forceinline__ int row_of(int t, int e, int z) { return (t * E + e) * 4 + z; }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ double2 ldg2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}
}  // namespace fast

template <bool FULL_S>
__global__ void __launch_bounds__(fast::THREADS, 4)
    slab3d_n4_tma(const __grid_constant__ CUtensorMap tmX, const SlabArgs a) {
  pdl_entry();
  if (skip_now(a.skip)) return;
  using namespace fast;
  extern __shared__ unsigned char smem_raw[];
  // align to 1024 B (128B-swizzle atoms) by integer offset so the pointer
  // keeps its shared-memory provenance (LDS/STS, not generic LD/ST)
  unsigned char* base = smem_raw + ((1024u - (fast::smem_u32(smem_raw) & 1023u)) & 1023u);
  double* Xs = reinterpret_cast<double*>(base);
  double* FA = Xs + TILE_DOUBLES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(FA + TILE_DOUBLES);
  const uint32_t bar_a = smem_u32(bar);

  const int tid = threadIdx.x;
  const int nx = a.g.nx, ny = a.g.ny, nz = a.g.nz;
  const long long ns = a.g.n_sdof;
  const int e0 = (a.seg_begin + blockIdx.x) * E;  // first cell of the pencil segment
  const int cx0 = e0 % nx;
  const int cy = (e0 / nx) % ny;
  const int cz = e0 / (nx * ny);

  if (tid == 0) {
    mbar_init(bar_a, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(bar_a, TILE_BYTES);
    tma_load_4d(smem_u32(Xs), &tmX, bar_a, 0, 0, e0, 0);
  }

  const bool nLx = a.sp.cL[0] != 0.0, nRx = a.sp.cR[0] != 0.0;
  const bool nLy = a.sp.cL[1] != 0.0, nRy = a.sp.cR[1] != 0.0;
  const bool nLz = a.sp.cL[2] != 0.0, nRz = a.sp.cR[2] != 0.0;

  // ---- phase-A identity (e, z, t) and its early global loads -------------
  const int zA = tid & 3, eA = (tid >> 2) & (E - 1), tA = tid >> 5;
  const int cellA = e0 + eA;
  const double* XtA = a.X + tA * ns;
  double yl[4] = {0, 0, 0, 0}, yr[4] = {0, 0, 0, 0};
  double hl[4] = {0, 0, 0, 0}, hr[4] = {0, 0, 0, 0};
  {
    const int cym = cy == 0 ? ny - 1 : cy - 1, cyp = cy == ny - 1 ? 0 : cy + 1;
    if (nLy) {
      const double* p = XtA + (long long)(cellA + (cym - cy) * nx) * 64 + zA * 16 + 12;
      const double2 v0 = fast::ldg2(p), v1 = fast::ldg2(p + 2);
      yl[0] = v0.x; yl[1] = v0.y; yl[2] = v1.x; yl[3] = v1.y;
    }
    if (nRy) {
      const double* p = XtA + (long long)(cellA + (cyp - cy) * nx) * 64 + zA * 16;
      const double2 v0 = fast::ldg2(p), v1 = fast::ldg2(p + 2);
      yr[0] = v0.x; yr[1] = v0.y; yr[2] = v1.x; yr[3] = v1.y;
    }
    if (eA == 0 && nLx) {
      const int c = e0 - cx0 + (cx0 == 0 ? nx - 1 : cx0 - 1);
      const double* p = XtA + (long long)c * 64 + zA * 16 + 3;
#pragma unroll
      for (int y = 0; y < 4; ++y) hl[y] = __ldg(p + 4 * y);
    }
    if (eA == E - 1 && nRx) {
      const int cxe = cx0 + E - 1;
      const int c = e0 - cx0 + (cxe == nx - 1 ? 0 : cxe + 1);
      const double* p = XtA + (long long)c * 64 + zA * 16;
#pragma unroll
      for (int y = 0; y < 4; ++y) hr[y] = __ldg(p + 4 * y);
    }
  }
  // ---- phase-B identity (e, x, y) and its early global loads -------------
  const int xB = tid & 3, yB = (tid >> 2) & 3, eB = tid >> 4;
  const int cellB = e0 + eB;
  const int qB = yB * 4 + xB;
  double zl[4] = {0, 0, 0, 0}, zr[4] = {0, 0, 0, 0}, w[4] = {0, 0, 0, 0};
  {
    const int czm = cz == 0 ? nz - 1 : cz - 1, czp = cz == nz - 1 ? 0 : cz + 1;
    if (nLz) {
      const double* p = a.X + (long long)(cellB + (czm - cz) * nx * ny) * 64 + 48 + qB;
#pragma unroll
      for (int t = 0; t < 4; ++t) zl[t] = __ldg(p + t * ns);
    }
    if (nRz) {
      const double* p = a.X + (long long)(cellB + (czp - cz) * nx * ny) * 64 + qB;
#pragma unroll
      for (int t = 0; t < 4; ++t) zr[t] = __ldg(p + t * ns);
    }
    if (a.has_w) {
      const double* p = a.W + (long long)cellB * 64 + qB;
#pragma unroll
      for (int z = 0; z < 4; ++z) w[z] = __ldg(p + 16 * z);
    }
  }

  while (!fast::mbar_try_wait(bar_a, 0)) {
  }

  // ---- phase A: x and y derivatives of the (y,x) plane at (t, e, z) -------
  {
    const int row = row_of(tA, eA, zA);
    const int sw = row & 7;
    double u[16];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double2 v = *reinterpret_cast<const double2*>(Xs + row * 16 + ((c ^ sw) << 1));
      u[2 * c] = v.x;
      u[2 * c + 1] = v.y;
    }
    if (nLx && eA > 0) {
      const int rl = row_of(tA, eA - 1, zA);
#pragma unroll
      for (int y = 0; y < 4; ++y) hl[y] = Xs[swz(rl, 4 * y + 3)];
    }
    if (nRx && eA < E - 1) {
      const int rr = row_of(tA, eA + 1, zA);
#pragma unroll
      for (int y = 0; y < 4; ++y) hr[y] = Xs[swz(rr, 4 * y)];
    }
    double f[16];
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        double g = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) g = fma(a.sp.V[0][x][k], u[4 * y + k], g);
#pragma unroll
        for (int k = 0; k < 4; ++k) g = fma(a.sp.V[1][y][k], u[4 * k + x], g);
        if (x == 0) g = fma(a.sp.cL[0], hl[y], g);
        if (x == 3) g = fma(a.sp.cR[0], hr[y], g);
        if (y == 0) g = fma(a.sp.cL[1], yl[x], g);
        if (y == 3) g = fma(a.sp.cR[1], yr[x], g);
        f[4 * y + x] = g;
      }
#pragma unroll
    for (int c = 0; c < 8; ++c)
      *reinterpret_cast<double2*>(FA + row * 16 + ((c ^ sw) << 1)) =
          make_double2(f[2 * c], f[2 * c + 1]);
  }
  __syncthreads();

  // ---- phase B: z derivative, temporal mixing, store ----------------------
  {
    double u[4][4], f[4][4];  // [t][z]
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int z = 0; z < 4; ++z) {
        const int o = swz(row_of(t, eB, z), qB);
        u[t][z] = Xs[o];
        f[t][z] = FA[o];
      }
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int z = 0; z < 4; ++z) {
        double g = f[t][z];
#pragma unroll
        for (int k = 0; k < 4; ++k) g = fma(a.sp.V[2][z][k], u[t][k], g);
        if (z == 0) g = fma(a.sp.cL[2], zl[t], g);
        if (z == 3) g = fma(a.sp.cR[2], zr[t], g);
        f[t][z] = g;
      }
    double* Rb = a.R + (long long)cellB * 64 + qB;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int z = 0; z < 4; ++z) {
        double acc = a.mx.c[r] * w[z];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc = fma(a.mx.T[r][j], u[j][z], acc);
        if (FULL_S) {
#pragma unroll
          for (int j = 0; j < 4; ++j) acc = fma(a.mx.S[r][j], f[j][z], acc);
        } else {
          acc = fma(a.mx.S[r][r], f[r][z], acc);
        }
        Rb[r * ns + 16 * z] = acc;
      }
  }
}

// ---------------------------------------------------------------------------
// d = 3, N = 3, n_tau = 4, persistent + double-buffered: every operand of a
// segment (8-element x-pencil tile, y/z face traces of the upwind/downwind
// neighbour rows, x halos, u_n) arrives by TMA into a 2-stage ring, so the
// loads of segment i+1 are in flight while segment i is computed.  No
// synchronous global loads remain; R is stored with coalesced STG.
// ---------------------------------------------------------------------------
namespace pst {
using fast::E;
constexpr int THREADS = 16 * E;
constexpr int MAIN = 16384;          // [t][e][z] x 128 B rows, 128B-swizzled
constexpr int FACE = 4096;           // y face: [t][e][z][x]; z face: [t][e][y][x]
constexpr int WBUF = 4096;           // u_n: [e][64]
constexpr int HALO = 1024;           // [t][z][y][2]
constexpr int OFF_YL = MAIN, OFF_YR = OFF_YL + FACE, OFF_ZL = OFF_YR + FACE,
              OFF_ZR = OFF_ZL + FACE, OFF_W = OFF_ZR + FACE, OFF_HL = OFF_W + WBUF,
              OFF_HR = OFF_HL + HALO;
constexpr int STAGE = ((OFF_HR + HALO + 1023) / 1024) * 1024;  // 39936
constexpr int FA_OFF = 2 * STAGE;
constexpr int BAR_OFF = FA_OFF + MAIN;
constexpr int SMEM_BYTES = BAR_OFF + 64 + 1024;

// Runtime stage layout: only the trace buffers the velocity signs need (for
// b > 0: y-, z- faces and the x- halo), so that three CTAs fit per SM.
struct Layout {
  int yl, yr, zl, zr, hl, hr;  // byte offsets within a stage (-1: not loaded)
  int stage;                   // bytes per stage (1024-aligned)
  int fa;                      // FA buffer offset
  int bar;                     // mbarrier offset
  int smem;                    // dynamic shared memory to request
};

inline Layout make_layout(bool lx, bool rx, bool ly, bool ry, bool lz, bool rz) {
  Layout L{};
  int off = MAIN;
  auto take = [&](bool need, int bytes) {
    if (!need) return -1;
    const int o = off;
    off += bytes;
    return o;
  };
  L.yl = take(ly, FACE);
  L.yr = take(ry, FACE);
  L.zl = take(lz, FACE);
  L.zr = take(rz, FACE);
  L.hl = take(lx, HALO);
  L.hr = take(rx, HALO);
  L.stage = ((off + 1023) / 1024) * 1024;
  L.fa = 2 * L.stage;
  L.bar = L.fa + MAIN;
  L.smem = L.bar + 64 + 1024;
  return L;
}

struct Maps {
  CUtensorMap main;   // 4-D {16, 4, cells, 4}, box {16, 4, E, 4}, swizzle 128B
  CUtensorMap yface;  // 5-D {4, 4, 4, cells, 4}, box {4, 1, 4, E, 4}
  CUtensorMap zface;  // 5-D, box {4, 4, 1, E, 4}
  CUtensorMap halo;   // 5-D, box {2, 4, 4, 1, 4}
  CUtensorMap w;      // 2-D {64, cells}, box {64, E}
};

__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

struct Need {
  bool lx, rx, ly, ry, lz, rz, w;
};

// Issue every TMA of segment `seg` into the stage at `sbase` (one thread).
__device__ __forceinline__ void issue(const Maps& m, const SlabArgs& a, const Need& nd,
                                      const Layout& L, int seg, unsigned char* sbase,
                                      uint32_t bar) {
  const int nx = a.g.nx, ny = a.g.ny, nz = a.g.nz;
  const int e0 = seg * E;
  const int cx0 = e0 % nx, cy = (e0 / nx) % ny, cz = e0 / (nx * ny);
  uint32_t bytes = MAIN;
  bytes += nd.ly ? FACE : 0;
  bytes += nd.ry ? FACE : 0;
  bytes += nd.lz ? FACE : 0;
  bytes += nd.rz ? FACE : 0;
  bytes += nd.lx ? HALO : 0;
  bytes += nd.rx ? HALO : 0;
  fast::mbar_expect_tx(bar, bytes);
  const uint32_t s = fast::smem_u32(sbase);
  fast::tma_load_4d(s, &m.main, bar, 0, 0, e0, 0);  // rows [t][cell][z]
  if (nd.ly) tma_load_5d(s + L.yl, &m.yface, bar, 0, 3, 0, e0 + ((cy == 0 ? ny - 1 : cy - 1) - cy) * nx, 0);
  if (nd.ry) tma_load_5d(s + L.yr, &m.yface, bar, 0, 0, 0, e0 + ((cy == ny - 1 ? 0 : cy + 1) - cy) * nx, 0);
  if (nd.lz) tma_load_5d(s + L.zl, &m.zface, bar, 0, 0, 3, e0 + ((cz == 0 ? nz - 1 : cz - 1) - cz) * nx * ny, 0);
  if (nd.rz) tma_load_5d(s + L.zr, &m.zface, bar, 0, 0, 0, e0 + ((cz == nz - 1 ? 0 : cz + 1) - cz) * nx * ny, 0);
  if (nd.lx) tma_load_5d(s + L.hl, &m.halo, bar, 2, 0, 0, e0 - cx0 + (cx0 == 0 ? nx - 1 : cx0 - 1), 0);
  if (nd.rx) {
    const int cxe = cx0 + E - 1;
    tma_load_5d(s + L.hr, &m.halo, bar, 0, 0, 0, e0 - cx0 + (cxe == nx - 1 ? 0 : cxe + 1), 0);
  }
}
}  // namespace pst

// RED: also max |R_i| and <R,R> (the Newton residual norm and the next
// GMRES right-hand side's norm), so no separate reduction pass reads R again
template <bool FULL_S, bool RED = false>
__global__ void __launch_bounds__(pst::THREADS, 3)
    slab3d_n4_persist(const __grid_constant__ pst::Maps maps, const SlabArgs a,
                      const pst::Layout lay) {
  pdl_entry();
  if (skip_now(a.skip)) return;
  using namespace pst;
  using fast::row_of;
  using fast::swz;
  extern __shared__ unsigned char smem_raw[];
  // align to 1024 B (128B-swizzle atoms) by integer offset so the pointer
  // keeps its shared-memory provenance (LDS/STS, not generic LD/ST)
  unsigned char* base = smem_raw + ((1024u - (fast::smem_u32(smem_raw) & 1023u)) & 1023u);
  double* FA = reinterpret_cast<double*>(base + lay.fa);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + lay.bar);
  const uint32_t bar0 = fast::smem_u32(bars), bar1 = fast::smem_u32(bars + 1);
  const int STG = lay.stage;

  const int tid = threadIdx.x;
  const long long ns = a.g.n_sdof;
  const int nseg = a.seg_end > 0 ? a.seg_end : a.g.n_cells / E;
  const Need nd{a.sp.cL[0] != 0.0, a.sp.cR[0] != 0.0, a.sp.cL[1] != 0.0, a.sp.cR[1] != 0.0,
                a.sp.cL[2] != 0.0, a.sp.cR[2] != 0.0, a.has_w != 0};

  if (tid == 0) {
    fast::mbar_init(bar0, 1);
    fast::mbar_init(bar1, 1);
    fast::fence_mbar_init();
  }
  __syncthreads();
  int seg = a.seg_begin + blockIdx.x;
  if (tid == 0 && seg < nseg) issue(maps, a, nd, lay, seg, base, bar0);

  // thread identities of the two phases.  (A warp-decoupled variant -- each
  // warp owning two cells in both phases, __syncwarp between them and
  // per-warp `empty` mbarriers instead of the CTA barriers -- measured 36 us
  // vs 29.7 us: the producer's empty-wait delays the next segment's TMA.)
  auto rowc = [](int t, int e, int z) { return (t * E + e) * 4 + z; };
  const int zA = tid & 3, eA = (tid >> 2) & (E - 1), tA = tid >> 5;
  const int xB = tid & 3, yB = (tid >> 2) & 3, eB = tid >> 4;
  const int qB = yB * 4 + xB;
  double rmax = 0.0, rss = 0.0;  // RED
  // u_n (the W term) is prefetched into registers one segment ahead
  double w[4] = {0, 0, 0, 0};
  if (nd.w && seg < nseg) {
    const double* p = a.W + (long long)(seg * E + eB) * 64 + qB;
#pragma unroll
    for (int z = 0; z < 4; ++z) w[z] = __ldcs(p + 16 * z);
  }

  for (int it = 0; seg < nseg; ++it, seg += gridDim.x) {
    const int st = it & 1;
    unsigned char* sb = base + st * STG;
    const double* Xs = reinterpret_cast<const double*>(sb);
    const int nxt = seg + gridDim.x;
    if (tid == 0) {
      if (nxt < nseg) {
        // stage st^1 was last read in iteration it-1, which ended with a CTA
        // barrier
        fence_proxy_async();
        issue(maps, a, nd, lay, nxt, base + (st ^ 1) * STG, st ? bar0 : bar1);
      }
    }
    double wn[4] = {0, 0, 0, 0};
    if (nd.w && nxt < nseg) {
      const double* p = a.W + (long long)(nxt * E + eB) * 64 + qB;
#pragma unroll
      for (int z = 0; z < 4; ++z) wn[z] = __ldcs(p + 16 * z);
    }
    while (!fast::mbar_try_wait(st ? bar1 : bar0, (it >> 1) & 1)) {
    }

    // ---- phase A: x and y derivatives of the (y,x) plane at (t, e, z) -----
    {
      const int row = rowc(tA, eA, zA);
      const int sw = row & 7;
      double u[16];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double2 v = *reinterpret_cast<const double2*>(Xs + row * 16 + ((c ^ sw) << 1));
        u[2 * c] = v.x;
        u[2 * c + 1] = v.y;
      }
      double hl[4] = {0, 0, 0, 0}, hr[4] = {0, 0, 0, 0};
      double yl[4] = {0, 0, 0, 0}, yr[4] = {0, 0, 0, 0};
      if (nd.lx) {
        if (eA > 0) {
          const int rl = rowc(tA, eA - 1, zA);
#pragma unroll
          for (int y = 0; y < 4; ++y) hl[y] = Xs[swz(rl, 4 * y + 3)];
        } else {
          const double* H = reinterpret_cast<const double*>(sb + lay.hl) + (tA * 4 + zA) * 8;
#pragma unroll
          for (int y = 0; y < 4; ++y) hl[y] = H[2 * y + 1];
        }
      }
      if (nd.rx) {
        if (eA < E - 1) {
          const int rr = rowc(tA, eA + 1, zA);
#pragma unroll
          for (int y = 0; y < 4; ++y) hr[y] = Xs[swz(rr, 4 * y)];
        } else {
          const double* H = reinterpret_cast<const double*>(sb + lay.hr) + (tA * 4 + zA) * 8;
#pragma unroll
          for (int y = 0; y < 4; ++y) hr[y] = H[2 * y];
        }
      }
      const int fo = ((tA * E + eA) * 4 + zA) * 4;
      if (nd.ly) {
        const double* Y = reinterpret_cast<const double*>(sb + lay.yl) + fo;
        const double2 v0 = *reinterpret_cast<const double2*>(Y);
        const double2 v1 = *reinterpret_cast<const double2*>(Y + 2);
        yl[0] = v0.x; yl[1] = v0.y; yl[2] = v1.x; yl[3] = v1.y;
      }
      if (nd.ry) {
        const double* Y = reinterpret_cast<const double*>(sb + lay.yr) + fo;
        const double2 v0 = *reinterpret_cast<const double2*>(Y);
        const double2 v1 = *reinterpret_cast<const double2*>(Y + 2);
        yr[0] = v0.x; yr[1] = v0.y; yr[2] = v1.x; yr[3] = v1.y;
      }
      double f[16];
#pragma unroll
      for (int y = 0; y < 4; ++y)
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          double g = 0.0;
#pragma unroll
          for (int k = 0; k < 4; ++k) g = fma(a.sp.V[0][x][k], u[4 * y + k], g);
#pragma unroll
          for (int k = 0; k < 4; ++k) g = fma(a.sp.V[1][y][k], u[4 * k + x], g);
          if (x == 0) g = fma(a.sp.cL[0], hl[y], g);
          if (x == 3) g = fma(a.sp.cR[0], hr[y], g);
          if (y == 0) g = fma(a.sp.cL[1], yl[x], g);
          if (y == 3) g = fma(a.sp.cR[1], yr[x], g);
          f[4 * y + x] = g;
        }
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<double2*>(FA + row * 16 + ((c ^ sw) << 1)) =
            make_double2(f[2 * c], f[2 * c + 1]);
    }
    __syncthreads();

    // ---- phase B: z derivative, temporal mixing, store ---------------------
    {
      const int e0 = seg * E;
      const int cellB = e0 + eB;
      double u[4][4], f[4][4];  // [t][z]
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          const int o = swz(rowc(t, eB, z), qB);
          u[t][z] = Xs[o];
          f[t][z] = FA[o];
        }
      double zl[4] = {0, 0, 0, 0}, zr[4] = {0, 0, 0, 0};
      if (nd.lz) {
        const double* Z = reinterpret_cast<const double*>(sb + lay.zl) + eB * 16 + qB;
#pragma unroll
        for (int t = 0; t < 4; ++t) zl[t] = Z[t * E * 16];
      }
      if (nd.rz) {
        const double* Z = reinterpret_cast<const double*>(sb + lay.zr) + eB * 16 + qB;
#pragma unroll
        for (int t = 0; t < 4; ++t) zr[t] = Z[t * E * 16];
      }
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          double g = f[t][z];
#pragma unroll
          for (int k = 0; k < 4; ++k) g = fma(a.sp.V[2][z][k], u[t][k], g);
          if (z == 0) g = fma(a.sp.cL[2], zl[t], g);
          if (z == 3) g = fma(a.sp.cR[2], zr[t], g);
          f[t][z] = g;
        }
      double* Rb = a.R + (long long)cellB * 64 + qB;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        // n_out < 4: only the first output blocks exist (the stage update
        // u_next = u + dt sum_j b_j F(U_j) has one)
        if (r >= a.n_out) break;
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          double acc = a.mx.c[r] * w[z];
#pragma unroll
          for (int j = 0; j < 4; ++j) acc = fma(a.mx.T[r][j], u[j][z], acc);
          if (FULL_S) {
#pragma unroll
            for (int j = 0; j < 4; ++j) acc = fma(a.mx.S[r][j], f[j][z], acc);
          } else {
            acc = fma(a.mx.S[r][r], f[r][z], acc);
          }
          Rb[r * ns + 16 * z] = acc;
          if (RED) {
            rmax = nan_max(rmax, fabs(acc));
            rss = fma(acc, acc, rss);
          }
        }
      }
    }
#pragma unroll
    for (int z = 0; z < 4; ++z) w[z] = wn[z];
    __syncthreads();  // stage st and FA free for reuse
  }
  if (RED) block_reduce_r(a, rmax, rss);
}

// ---------------------------------------------------------------------------
// host-side launch helpers
// ---------------------------------------------------------------------------
// blocks of the lane kernel: one lane per (element, temporal block), 32 / NT
// elements per warp, 8 warps per block
long long lane_blocks(long long nx, int nt) {
  const long long epw = 32 / nt;
  const long long warps = (nx + epw - 1) / epw;
  return (warps * 32 + 255) / 256;
}

// the Newton residual's fused reductions requested (and not an FD action);
// the reducing instance writes one partial per block, so its grid must fit
// the kPartialDoubles slots in front of the completion counter -- larger
// meshes take the plain kernel plus a separate reduction pass
bool lane_reduces(const SlabArgs& a) {
  return a.red_max != nullptr && a.red_ss != nullptr && a.red_part != nullptr &&
         a.fdv == nullptr && a.n_in >= 1 && lane_blocks(a.g.nx, a.n_in) <= kPartialDoubles;
}

template <int N1>
int launch1d(const SlabArgs& a, cudaStream_t s) {
  // large meshes: one lane per (element, temporal block) when n_in == n_tau
  // covers the mix (n_out <= n_in) and the lanes fill a warp evenly
  if (a.g.nx >= 4096 && a.n_out <= a.n_in && !std::getenv("STG_1D_V1")) {
    auto go = [&](auto nt_tag) {
      constexpr int NT = decltype(nt_tag)::value;
      const int blocks = int(lane_blocks(a.g.nx, NT));
      if (lane_reduces(a)) {
        cudaMemsetAsync(a.red_max, 0, sizeof(unsigned long long), s);
        launch_ex(kPdlSlab, slab1d_lane_kernel<N1, NT, true>, blocks, 256, 0, s, a);
      } else {
        launch_ex(kPdlSlab, slab1d_lane_kernel<N1, NT, false>, blocks, 256, 0, s, a);
      }
      return 1;
    };
    switch (a.n_in) {
      case 2: return go(std::integral_constant<int, 2>{});
      case 3: return go(std::integral_constant<int, 3>{});
      case 4: return go(std::integral_constant<int, 4>{});
      case 5: return go(std::integral_constant<int, 5>{});
      case 6: return go(std::integral_constant<int, 6>{});
      default: break;
    }
  }
  const int blocks = (a.g.nx + kThreads1d - 1) / kThreads1d;
  launch_ex(kPdlSlab, slab1d_kernel<N1>, blocks, kThreads1d, 0, s, a);
  return 1;
}

int num_sms_cached() {
  static int cache[kMaxDevices];
  const int dev = device_slot();
  int& n = cache[dev];
  if (!n) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n = v > 0 ? v : 148;
  }
  return n;
}

// E = 32 cells per segment for the plane kernel (lanes = cells)
static const int kPlaneEnv = [] {
  const char* v = std::getenv("STG_2D_PLANE_E");
  return v ? std::atoi(v) : 32;
}();

template <int N1, int NT, int E>
bool plane2d_ok(const SlabArgs& a) {
  using P = Plane2d<N1, NT, E>;
  return !a.full_s && a.n_in == NT && a.n_out == NT && a.g.n_cells % E == 0 &&
         (reinterpret_cast<uintptr_t>(a.X) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(a.R) & 15) == 0 &&
         (!a.has_w || (reinterpret_cast<uintptr_t>(a.W) & 15) == 0) && a.g.n_sdof % 2 == 0 &&
         P::SMEM <= 227 * 1024 && !std::getenv("STG_2D_V1");
}

template <int N1, int NT, int E>
bool plane3_ok(const SlabArgs& a) {
  return !a.full_s && a.n_in == NT && a.n_out == NT && a.g.n_cells % E == 0 &&
         (reinterpret_cast<uintptr_t>(a.X) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(a.R) & 15) == 0 && a.g.n_sdof % 2 == 0 &&
         Plane3<N1, NT, E>::SMEM <= 113 * 1024;
}

// the launch that ran last on this thread formed the residual norms (RED)
thread_local bool t_last_reduced = false;

template <int N1, int NT, int E>
int launch_plane3(const SlabArgs& a, cudaStream_t s) {
  using Q = Plane3<N1, NT, E>;
  static int occ_dev[kMaxDevices];
  int& occ = occ_dev[device_slot()];
  if (occ <= 0) {
    for (auto k : {slab2d_plane3<N1, NT, E, false>, slab2d_plane3<N1, NT, E, true>})
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Q::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, slab2d_plane3<N1, NT, E, true>, Q::THREADS,
                                                  Q::SMEM);
    if (occ < 1) occ = 1;
  }
  const int nseg = a.g.n_cells / E;
  int grid = occ * num_sms_cached();
  if (grid > nseg) grid = nseg;
  const bool red = a.red_max != nullptr && a.red_ss != nullptr && a.red_part != nullptr &&
                   a.seg_end == 0 && grid <= kPartialDoubles;
  if (red) cudaMemsetAsync(a.red_max, 0, sizeof(unsigned long long), s);  // the atomic max
  launch_ex(kPdlSlab, red ? slab2d_plane3<N1, NT, E, true> : slab2d_plane3<N1, NT, E, false>,
            grid, Q::THREADS, Q::SMEM, s, a);
  t_last_reduced = red;
  return 1;
}

template <int N1, int NT, int E, int MINB>
int launch_plane2d(const SlabArgs& a, cudaStream_t s) {
  using Q = Plane2d<N1, NT, E>;
  static int occ_dev[kMaxDevices];  // 0: not set up on that device yet
  int& occ = occ_dev[device_slot()];
  if (occ <= 0) {
    cudaFuncSetAttribute(slab2d_plane<N1, NT, E, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Q::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, slab2d_plane<N1, NT, E, MINB>,
                                                  Q::THREADS, Q::SMEM);
    if (occ < 1) occ = 1;
  }
  const int nseg = a.g.n_cells / E;
  int grid = occ * num_sms_cached();
  if (grid > nseg) grid = nseg;
  launch_ex(kPdlSlab, slab2d_plane<N1, NT, E, MINB>, grid, Q::THREADS, Q::SMEM, s, a);
  return 1;
}

template <int N1, int NT>
int launch2d_t(const SlabArgs& a, cudaStream_t s) {
  using Sh = Shape2d<N1, NT>;
  using P = P2d<N1, NT>;
  if constexpr (N1 <= 5) {  // n = 6 would spill the register tile
    if (a.x_bcast) {  // only the 3-stage plane kernel reads a one-block X
      static const bool p2b = std::getenv("STG_2D_PLANE2") != nullptr;
      if (!p2b && kPlaneEnv == 32 && plane3_ok<N1, NT, 32>(a))
        return launch_plane3<N1, NT, 32>(a, s);
      return -1;
    }
    if (kPlaneEnv == 16 && plane2d_ok<N1, NT, 16>(a)) return launch_plane2d<N1, NT, 16, 3>(a, s);
    if (kPlaneEnv == 33 && plane2d_ok<N1, NT, 32>(a)) return launch_plane2d<N1, NT, 32, 1>(a, s);
    // 2 CTAs/SM: caps the tile kernel at 200 registers (202 would round to
    // 6656 per warp and leave room for one 160-thread CTA only)
    // default: the 3-stage in-place plane kernel (c2 R(U) 31.9 -> 29.6 us);
    // STG_2D_PLANE2=1 keeps the 2-stage kernel with its output staging
    static const bool p2 = std::getenv("STG_2D_PLANE2") != nullptr;
    if (!p2 && kPlaneEnv == 32 && plane3_ok<N1, NT, 32>(a)) return launch_plane3<N1, NT, 32>(a, s);
    if (plane2d_ok<N1, NT, 32>(a)) return launch_plane2d<N1, NT, 32, 2>(a, s);
  }
  if (a.x_bcast) return -1;
  if (a.g.n_cells % Sh::E == 0 && (reinterpret_cast<uintptr_t>(a.X) & 15) == 0 &&
      (a.g.n_sdof % 2) == 0 && !std::getenv("STG_2D_NONPERSIST")) {
    static int occ_dev[kMaxDevices];
    int& occ = occ_dev[device_slot()];
    if (occ <= 0) {
      cudaFuncSetAttribute(slab2d_persist<N1, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           P::SMEM);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, slab2d_persist<N1, NT>, Sh::THREADS,
                                                    P::SMEM);
      if (occ < 1) occ = 1;
    }
    const int nseg = a.g.n_cells / Sh::E;
    int grid = occ * num_sms_cached();
    if (grid > nseg) grid = nseg;
    launch_ex(kPdlSlab, slab2d_persist<N1, NT>, grid, Sh::THREADS, P::SMEM, s, a);
    return 1;
  }
  const int blocks = (a.g.n_cells + Sh::E - 1) / Sh::E;
  launch_ex(kPdlSlab, slab2d_kernel<N1, NT>, blocks, Sh::THREADS, 0, s, a);
  return 1;
}

template <int N1>
int launch2d_n(const SlabArgs& a, cudaStream_t s) {
  switch (a.n_in) {
    case 1: return launch2d_t<N1, 1>(a, s);
    case 2: return launch2d_t<N1, 2>(a, s);
    case 3: return launch2d_t<N1, 3>(a, s);
    case 4: return launch2d_t<N1, 4>(a, s);
    case 5: return launch2d_t<N1, 5>(a, s);
    case 6: return launch2d_t<N1, 6>(a, s);
    default: return -1;
  }
}

template <int D, int N1>
int launch_generic_t(const SlabArgs& a, cudaStream_t s) {
  using Sh = GenericShape<D, N1>;
  const int blocks = (a.g.n_cells + Sh::E - 1) / Sh::E;
  const size_t smem = size_t(Sh::E) * kMaxT * Sh::NPC * sizeof(double);
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(slab_generic_kernel<D, N1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
  }
  launch_ex(kPdlSlab, slab_generic_kernel<D, N1>, blocks, Sh::THREADS, smem, s, a);
  return 1;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

}  // namespace

// the generic launchers reduce R only in the d = 1 lane kernel (the d = 2
// plane kernel's reducing instance spilled and gained nothing on c2)
bool slab_generic_reduces(const SlabArgs& a) {
  if (a.g.dim == 2) return t_last_reduced;  // (asked right after the launch)
  return a.g.dim == 1 && lane_reduces(a) && a.g.nx >= 4096 && a.n_out <= a.n_in &&
         a.n_in >= 2 && a.n_in <= 6 && a.g.n1 >= 2 && a.g.n1 <= 6 && !std::getenv("STG_1D_V1");
}

int launch_slab_generic(const SlabArgs& a, cudaStream_t s) {
  const int d = a.g.dim, n1 = a.g.n1;
  t_last_reduced = false;
  // a one-block X (x_bcast) is read by the d = 2 plane kernel only: -1
  // elsewhere, before anything is launched (the caller writes the broadcast
  // out and calls again)
  if (a.x_bcast && !(d == 2 && a.model == int(Model::advection) && a.n_out <= a.n_in &&
                     slab_fast_bcast_ok() && !std::getenv("STG_GENERIC_2D")))
    return -1;
  if (d == 1) {
    switch (n1) {
      case 2: return launch1d<2>(a, s);
      case 3: return launch1d<3>(a, s);
      case 4: return launch1d<4>(a, s);
      case 5: return launch1d<5>(a, s);
      case 6: return launch1d<6>(a, s);
      default: return -1;
    }
  }
  if (a.model != int(Model::advection)) return -1;
  if (d == 2 && a.n_out <= a.n_in && !std::getenv("STG_GENERIC_2D")) {
    switch (n1) {
      case 2: return launch2d_n<2>(a, s);
      case 3: return launch2d_n<3>(a, s);
      case 4: return launch2d_n<4>(a, s);
      case 5: return launch2d_n<5>(a, s);
      case 6: return launch2d_n<6>(a, s);
      default: return -1;
    }
  }
  if (d == 2) {
    switch (n1) {
      case 2: return launch_generic_t<2, 2>(a, s);
      case 3: return launch_generic_t<2, 3>(a, s);
      case 4: return launch_generic_t<2, 4>(a, s);
      case 5: return launch_generic_t<2, 5>(a, s);
      case 6: return launch_generic_t<2, 6>(a, s);
      default: return -1;
    }
  }
  if (d == 3) {
    switch (n1) {
      case 2: return launch_generic_t<3, 2>(a, s);
      case 3: return launch_generic_t<3, 3>(a, s);
      case 4: return launch_generic_t<3, 4>(a, s);
      case 5: return launch_generic_t<3, 5>(a, s);
      default: return -1;
    }
  }
  return -1;
}

bool fd_fused_supported(const SlabArgs& a) {
  return a.g.dim == 1 && a.model == int(Model::burgers) && a.g.nx >= 4096 &&
         a.n_out <= a.n_in && a.n_in >= 2 && a.n_in <= 6 && a.g.n1 >= 2 && a.g.n1 <= 6 &&
         !std::getenv("STG_1D_V1");
}

namespace {
int fast_variant();
}  // namespace

bool slab_fast_supported(const SlabArgs& a) {
  // n_out < 4 (fewer output blocks than stages: the stage update u_next) is
  // taken by the persistent kernel only
  const bool nout_ok = a.n_out == 4 || (a.n_out >= 1 && a.n_out < 4 && fast_variant() != 1);
  return a.g.dim == 3 && a.g.n1 == 4 && a.n_in == 4 && nout_ok &&
         a.model == int(Model::advection) && a.g.nx % fast::E == 0 &&
         (reinterpret_cast<uintptr_t>(a.X) & 15) == 0 && get_encode() != nullptr;
}

namespace {
bool encode(EncodeFn enc, CUtensorMap* map, const double* base, int rank, const cuuint64_t* gdim,
            const cuuint64_t* gstride, const cuuint32_t* box, CUtensorMapSwizzle swz) {
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(base), gdim, gstride,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int num_sms() { return num_sms_cached(); }

int fast_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("STG_FAST_VARIANT");
    v = e ? std::atoi(e) : 2;
  }
  return v;
}
}  // namespace

bool slab_fast_reduces(const SlabArgs& a) {
  return a.red_max != nullptr && a.red_ss != nullptr && a.red_part != nullptr &&
         a.seg_end == 0 && slab_fast_supported(a) && fast_variant() != 1;
}

// whether the driver encodes a tensor map whose temporal stride is 0 (X one
// spatial block read as all n_in: SlabArgs::x_bcast)
bool slab_fast_bcast_ok() {
  static const int ok = [] {
    EncodeFn enc = get_encode();
    if (!enc || std::getenv("STG_NO_LAZY_GUESS")) return 0;
    alignas(64) static double dummy[8];
    CUtensorMap map;
    const cuuint64_t gdim[4] = {16, 4, pst::E, 4};
    const cuuint64_t gstride[3] = {128, 512, 0};
    const cuuint32_t box[4] = {16, 4, pst::E, 4};
    return encode(enc, &map, dummy, 4, gdim, gstride, box, CU_TENSOR_MAP_SWIZZLE_128B) ? 1 : 0;
  }();
  return ok != 0;
}

int launch_slab_fast(const SlabArgs& a, cudaStream_t s) {
  EncodeFn enc = get_encode();
  if (!enc) return -1;
  if (a.x_bcast && !slab_fast_bcast_ok()) return -1;
  const cuuint64_t cells = cuuint64_t(a.g.n_cells);
  const cuuint64_t tstride = a.x_bcast ? 0 : cuuint64_t(a.g.n_sdof) * 8;
  if (fast_variant() == 1) {
    CUtensorMap map;
    const cuuint64_t gdim[4] = {16, 4, cells, 4};
    const cuuint64_t gstride[3] = {128, 512, tstride};
    const cuuint32_t box[4] = {16, 4, fast::E, 4};
    if (!encode(enc, &map, a.X, 4, gdim, gstride, box, CU_TENSOR_MAP_SWIZZLE_128B)) return -1;
    const int blocks = (a.seg_end > 0 ? a.seg_end : a.g.n_cells / fast::E) - a.seg_begin;
    if (blocks <= 0) return 0;
    if (a.full_s) {
      launch_ex(kPdlSlab, slab3d_n4_tma<true>, blocks, fast::THREADS, fast::SMEM_BYTES, s, map, a);
    } else {
      launch_ex(kPdlSlab, slab3d_n4_tma<false>, blocks, fast::THREADS, fast::SMEM_BYTES, s, map, a);
    }
    return 1;
  }
  pst::Maps m;
  {
    // dims {yx (16), z (4), cell, t}: [t][cell][z] rows of 128 B, so each
    // TMA streams 4 KB contiguous runs per temporal block (a cell-outermost
    // box, [cell][t][z], measured 36 us vs 30 us: 512 B runs)
    const cuuint64_t gdim[4] = {16, 4, cells, 4};
    const cuuint64_t gstride[3] = {128, 512, tstride};
    const cuuint32_t box[4] = {16, 4, pst::E, 4};
    if (!encode(enc, &m.main, a.X, 4, gdim, gstride, box, CU_TENSOR_MAP_SWIZZLE_128B)) return -1;
  }
  {
    const cuuint64_t gdim[5] = {4, 4, 4, cells, 4};
    const cuuint64_t gstride[4] = {32, 128, 512, tstride};
    const cuuint32_t by[5] = {4, 1, 4, pst::E, 4};
    const cuuint32_t bz[5] = {4, 4, 1, pst::E, 4};
    const cuuint32_t bh[5] = {2, 4, 4, 1, 4};
    if (!encode(enc, &m.yface, a.X, 5, gdim, gstride, by, CU_TENSOR_MAP_SWIZZLE_NONE)) return -1;
    if (!encode(enc, &m.zface, a.X, 5, gdim, gstride, bz, CU_TENSOR_MAP_SWIZZLE_NONE)) return -1;
    if (!encode(enc, &m.halo, a.X, 5, gdim, gstride, bh, CU_TENSOR_MAP_SWIZZLE_NONE)) return -1;
  }
  m.w = m.main;  // u_n is prefetched into registers (no TMA box)
  const pst::Layout lay =
      pst::make_layout(a.sp.cL[0] != 0.0, a.sp.cR[0] != 0.0, a.sp.cL[1] != 0.0,
                       a.sp.cR[1] != 0.0, a.sp.cL[2] != 0.0, a.sp.cR[2] != 0.0);
  const bool red = slab_fast_reduces(a);
  auto kern = a.full_s ? (red ? slab3d_n4_persist<true, true> : slab3d_n4_persist<true, false>)
                       : (red ? slab3d_n4_persist<false, true> : slab3d_n4_persist<false, false>);
  static bool attr_dev[kMaxDevices];
  bool& attr = attr_dev[device_slot()];
  if (!attr) {  // the largest layout (every trace buffer) bounds the request
    for (auto k : {slab3d_n4_persist<true, false>, slab3d_n4_persist<false, false>,
                   slab3d_n4_persist<true, true>, slab3d_n4_persist<false, true>})
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, pst::SMEM_BYTES);
    attr = true;
  }
  const int nseg = (a.seg_end > 0 ? a.seg_end : a.g.n_cells / pst::E) - a.seg_begin;
  if (nseg <= 0) return 0;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, pst::THREADS, lay.smem);
  static int per_sm_cap = [] {
    const char* e = std::getenv("STG_FAST_CTAS_PER_SM");
    return e ? std::atoi(e) : 3;
  }();
  if (occ > per_sm_cap) occ = per_sm_cap;
  if (occ < 1) occ = 1;
  int grid = occ * num_sms();
  if (grid > nseg) grid = nseg;
  // STG_FAST_GRID=g: A/B knob for the persistent grid size (scripts/grid_sweep.sh:
  // 410 CTAs, ten equal rounds of the 4096 c4 segments, is no faster than 444)
  static const int grid_env = [] {
    const char* e = std::getenv("STG_FAST_GRID");
    return e ? std::atoi(e) : 0;
  }();
  if (grid_env > 0 && grid_env < grid) grid = grid_env;
  if (red) cudaMemsetAsync(a.red_max, 0, sizeof(unsigned long long), s);
  launch_ex(a.no_pdl ? 0 : kPdlSlab, kern, grid, pst::THREADS, lay.smem, s, m, a, lay);
  return 1;
}

}  // namespace stg
