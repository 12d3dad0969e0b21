// Fused small-problem solver: a whole Newton-GMRES slab / stage solve in ONE
// launch of ONE thread block, for 1-D advection problems that fit in shared
// memory (the c1 configuration: 1,024 DOF).  Such solves are latency bound:
// the host-driven path pays a kernel launch per vector operation and a
// device->host round trip per Arnoldi step (~80 us per GMRES iteration at
// c1).  Here every step stays on the SM: the slab operator (restating
// SpatialOperator::rhs spatial.hpp:107-266 + the slab / stage mix,
// kernels.hpp), the element-block preconditioner, classical Gram-Schmidt
// Arnoldi with the same Pythagorean normalisation and DGKS re-orthogonalisation
// test as the host GMRES (stg.cpp), Givens rotations, back substitution and
// the Newton loop of newton_solve (newton.hpp:102-130).  Work vectors live in
// shared memory; the Krylov basis (n_dof * (m+1) doubles) lives in global
// memory and stays L2-resident.  Block reductions are fixed-order, so results
// are deterministic.
#include <cmath>

#include "kernels.hpp"

namespace stg {
namespace {

constexpr int kSmallThreads = 256;
constexpr int kDotMax = kSmallMaxRestart + 2;  // dots per fused pass
constexpr int kWarps = kSmallThreads / 32;

struct SmallShared {
  double* U;    // Newton iterate (n)
  double* R;    // residual / rhs (n)
  double* du;   // Newton update = GMRES solution (n)
  double* z;    // preconditioned vector / scratch (n)
  double* w;    // Arnoldi vector (n)
  double* W;    // u_n or u (ns)
  double* B;    // element-block inverse (nb * nb) or null
};

__device__ __forceinline__ double warp_sum_s(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Krylov basis: the first `in_smem` vectors live in shared memory (stride n),
// the rest in global memory (stride ld, L2-resident).
struct Basis {
  double* sm;
  double* gl;
  int in_smem;
  int n;
  long long ld;
  __device__ double* operator()(int j) const {
    return j < in_smem ? sm + (long long)j * n : gl + (long long)(j - in_smem) * ld;
  }
};

// out[j] = <V_j, x> for j < cnt: warp w reduces vectors j = w, w + kWarps, ...
// over all n entries (lane-strided, fixed order), so the code stays compact
// (a single-CTA latency-bound kernel is sensitive to instruction-cache misses).
__device__ __noinline__ void basis_dots(const Basis& V, int cnt, const double* x, int n, double* out) {
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  for (int j = wp; j < cnt; j += kWarps) {
    const double* v = V(j);
    double p = 0.0;
#pragma unroll 4
    for (int i = lane; i < n; i += 32) p = fma(v[i], x[i], p);
    p = warp_sum_s(p);
    if (lane == 0) out[j] = p;
  }
  __syncthreads();
}

// out[0] = <x, y>
__device__ __noinline__ void block_dot(const double* x, const double* y, int n, double (*red)[kDotMax + 1],
                          double* out) {
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  double p = 0.0;
  for (int i = threadIdx.x; i < n; i += kSmallThreads) p = fma(x[i], y[i], p);
  p = warp_sum_s(p);
  if (lane == 0) red[wp][0] = p;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < kWarps; ++q) s += red[q][0];
    out[0] = s;
  }
  __syncthreads();
}

__device__ __noinline__ double block_maxabs(const double* x, int n, double (*red)[kDotMax + 1]) {
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  double m = 0.0;
  for (int i = threadIdx.x; i < n; i += kSmallThreads) m = fmax(m, fabs(x[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  if (lane == 0) red[wp][0] = m;
  __syncthreads();
  double r = 0.0;
  for (int q = 0; q < kWarps; ++q) r = fmax(r, red[q][0]);
  __syncthreads();
  return r;
}

// R = sum_j T X_j + sum_j S F(X_j) + c W over n_out blocks (1-D advection);
// one thread per (cell, node).  X, R may live in shared or global memory.
// Coefficients staged in shared memory: V (N1 x N1), cL, cR of axis 0 and the
// three mixes T / S / c (kernel parameters indexed by lane-divergent values
// would serialise in the constant cache).
struct SmallCoef {
  double V[kMaxN][kMaxN];
  double cL, cR;
  MixCoef mx[3];  // residual, Jacobian, rk u_next
};

template <int N1>
__device__ __noinline__ void apply_1d(const SmallCoef& sc, const MixCoef& mx, int nt, int n_out,
                         const double* X, const double* W, double* R, int K, long long ns) {
  for (int q = threadIdx.x; q < K * N1; q += kSmallThreads) {
    const int c = q / N1, i = q - (q / N1) * N1;
    const int cl = c == 0 ? K - 1 : c - 1, cr = c == K - 1 ? 0 : c + 1;
    const double wv = W ? W[c * N1 + i] : 0.0;
    for (int r = 0; r < n_out; ++r) {
      double acc = mx.c[r] * wv;
      for (int j = 0; j < nt; ++j) {
        const double* Xj = X + j * ns;
        double g = 0.0;
        if (mx.S[r][j] != 0.0) {  // F(X_j) at node i (recomputed per output row)
#pragma unroll
          for (int k = 0; k < N1; ++k) g = fma(sc.V[i][k], Xj[c * N1 + k], g);
          if (i == 0) g = fma(sc.cL, Xj[cl * N1 + N1 - 1], g);
          if (i == N1 - 1) g = fma(sc.cR, Xj[cr * N1], g);
        }
        acc = fma(mx.T[r][j], Xj[c * N1 + i], acc);
        acc = fma(mx.S[r][j], g, acc);
      }
      R[r * ns + c * N1 + i] = acc;
    }
  }
}

// out = P^-1 in: element-block (nb = nt*N1) inverse B, or the identity
template <int N1>
__device__ __noinline__ void precond_1d(const double* B, int nt, const double* in, double* out, int K,
                           long long ns) {
  const int nb = nt * N1;
  for (int q = threadIdx.x; q < K * nb; q += kSmallThreads) {
    const int c = q / nb, row = q - (q / nb) * nb;
    const int r = row / N1, i = row - (row / N1) * N1;
    if (!B) {
      out[r * ns + c * N1 + i] = in[r * ns + c * N1 + i];
      continue;
    }
    double acc = 0.0;
    for (int col = 0; col < nb; ++col) {
      const int j = col / N1, k = col - (col / N1) * N1;
      acc = fma(B[row * (nb + 1) + col], in[j * ns + c * N1 + k], acc);  // odd pitch
    }
    out[r * ns + c * N1 + i] = acc;
  }
}

template <int N1>
__global__ void __launch_bounds__(kSmallThreads)
    small_solve_kernel(const __grid_constant__ SmallSolveArgs a) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double red[kWarps][kDotMax + 1];
  __shared__ double Hs[kSmallMaxRestart + 1][kSmallMaxRestart];
  __shared__ double gs[kSmallMaxRestart + 1], cs[kSmallMaxRestart], sn[kSmallMaxRestart];
  __shared__ double ys[kSmallMaxRestart], hv[kDotMax], hv2[kDotMax];
  __shared__ double bc[8];  // broadcast scalars
  __shared__ int flags[4];
  const int n = a.n, K = a.K, nt = a.nt, m = a.restart;
  const long long ns = a.ns;
  SmallShared s;
  s.U = smem;
  s.R = s.U + n;
  s.du = s.R + n;
  s.z = s.du + n;
  s.w = s.z + n;
  s.W = s.w + n;
  s.B = a.B ? s.W + ns : nullptr;
  // basis: as many vectors as fit in the rest of the dynamic shared memory
  Basis V;
  V.sm = s.W + ns + (a.B ? (nt * N1) * (nt * N1 + 1) : 0);
  V.gl = a.V;
  V.in_smem = a.basis_in_smem;
  V.n = n;
  V.ld = a.ld;
  const int nb = nt * N1;
  __shared__ SmallCoef sc;
  if (threadIdx.x == 0) {
    for (int i = 0; i < N1; ++i)
      for (int k = 0; k < N1; ++k) sc.V[i][k] = a.sp.V[0][i][k];
    sc.cL = a.sp.cL[0];
    sc.cR = a.sp.cR[0];
    sc.mx[0] = a.mx_res;
    sc.mx[1] = a.mx_jac;
    sc.mx[2] = a.mx_next;
  }
  for (int i = threadIdx.x; i < ns; i += kSmallThreads) s.W[i] = a.W[i];
  if (s.B)
    for (int i = threadIdx.x; i < nb * nb; i += kSmallThreads)
      s.B[(i / nb) * (nb + 1) + i % nb] = a.B[i];
  // initial guess 1 (x) W (stdg.hpp:131, lodg.hpp:131)
  for (int i = threadIdx.x; i < n; i += kSmallThreads) s.U[i] = a.W[i % ns];
  __syncthreads();

  auto residual = [&]() {
    apply_1d<N1>(sc, sc.mx[0], nt, nt, s.U, s.W, s.R, K, ns);
    __syncthreads();
  };
  // Jacobian action w = J x (the mix without the constant coupling)
  auto jac = [&](const double* x, double* y) {
    apply_1d<N1>(sc, sc.mx[1], nt, nt, x, nullptr, y, K, ns);
    __syncthreads();
  };

  residual();
  double norm = block_maxabs(s.R, n, red);
  const double norm0 = norm;
  int newton_it = 0, lin_total = 0, nhist = 0, status = 0;
  double final_rel = 0.0;
  if (threadIdx.x == 0) a.out->history[nhist] = norm;
  ++nhist;
  while (!(norm <= a.abs_tol || norm <= a.rel_tol * norm0)) {
    if (newton_it >= a.max_iter) {
      status = 1;  // NonconvergenceError
      break;
    }
    // b = -R, du = 0
    for (int i = threadIdx.x; i < n; i += kSmallThreads) {
      s.R[i] = -s.R[i];
      s.du[i] = 0.0;
    }
    __syncthreads();
    block_dot(s.R, s.R, n, red, bc);
    const double bnorm = sqrt(bc[0]);
    int total = 0;
    bool conv = bnorm == 0.0;
    // a NaN / infinite residual fails the linear solve at once (the
    // reference's GMRES does not converge on it, newton.hpp:74-76)
    const bool finite = isfinite(bnorm);
    double rel = finite ? 0.0 : bnorm;
    while (!conv && finite) {
      // r = b - J du  -> V_0 = r / ||r||
      jac(s.du, s.w);
      for (int i = threadIdx.x; i < n; i += kSmallThreads) s.w[i] = s.R[i] - s.w[i];
      __syncthreads();
      block_dot(s.w, s.w, n, red, bc);
      const double beta = sqrt(bc[0]);
      rel = beta / bnorm;
      if (rel <= a.tol) {
        conv = true;
        break;
      }
      if (total >= a.max_it) break;
      for (int i = threadIdx.x; i < n; i += kSmallThreads) V(0)[i] = s.w[i] / beta;
      if (threadIdx.x == 0) {
        for (int i = 0; i <= m; ++i) gs[i] = 0.0;
        gs[0] = beta;
      }
      __syncthreads();
      int k = 0;
      for (; k < m && total < a.max_it; ++k) {
        ++total;
        double* vn = V(k + 1);
        precond_1d<N1>(s.B, nt, V(k), s.z, K, ns);
        __syncthreads();
        jac(s.z, s.w);
        const int kk = k + 1;
        // [h_0..h_k, <w,w>]
        // [h_0..h_k, <w,w>] in one pass: V_{k+1} holds w for the fused dot
        for (int i = threadIdx.x; i < n; i += kSmallThreads) vn[i] = s.w[i];
        __syncthreads();
        basis_dots(V, kk + 1, s.w, n, hv);
        if (threadIdx.x == 0) {
          const double ww = hv[kk];
          double hh = 0.0;
          for (int j = 0; j < kk; ++j) hh += hv[j] * hv[j];
          const double est = ww - hh;
          bc[1] = est > 1e-28 * ww ? 1.0 / sqrt(est) : (ww > 0.0 ? 1.0 / sqrt(ww) : 1.0);
          bc[2] = ww;
          bc[3] = hh;
        }
        __syncthreads();
        const double sc = bc[1];
        for (int i = threadIdx.x; i < n; i += kSmallThreads) {
          double v = s.w[i];
          for (int j = 0; j < kk; ++j) v = fma(-hv[j], V(j)[i], v);
          vn[i] = v * sc;
        }
        __syncthreads();
        block_dot(vn, vn, n, red, bc + 4);  // <vn, vn> after scaling
        const double ww = bc[2], hh = bc[3], nv2 = bc[4];
        const double sigma = 1.0 / sc;
        double hn = sigma;
        if (threadIdx.x == 0)
          for (int j = 0; j < kk; ++j) Hs[j][k] = hv[j];
        if (!(ww - hh > 1e-4 * ww) || fabs(nv2 - 1.0) > 1e-10) {
          // one more classical Gram-Schmidt pass on the stored vector
          basis_dots(V, kk, vn, n, hv2);
          for (int i = threadIdx.x; i < n; i += kSmallThreads) {
            double v = vn[i];
            for (int j = 0; j < kk; ++j) v = fma(-hv2[j], V(j)[i], v);
            vn[i] = v;
          }
          __syncthreads();
          block_dot(vn, vn, n, red, bc + 5);
          const double nrm2 = bc[5];
          const double inv = nrm2 > 0.0 ? 1.0 / sqrt(nrm2) : 1.0;
          for (int i = threadIdx.x; i < n; i += kSmallThreads) vn[i] *= inv;
          if (threadIdx.x == 0)
            for (int j = 0; j < kk; ++j) Hs[j][k] += sigma * hv2[j];
          hn = sigma * sqrt(nrm2);
          __syncthreads();
        }
        if (!(ww > 0.0)) hn = 0.0;
        if (threadIdx.x == 0) {
          Hs[k + 1][k] = hn;
          for (int j = 0; j < k; ++j) {
            const double t0 = cs[j] * Hs[j][k] + sn[j] * Hs[j + 1][k];
            Hs[j + 1][k] = -sn[j] * Hs[j][k] + cs[j] * Hs[j + 1][k];
            Hs[j][k] = t0;
          }
          const double den = hypot(Hs[k][k], Hs[k + 1][k]);
          cs[k] = den == 0.0 ? 1.0 : Hs[k][k] / den;
          sn[k] = den == 0.0 ? 0.0 : Hs[k + 1][k] / den;
          Hs[k][k] = den;
          Hs[k + 1][k] = 0.0;
          gs[k + 1] = -sn[k] * gs[k];
          gs[k] = cs[k] * gs[k];
          flags[0] = (fabs(gs[k + 1]) / bnorm <= a.tol || hn == 0.0 || !isfinite(hn)) ? 1 : 0;
        }
        __syncthreads();
        if (flags[0]) {
          ++k;
          break;
        }
      }
      // y = H^-1 g, du += P^-1 (V y)
      if (threadIdx.x == 0) {
        for (int i = k - 1; i >= 0; --i) {
          double acc = gs[i];
          for (int j = i + 1; j < k; ++j) acc -= Hs[i][j] * ys[j];
          ys[i] = acc / Hs[i][i];
        }
      }
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += kSmallThreads) {
        double v = 0.0;
        for (int j = 0; j < k; ++j) v = fma(ys[j], V(j)[i], v);
        s.w[i] = v;
      }
      __syncthreads();
      precond_1d<N1>(s.B, nt, s.w, s.z, K, ns);
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += kSmallThreads) s.du[i] += s.z[i];
      __syncthreads();
    }
    lin_total += total;
    final_rel = rel;
    if (!conv) {
      status = 2;  // linear_solve: GMRES did not converge
      break;
    }
    for (int i = threadIdx.x; i < n; i += kSmallThreads) s.U[i] += s.du[i];
    __syncthreads();
    ++newton_it;
    residual();
    norm = block_maxabs(s.R, n, red);
    if (threadIdx.x == 0 && nhist < STG_MAX_HISTORY_DEV) a.out->history[nhist] = norm;
    ++nhist;
  }
  // results
  for (int i = threadIdx.x; i < n; i += kSmallThreads) a.U_out[i] = s.U[i];
  if (a.u_next) {
    if (a.rk) {  // u_next = u + dt sum_j b_j F(U_j)  (lodg.hpp:142-145)
      apply_1d<N1>(sc, sc.mx[2], nt, 1, s.U, s.W, a.u_next, K, ns);
    } else {
      for (int i = threadIdx.x; i < ns; i += kSmallThreads) a.u_next[i] = s.U[(nt - 1) * ns + i];
    }
  }
  if (threadIdx.x == 0) {
    a.out->status = status;
    a.out->newton_iterations = newton_it;
    a.out->linear_iterations = lin_total;
    a.out->final_residual = norm;
    a.out->n_history = nhist < STG_MAX_HISTORY_DEV ? nhist : STG_MAX_HISTORY_DEV;
    a.out->gmres_rel = final_rel;
  }
}

}  // namespace

size_t small_solve_smem(int n, long long ns, int nb, bool precond) {
  return sizeof(double) * (5 * size_t(n) + size_t(ns) + (precond ? size_t(nb) * (nb + 1) : 0));
}
constexpr size_t kSmallDynMax = 200 * 1024;  // dynamic shared memory budget

bool small_solve_supported(const Geometry& g, int nt, int model, int restart) {
  const int nb = nt * g.n1;
  const int n = int(g.n_sdof) * nt;
  return g.dim == 1 && model == int(Model::advection) && restart >= 1 &&
         restart <= kSmallMaxRestart && g.n1 >= 2 && g.n1 <= 6 &&
         small_solve_smem(n, g.n_sdof, nb, true) <= 200 * 1024 && n <= 16384;
}

int launch_small_solve(SmallSolveArgs a, cudaStream_t s) {
  const size_t base = small_solve_smem(a.n, a.ns, a.nt * a.n1, a.B != nullptr);
  const size_t vec = sizeof(double) * size_t(a.n);
  int fit = base < kSmallDynMax ? int((kSmallDynMax - base) / vec) : 0;
  if (fit > a.restart + 1) fit = a.restart + 1;
  a.basis_in_smem = fit;
  const size_t smem = base + size_t(fit) * vec;
  switch (a.n1) {
#define STG_SMALL_CASE(N)                                                                     \
  case N:                                                                                     \
    cudaFuncSetAttribute(small_solve_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         int(smem));                                                          \
    small_solve_kernel<N><<<1, kSmallThreads, smem, s>>>(a);                                  \
    return 1;
    STG_SMALL_CASE(2)
    STG_SMALL_CASE(3)
    STG_SMALL_CASE(4)
    STG_SMALL_CASE(5)
    STG_SMALL_CASE(6)
#undef STG_SMALL_CASE
    default:
      return -1;
  }
}

}  // namespace stg
