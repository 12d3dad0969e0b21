// Block-Jacobi preconditioners for the slab / stage Jacobians (right
// preconditioning inside GMRES; "start with Jacobi ...
// then temporal-block (N_tau x N_tau per spatial node) or element-block").
//
//  * temporal-block Jacobi (TBJ): for every spatial node, the n_tau x n_tau
//    diagonal block T + v_k S of the linear-advection slab Jacobian, where
//    v_k = sum_a V_a(i_a, i_a) depends only on the node's position in the cell
//    (its "class").  The host inverts the npc class blocks; the apply kernel is
//    one HBM pass (read n_dof, write n_dof).
//  * element-block Jacobi (EBJ, d = 1): the exact element-local block of the
//    Jacobian, (n_tau*n1)^2 per element, inverted on the device.  For linear
//    advection all elements share one block; for Burgers the blocks depend on
//    the state and are rebuilt per Newton iteration from the exact
//    linearisation.
#include "kernels.hpp"

namespace stg {
namespace {

constexpr int kPB = 256;

// out[t][cell][k] = sum_j Minv[k][t][j] in[j][cell][k].  The class table
// (npc * NT^2 doubles) is staged in shared memory; the cell loop is
// grid-strided in 32-bit cell units so the node class is threadIdx-derived.
template <int NT>
__global__ void __launch_bounds__(kPB) k_tblock(double* __restrict__ out,
                                                const double* __restrict__ in,
                                                const double* __restrict__ minv, int npc,
                                                int ncells, long long ns) {
  // smem layout [t][j][k]: consecutive nodes (threads) read consecutive words
  // (the global table is [k][t][j]; a [k]-major smem copy would be a 32-way
  // bank conflict for npc = 64)
  extern __shared__ double tab[];
  for (int q = threadIdx.x; q < npc * NT * NT; q += blockDim.x) {
    const int k = q / (NT * NT), tj = q - k * NT * NT;
    tab[tj * npc + k] = minv[q];
  }
  __syncthreads();
  const unsigned total = unsigned(ncells) * unsigned(npc);  // < 2^31 (checked on the host)
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int k = int(i % unsigned(npc));
    double x[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) x[j] = __ldcs(in + j * ns + i);
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < NT; ++j) acc = fma(tab[(t * NT + j) * npc + k], x[j], acc);
      out[t * ns + i] = acc;
    }
  }
}

// out_e = B_e in_e over the element's nt*n1 DOFs (gathered from the
// stage-major layout); one warp per element, lane r computes row r (nb <= 32).
template <int NB>
__global__ void __launch_bounds__(256) k_eblock(double* __restrict__ out,
                                                const double* __restrict__ in,
                                                const double* __restrict__ B, long long bstride,
                                                int nt, int n1, int ncells, long long ns) {
  __shared__ double xs[8][NB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nb = nt * n1;
  for (int c = blockIdx.x * 8 + wid; c < ncells; c += gridDim.x * 8) {
    for (int r = lane; r < nb; r += 32) {
      const int t = r / n1, k = r - t * n1;
      xs[wid][r] = in[t * ns + (long long)c * n1 + k];
    }
    __syncwarp();
    const double* Bc = B + (size_t)c * bstride;
    for (int r = lane; r < nb; r += 32) {
      double acc = 0.0;
      for (int q = 0; q < nb; ++q) acc = fma(Bc[(size_t)r * nb + q], xs[wid][q], acc);
      const int t = r / n1, k = r - t * n1;
      out[t * ns + (long long)c * n1 + k] = acc;
    }
    __syncwarp();
  }
}

// Build and invert the element blocks of the 1-D Burgers slab / stage Jacobian
// at U: column (j, q) = element response to a unit input at temporal node j,
// node q (neighbour inputs zero; neighbour STATES enter through the exact
// linearisation).  One thread per element; Gauss-Jordan with partial
// pivoting on a thread-private (local-memory) nb x 2nb tableau.
template <int N1>
__global__ void __launch_bounds__(128) k_build_burgers_eblock(double* __restrict__ Binv,
                                                              const double* __restrict__ U,
                                                              const SlabArgs a) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int K = a.g.nx;
  if (c >= K) return;
  const int nt = a.n_in;
  const int nb = nt * N1;
  const long long ns = a.g.n_sdof;
  const int cl = c == 0 ? K - 1 : c - 1, cr = c == K - 1 ? 0 : c + 1;
  double* M = Binv + (size_t)c * nb * nb;  // built in place, then inverted
  double aug[kMaxT * N1][kMaxT * N1];       // local memory
  // J_F(U_j) restricted to the element, for every temporal node j
  double jf[kMaxT][N1][N1];
  for (int j = 0; j < nt; ++j) {
    double u[N1];
    for (int i = 0; i < N1; ++i) u[i] = U[j * ns + (long long)c * N1 + i];
    const double ul = U[j * ns + (long long)cl * N1 + N1 - 1];
    const double ur = U[j * ns + (long long)cr * N1];
    for (int q = 0; q < N1; ++q) {
      // derivative of F_i w.r.t. u_q (own element; neighbours held fixed)
      for (int i = 0; i < N1; ++i) {
        double vol = 0.0;
        for (int k = 0; k < N1; ++k) {
          const double dvi = (i == q ? 1.0 : 0.0), dvk = (k == q ? 1.0 : 0.0);
          vol += 2.0 * a.sp.Dm[i][k] *
                 ((2.0 * u[i] + u[k]) * dvi + (u[i] + 2.0 * u[k]) * dvk) / 6.0;
        }
        double g = -a.sp.sc * vol;
        if (i == N1 - 1 && q == N1 - 1) {
          // d/duL of LLF(uL, ur) - f(uL) at the right face
          const double aL = fabs(u[N1 - 1]), aR = fabs(ur);
          double dH;
          if (aL >= aR)
            dH = 0.5 * u[N1 - 1] + 0.5 * (u[N1 - 1] >= 0 ? 1.0 : -1.0) * (u[N1 - 1] - ur) + 0.5 * aL;
          else
            dH = 0.5 * u[N1 - 1] + 0.5 * aR;
          g -= a.sp.sc * (dH - u[N1 - 1]) * a.sp.inv_wN;
        }
        if (i == 0 && q == 0) {
          // d/duR of LLF(ul, uR) - f(uR) at the left face
          const double aL = fabs(ul), aR = fabs(u[0]);
          double dH;
          if (aL >= aR)
            dH = 0.5 * u[0] - 0.5 * aL;
          else
            dH = 0.5 * u[0] + 0.5 * (u[0] >= 0 ? 1.0 : -1.0) * (ul - u[0]) - 0.5 * aR;
          g += a.sp.sc * (dH - u[0]) * a.sp.inv_w0;
        }
        jf[j][i][q] = g;
      }
    }
  }
  // block (r,i),(j,q) = T(r,j) delta_iq + S(r,j) jf[j][i][q]
  for (int r = 0; r < nt; ++r)
    for (int i = 0; i < N1; ++i)
      for (int j = 0; j < nt; ++j)
        for (int q = 0; q < N1; ++q) {
          aug[r * N1 + i][j * N1 + q] =
              (i == q ? a.mx.T[r][j] : 0.0) + a.mx.S[r][j] * jf[j][i][q];
        }
  // invert in place (Gauss-Jordan, partial pivoting), result to M
  double inv[kMaxT * N1][kMaxT * N1];
  for (int r = 0; r < nb; ++r)
    for (int q = 0; q < nb; ++q) inv[r][q] = r == q ? 1.0 : 0.0;
  for (int col = 0; col < nb; ++col) {
    int p = col;
    for (int r = col + 1; r < nb; ++r)
      if (fabs(aug[r][col]) > fabs(aug[p][col])) p = r;
    if (p != col)
      for (int q = 0; q < nb; ++q) {
        double t0 = aug[col][q];
        aug[col][q] = aug[p][q];
        aug[p][q] = t0;
        t0 = inv[col][q];
        inv[col][q] = inv[p][q];
        inv[p][q] = t0;
      }
    const double piv = aug[col][col];
    const double ip = 1.0 / piv;
    for (int q = 0; q < nb; ++q) {
      aug[col][q] *= ip;
      inv[col][q] *= ip;
    }
    for (int r = 0; r < nb; ++r) {
      if (r == col) continue;
      const double f = aug[r][col];
      if (f == 0.0) continue;
      for (int q = 0; q < nb; ++q) {
        aug[r][q] = fma(-f, aug[col][q], aug[r][q]);
        inv[r][q] = fma(-f, inv[col][q], inv[r][q]);
      }
    }
  }
  for (int r = 0; r < nb; ++r)
    for (int q = 0; q < nb; ++q) M[(size_t)r * nb + q] = inv[r][q];
}

int pgrid(long long n) {
  long long g = (n + kPB - 1) / kPB;
  if (g > 148 * 8) g = 148 * 8;
  return int(g < 1 ? 1 : g);
}

}  // namespace

void precond_tblock(double* out, const double* in, const double* minv, int nt, int npc,
                    long long ns, cudaStream_t s) {
  const int ncells = int(ns / npc);  // ns < 2^31 for every supported mesh (validate_desc)
  const size_t smem = size_t(npc) * nt * nt * sizeof(double);
  const int g = pgrid(ns);
  switch (nt) {
    case 2: k_tblock<2><<<g, kPB, smem, s>>>(out, in, minv, npc, ncells, ns); break;
    case 3: k_tblock<3><<<g, kPB, smem, s>>>(out, in, minv, npc, ncells, ns); break;
    case 4: k_tblock<4><<<g, kPB, smem, s>>>(out, in, minv, npc, ncells, ns); break;
    case 5: k_tblock<5><<<g, kPB, smem, s>>>(out, in, minv, npc, ncells, ns); break;
    default: k_tblock<6><<<g, kPB, smem, s>>>(out, in, minv, npc, ncells, ns); break;
  }
}

void precond_eblock(double* out, const double* in, const double* B, long long bstride, int nt,
                    int n1, int ncells, long long ns, cudaStream_t s) {
  int g = (ncells + 7) / 8;
  if (g > 148 * 16) g = 148 * 16;
  k_eblock<kMaxT * kMaxN><<<g, 256, 0, s>>>(out, in, B, bstride, nt, n1, ncells, ns);
}

bool build_burgers_eblock(double* Binv, const double* U, const SlabArgs& a, cudaStream_t s) {
  const int blocks = (a.g.nx + 127) / 128;
  switch (a.g.n1) {
    case 2: k_build_burgers_eblock<2><<<blocks, 128, 0, s>>>(Binv, U, a); return true;
    case 3: k_build_burgers_eblock<3><<<blocks, 128, 0, s>>>(Binv, U, a); return true;
    case 4: k_build_burgers_eblock<4><<<blocks, 128, 0, s>>>(Binv, U, a); return true;
    default: return false;
  }
}

}  // namespace stg
