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
#include <algorithm>
#include <type_traits>

#include "kernels.hpp"
#include "krylov.cuh"

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
                                                int ncells, long long ns, Skip skip) {
  pdl_entry();
  if (skip_now(skip)) return;
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
                                                int nt, int n1, int ncells, long long ns,
                                                Skip skip) {
  pdl_entry();
  if (skip_now(skip)) return;
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
// linearisation).  Two elements per warp: lane (h, l) with l < NB owns row
// l = (r, i) of element 2w + h's block and of the identity, in registers.
// In-place Gauss-Jordan with partial pivoting WITHOUT row exchanges: at
// column `col` the unused lane of the half with the largest |a[col]| (four
// xor-shuffles of a key from the magnitude's top 28 bits and the lane,
// lowest lane on ties) becomes the
// pivot, normalises its row (the pivot entry becomes 1/pivot) and publishes
// it through shared memory (one 16-byte load per two entries for the other
// lanes); every other lane eliminates it (its own pivot-column entry
// becomes -a[col]/pivot).  At the end the pivot lane of column col holds
// row col of the inverse, its entry at position c' belonging to column
// piv[c'].  (The augmented [A | I] version with a shuffle-tree pivot search
// took 198 us for the 65,536 c3 blocks; one element per warp with shuffled
// rows 853 us.)
//
// With G != nullptr it also forms the inflow coupling of the upwind sweep
// (k_sweep_win): G_e = B_e^-1 L_e, where L_e is the block of the
// Jacobian coupling element e's rows to its left neighbour's outflow trace,
// nonzero in rows (r, node 0) only: L_e[(r, 0)][j] = S(r, j) l_{e,j},
// l_{e,j} = (2/h)(1/w_0) dH/du_L (u_{e-1,N}(t_j), u_{e,0}(t_j)) (the LLF
// flux of the left face, spatial.hpp:20-25 with f = u^2/2).  Stored fp32
// [e][row][j], NT floats per row.
template <int N1, int NT>
__global__ void __launch_bounds__(128) k_build_burgers_eblock(float* __restrict__ Binv,
                                                              float* __restrict__ G,
                                                              const double* __restrict__ U,
                                                              const SlabArgs a) {
  pdl_entry();
  constexpr int NB = N1 * NT;
  static_assert(NB <= 16 && NB % 2 == 0, "two elements per warp, even block size");
  constexpr int PS = NB + 4;  // published-row stride (doubles): halves on different banks
  __shared__ __align__(16) double pub[4][2][PS];
  const int lane = threadIdx.x & 31, h = lane >> 4, l = lane & 15, wib = threadIdx.x >> 5;
  const int K = a.g.nx;
  const int c = int(((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5) * 2 + h);
  const bool live = c < K;
  const int ce = live ? c : K - 1;  // dead half-warps mirror a live element (no stores)
  const long long ns = a.g.n_sdof;
  const int cl = ce == 0 ? K - 1 : ce - 1, cr = ce == K - 1 ? 0 : ce + 1;
  const bool act = l < NB;
  const int r = act ? l / N1 : 0, i = act ? l - (l / N1) * N1 : 0;
  double row[NB], lin[NT];
  // row i of D by selects (a dynamic index into the parameter struct, or
  // into u[], would go through local memory)
  double dmi[N1];
#pragma unroll
  for (int k = 0; k < N1; ++k) {
    double v = a.sp.Dm[0][k];
#pragma unroll
    for (int ii = 1; ii < N1; ++ii) v = i == ii ? a.sp.Dm[ii][k] : v;
    dmi[k] = v;
  }
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    double u[N1];
#pragma unroll
    for (int k = 0; k < N1; ++k) u[k] = U[j * ns + (long long)ce * N1 + k];
    double ui = u[0];
#pragma unroll
    for (int ii = 1; ii < N1; ++ii) ui = i == ii ? u[ii] : ui;
    const double ul = U[j * ns + (long long)cl * N1 + N1 - 1];
    const double ur = U[j * ns + (long long)cr * N1];
    {  // d/du_L of LLF(ul, u_0) at the left face: the inflow coupling l_{e,j}
      const double aL = fabs(ul), aR = fabs(u[0]);
      const double dH = aL >= aR ? 0.5 * ul + 0.5 * (ul >= 0 ? 1.0 : -1.0) * (ul - u[0]) + 0.5 * aL
                                 : 0.5 * ul + 0.5 * aR;
      lin[j] = a.sp.sc * a.sp.inv_w0 * dH;
    }
    // d F_i(U_j) / d u_q, own element, neighbour states fixed:
    //   -(2/h)/3 [ delta_iq sum_k D_ik (2 u_i + u_k) + D_iq (u_i + 2 u_q) ]
    // plus, at q = i, the own-trace derivative of the face flux
    double sdi = 0.0;
#pragma unroll
    for (int k = 0; k < N1; ++k) sdi = fma(dmi[k], 2.0 * ui + u[k], sdi);
    double face = 0.0;
    if (i == N1 - 1) {  // d/duL of LLF(uL, ur) - f(uL), right face
      const double aL = fabs(u[N1 - 1]), aR = fabs(ur);
      const double dH = aL >= aR ? 0.5 * u[N1 - 1] +
                                       0.5 * (u[N1 - 1] >= 0 ? 1.0 : -1.0) * (u[N1 - 1] - ur) +
                                       0.5 * aL
                                 : 0.5 * u[N1 - 1] + 0.5 * aR;
      face = -a.sp.sc * (dH - u[N1 - 1]) * a.sp.inv_wN;
    }
    if (i == 0) {  // d/duR of LLF(ul, uR) - f(uR), left face
      const double aL = fabs(ul), aR = fabs(u[0]);
      const double dH = aL >= aR ? 0.5 * u[0] - 0.5 * aL
                                 : 0.5 * u[0] + 0.5 * (u[0] >= 0 ? 1.0 : -1.0) * (ul - u[0]) -
                                       0.5 * aR;
      face += a.sp.sc * (dH - u[0]) * a.sp.inv_w0;
    }
    const double trj = a.mx.T[r][j], srj = a.mx.S[r][j], c3 = -a.sp.sc * (1.0 / 3.0);
#pragma unroll
    for (int q = 0; q < N1; ++q) {
      double g = c3 * ((i == q ? sdi : 0.0) + dmi[q] * (ui + 2.0 * u[q]));
      if (i == q) g += face;
      row[j * N1 + q] = act ? (i == q ? trj : 0.0) + srj * g : 0.0;
    }
  }
  // in-place Gauss-Jordan: row[] becomes the lane's row of (P B)^-1, P the
  // pivot order (no row exchanges: the pivot lane of column col ends up with
  // row col of B^-1, its entry at position c' belonging to column piv[c'])
  bool used = !act;
  int my_col = 0;
  int piv[NB];
  double* P = pub[wib][h];
#pragma unroll
  for (int col = 0; col < NB; ++col) {
    // pivot lane of this half: the largest |row[col]| among unused lanes by
    // the top 28 bits of the magnitude (ties in those bits -- a relative
    // difference below 2^-16 -- go to the lowest lane)
    // key: magnitude's top 28 bits above (15 - lane): unique per lane, the
    // lowest lane wins ties; a max over the half by four xor-shuffles
    unsigned key =
        used ? 0u
             : ((unsigned((unsigned long long)__double_as_longlong(fabs(row[col])) >> 32) & ~15u) |
                unsigned(15 - l));
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, o));
    const int idx = 15 - int(key & 15u);
    piv[col] = idx;
    if (l == idx) {
      // fp32 seed + two Newton steps: fp64-accurate, no division sequence
      const double pv = row[col];
      double ip = double(__frcp_rn(float(pv)));
      ip = ip * fma(-pv, ip, 2.0);
      ip = ip * fma(-pv, ip, 2.0);
#pragma unroll
      for (int q = 0; q < NB; ++q) row[q] = q == col ? ip : row[q] * ip;
#pragma unroll
      for (int q = 0; q < NB; q += 2)
        *reinterpret_cast<double2*>(P + q) = make_double2(row[q], row[q + 1]);
      used = true;
      my_col = col;
    }
    __syncwarp();
    if (l != idx) {
      const double f = row[col];
#pragma unroll
      for (int q = 0; q < NB; q += 2) {
        const double2 pr = *reinterpret_cast<const double2*>(P + q);
        row[q] = q == col ? -f * pr.x : fma(-f, pr.x, row[q]);
        row[q + 1] = q + 1 == col ? -f * pr.y : fma(-f, pr.y, row[q + 1]);
      }
    }
    __syncwarp();  // the published row is consumed before the next pivot writes
  }
  if (act && live) {  // stored in fp32: a preconditioner; GMRES itself stays fp64
    // the pivot lane of column c owns the identity column of row piv[c]
    float* M = Binv + (size_t)c * NB * NB + (size_t)my_col * NB;
#pragma unroll
    for (int q = 0; q < NB; ++q) M[piv[q]] = float(row[q]);
    if (G) {  // row my_col of B_e^-1 L_e (entries of B_e^-1 at columns (r, node 0))
      double b0[NT];
#pragma unroll
      for (int r2 = 0; r2 < NT; ++r2) {
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < NB; ++q) v = piv[q] == r2 * N1 ? row[q] : v;
        b0[r2] = v;
      }
      float* Gr = G + ((size_t)c * NB + my_col) * NT;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int r2 = 0; r2 < NT; ++r2) acc = fma(b0[r2], a.mx.S[r2][j], acc);
        Gr[j] = float(acc * lin[j]);
      }
    }
  }
}

// Per-element blocks (bstride > 0), nb <= 16: two elements per warp, lane
// (h, r) computes row r of element 2w + h; x is exchanged by shuffles and
// the block row is read with 16-byte loads.
template <int NB>
__global__ void __launch_bounds__(256) k_eblock2(double* __restrict__ out,
                                                 const double* __restrict__ in,
                                                 const float* __restrict__ B, int n1,
                                                 int ncells, long long ns, Skip skip) {
  pdl_entry();
  if (skip_now(skip)) return;
  static_assert(NB <= 16 && NB % 2 == 0, "two elements per warp");
  const int lane = threadIdx.x & 31, h = lane >> 4, r = lane & 15;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long pair = warp; pair * 2 < ncells; pair += nwarps) {
    const long long c = pair * 2 + h;
    const bool act = r < NB && c < ncells;
    const int t = r / n1, k = r - (r / n1) * n1;
    const double x = act ? in[t * ns + c * n1 + k] : 0.0;
    const float* Brow = B + (size_t)(act ? c : 0) * NB * NB + (size_t)(act ? r : 0) * NB;
    // the row as 16-byte loads where it is 16-byte aligned (NB % 4 == 0)
    float bv[NB];
    if (NB % 4 == 0) {
#pragma unroll
      for (int q4 = 0; q4 < NB / 4; ++q4) {
        const float4 v = act ? __ldg(reinterpret_cast<const float4*>(Brow) + q4)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
        bv[4 * q4] = v.x;
        bv[4 * q4 + 1] = v.y;
        bv[4 * q4 + 2] = v.z;
        bv[4 * q4 + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int q2 = 0; q2 < NB / 2; ++q2) {
        const float2 v = act ? __ldg(reinterpret_cast<const float2*>(Brow) + q2)
                             : make_float2(0.f, 0.f);
        bv[2 * q2] = v.x;
        bv[2 * q2 + 1] = v.y;
      }
    }
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < NB; ++q)
      acc = fma(double(bv[q]), __shfl_sync(0xffffffffu, x, (h << 4) + q), acc);
    if (act) out[t * ns + c * n1 + k] = acc;
  }
}

// ---- d = 1 upwind block sweep (block Gauss-Seidel in +x, periodic) --------
// P = blockdiag(B_e) + L: the element blocks plus the inflow coupling of each
// element to its left neighbour (the Jacobian without its downwind part, an
// O(jump) term for LLF with u > 0).  P z = r is the recurrence
//   z_e = y_e - G_e s_{e-1},  y_e = B_e^-1 r_e,  G_e = B_e^-1 L_e,
//   s_e = (z_e at node N, all temporal nodes) = a_e + C_e s_{e-1},
//   a_e = y_e at node N, C_e = -G_e rows at node N,
// around the periodic ring.  The influence of s_{e-m} on s_e is the product
// C_e ... C_{e-m+1}, which decays geometrically (c3, CFL ~1.5: |C_e| ~ 0.54,
// the product over 16 elements ~1e-11, over 32 ~1e-23; CFL 6: ~4e-6 over
// 32), so every element starts the recurrence from s = 0 kSwHalo elements
// upstream -- the sweep is exact up to that product, in one pass with no
// global scan:
//   k_eblock2   : y = B^-1 r (into a work vector);
//   k_sweep_win : per chunk of kSwCh elements, the chunk and its kSwHalo
//                 upstream elements' C_e and a_e staged in shared memory;
//                 each owned element runs the recurrence over its window;
//                 then z_e = y_e - G_e s_{e-1} (lane per block row).
// Where the flow runs in -x the inflow coupling vanishes (dH/du_L = 0 without
// jumps) and the sweep reduces to the element-block Jacobi there.
constexpr int kSwCh = 256;   // owned elements per CTA (= threads)
constexpr int kSwHalo = 16;  // upstream window

// vv != nullptr: also <z, z> into *vv (fixed-order block partials, the last
// block finishes), which the following FD Jacobian action needs for its step
template <int N1, int NT>
__global__ void __launch_bounds__(kSwCh) k_sweep_win(double* __restrict__ out,
                                                     const double* __restrict__ y,
                                                     const float* __restrict__ G, int ncells,
                                                     long long ns, Skip skip, double* part,
                                                     double* vv, unsigned* counter) {
  pdl_entry();
  if (skip_now(skip)) return;
  constexpr int NB = N1 * NT, NE = kSwCh + kSwHalo;
  static_assert(NT == 4, "one float4 per coupling row");
  // C_e and a_e of the window, converted to fp64 once (F2F.F64.F32 issues at
  // a fraction of the FP64 rate: converting inside the recurrence cost 3x)
  // element index fastest: the recurrence's lanes read consecutive doubles
  extern __shared__ double sw_smem[];
  double(*Cs)[NT][NE] = reinterpret_cast<double(*)[NT][NE]>(sw_smem);  // C_e [r][q][e]
  double(*As)[NE] = reinterpret_cast<double(*)[NE]>(sw_smem + NE * NT * NT);  // a_e [r][e]
  double(*Ss)[NT + 1] = reinterpret_cast<double(*)[NT + 1]>(sw_smem + NE * (NT * NT + NT));
  const int e0 = blockIdx.x * kSwCh;
  for (int j = threadIdx.x; j < NE; j += kSwCh) {
    int el = e0 - kSwHalo + j;
    el = el < 0 ? el + ncells * ((kSwHalo + ncells - 1) / ncells) : el;
    el = el % ncells;
    const float* Ge = G + (size_t)el * NB * NT;
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      const float4 c = __ldg(reinterpret_cast<const float4*>(Ge + (i * N1 + N1 - 1) * NT));
      Cs[i][0][j] = -double(c.x);
      Cs[i][1][j] = -double(c.y);
      Cs[i][2][j] = -double(c.z);
      Cs[i][3][j] = -double(c.w);
      As[i][j] = y[i * ns + (long long)el * N1 + N1 - 1];
    }
  }
  __syncthreads();
  {
    const int i = threadIdx.x;
    double st[NT] = {};
#pragma unroll 4
    for (int k = 0; k < kSwHalo; ++k) {
      const int j = i + k;
      double nx[NT];
#pragma unroll
      for (int r = 0; r < NT; ++r) {
        double v = As[r][j];
#pragma unroll
        for (int q = 0; q < NT; ++q) v = fma(Cs[r][q][j], st[q], v);
        nx[r] = v;
      }
#pragma unroll
      for (int r = 0; r < NT; ++r) st[r] = nx[r];
    }
#pragma unroll
    for (int r = 0; r < NT; ++r) Ss[i][r] = st[r];
  }
  __syncthreads();
  // z_e = y_e - G_e s_{e-1}: per temporal node t, thread q of the chunk's
  // kSwCh * N1 nodes (coalesced); all loads of a batch issued first
  constexpr int PER = NT * kSwCh * N1 / kSwCh, BATCH = PER / 2;
  double zz = 0.0;
#pragma unroll
  for (int b0 = 0; b0 < PER; b0 += BATCH) {
    float4 g[BATCH];
    double yv[BATCH];
#pragma unroll
    for (int b = 0; b < BATCH; ++b) {
      const int q = (b0 + b) * kSwCh + threadIdx.x;  // (t, element, node), node fastest
      const int t = q / (kSwCh * N1), rem = q - t * (kSwCh * N1);
      const int il = rem / N1, k = rem - il * N1;
      const long long c = (long long)e0 + il;
      const bool act = c < ncells;
      g[b] = act ? __ldg(reinterpret_cast<const float4*>(G + ((size_t)c * NB + t * N1 + k) * NT))
                 : make_float4(0.f, 0.f, 0.f, 0.f);
      yv[b] = act ? y[t * ns + c * N1 + k] : 0.0;
    }
#pragma unroll
    for (int b = 0; b < BATCH; ++b) {
      const int q = (b0 + b) * kSwCh + threadIdx.x;
      const int t = q / (kSwCh * N1), rem = q - t * (kSwCh * N1);
      const int il = rem / N1, k = rem - il * N1;
      const long long c = (long long)e0 + il;
      if (c < ncells) {
        double z = yv[b];
        z = fma(-double(g[b].x), Ss[il][0], z);
        z = fma(-double(g[b].y), Ss[il][1], z);
        z = fma(-double(g[b].z), Ss[il][2], z);
        z = fma(-double(g[b].w), Ss[il][3], z);
        out[t * ns + c * N1 + k] = z;
        zz = fma(z, z, zz);
      }
    }
  }
  if (vv) {
    __shared__ double red[kSwCh / 32];
    const double w = warp_sum(zz);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = w;
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = 0.0;
#pragma unroll
      for (int q = 0; q < kSwCh / 32; ++q) b += red[q];
      part[blockIdx.x] = b;
    }
    if (is_last_block(counter)) block_finish_sum(part, gridDim.x, 1, vv, counter);
  }
}

// ---- off-block-diagonal residual r - L y (polynomial preconditioner) ------
// L = J - blockdiag(J): the neighbour couplings of the constant-velocity
// advection Jacobian, S (x) (the cL / cR face terms of SpatialCoef), so
//   out[t][c][i] = r[t][c][i] - sum_j S(t, j) sum_a ( [i_a = 0] cL_a y_j[c - e_a][i_a <- N]
//                                                + [i_a = N] cR_a y_j[c + e_a][i_a <- 0] ).
// With the exact element-block inverse P0 (FDM), one Neumann step of the
// polynomial preconditioner is y <- P0^-1 (r - L y).  One thread per spatial
// node (all temporal nodes); interior nodes copy r.
template <int D, int N1, int NT>
__global__ void __launch_bounds__(256) k_offdiag(double* __restrict__ out,
                                                 const double* __restrict__ r,
                                                 const double* __restrict__ y,
                                                 const SpatialCoef sp, const MixCoef mx,
                                                 const Geometry g, Skip skip) {
  pdl_entry();
  if (skip_now(skip)) return;
  constexpr int NPC = D == 1 ? N1 : (D == 2 ? N1 * N1 : N1 * N1 * N1);
  const long long ns = g.n_sdof;
  for (long long sidx = blockIdx.x * (long long)blockDim.x + threadIdx.x; sidx < ns;
       sidx += (long long)gridDim.x * blockDim.x) {
    const int cell = int(sidx / NPC), node = int(sidx - (long long)cell * NPC);
    const int idx[3] = {node % N1, (node / N1) % N1, node / (N1 * N1)};
    const int ci[3] = {cell % g.nx, (cell / g.nx) % g.ny, cell / (g.nx * g.ny)};
    const int nc[3] = {g.nx, g.ny, g.nz};
    const int st[3] = {1, N1, N1 * N1};
    double nb[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) nb[j] = 0.0;
    bool any = false;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const int cstride = a == 0 ? 1 : (a == 1 ? g.nx : g.nx * g.ny);
      if (idx[a] == 0 && sp.cL[a] != 0.0) {
        const int cn = cell + (ci[a] == 0 ? (nc[a] - 1) : -1) * cstride;
        const long long o = (long long)cn * NPC + node + (N1 - 1) * st[a];
#pragma unroll
        for (int j = 0; j < NT; ++j) nb[j] = fma(sp.cL[a], y[j * ns + o], nb[j]);
        any = true;
      }
      if (idx[a] == N1 - 1 && sp.cR[a] != 0.0) {
        const int cn = cell + (ci[a] == nc[a] - 1 ? -(nc[a] - 1) : 1) * cstride;
        const long long o = (long long)cn * NPC + node - (N1 - 1) * st[a];
#pragma unroll
        for (int j = 0; j < NT; ++j) nb[j] = fma(sp.cR[a], y[j * ns + o], nb[j]);
        any = true;
      }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      double v = r[t * ns + sidx];
      if (any) {
#pragma unroll
        for (int j = 0; j < NT; ++j) v = fma(-mx.S[t][j], nb[j], v);
      }
      out[t * ns + sidx] = v;
    }
  }
}

int pgrid(long long n) {
  long long g = (n + kPB - 1) / kPB;
  if (g > 148 * 8) g = 148 * 8;
  return int(g < 1 ? 1 : g);
}

}  // namespace

void precond_tblock(double* out, const double* in, const double* minv, int nt, int npc,
                    long long ns, cudaStream_t s, Skip skip) {
  const int ncells = int(ns / npc);  // ns < 2^31 for every supported mesh (validate_desc)
  const size_t smem = size_t(npc) * nt * nt * sizeof(double);
  const int g = pgrid(ns);
  switch (nt) {
    case 2: launch_ex(kPdlPrecond, k_tblock<2>, g, kPB, smem, s, out, in, minv, npc, ncells, ns, skip); break;
    case 3: launch_ex(kPdlPrecond, k_tblock<3>, g, kPB, smem, s, out, in, minv, npc, ncells, ns, skip); break;
    case 4: launch_ex(kPdlPrecond, k_tblock<4>, g, kPB, smem, s, out, in, minv, npc, ncells, ns, skip); break;
    case 5: launch_ex(kPdlPrecond, k_tblock<5>, g, kPB, smem, s, out, in, minv, npc, ncells, ns, skip); break;
    default: launch_ex(kPdlPrecond, k_tblock<6>, g, kPB, smem, s, out, in, minv, npc, ncells, ns, skip); break;
  }
}

void precond_eblock(double* out, const double* in, const double* B, long long bstride, int nt,
                    int n1, int ncells, long long ns, cudaStream_t s, Skip skip) {
  int g = (ncells + 7) / 8;
  if (g > 148 * 16) g = 148 * 16;
  launch_ex(kPdlPrecond, k_eblock<kMaxT * kMaxN>, g, 256, 0, s, out, in, B, bstride, nt, n1, ncells, ns, skip);
}

// ---- d = 2 element-block Jacobi with one shared dense block ----------------
// Y = B X for every element, B (nb x nb, nb = n_tau * n^2 <= kDenseMax) the
// inverse of the element-local Jacobian block.  It is a GEMM
// (nb x nb) x (nb x n_cells) on the stage-major layout: a CTA stages B^T in
// shared memory once, then loops over tiles of TE = 32 elements -- gather the
// tile transposed into shared memory, a 4 x 4 register tile per thread
// (rows x elements), the result staged back through shared memory and
// written coalesced.  FP64-pipe bound (nb FMAs per DOF).
constexpr int kDenseMax = 128;
constexpr int kTE = 64;            // elements per tile
constexpr int kTEp = kTE + 1;      // odd row pitch: conflict-free transposed staging
constexpr int kDenseThreads = 32 * (kTE / 4);  // 32 row groups x 16 element groups
constexpr int kPre = 128 * kTE / kDenseThreads;  // prefetched doubles per thread

__global__ void __launch_bounds__(kDenseThreads, 1)
    k_eblock_dense(double* __restrict__ out, const double* __restrict__ in,
                   const double* __restrict__ B, int nb, int npc, int nt, int ncells,
                   long long ns, Skip skip) {
  pdl_entry();
  if (skip_now(skip)) return;
  extern __shared__ double sm[];
  constexpr int NBP = 128;                  // padded row count of B^T (4 rows x 32 groups)
  double* Bt = sm;                          // [nb][NBP]: Bt[k][row] = B[row][k]
  double* Xs = Bt + (size_t)nb * NBP;       // [NBP][kTEp]: input tile, then output tile
  const int tid = threadIdx.x;
  for (int q = tid; q < nb * NBP; q += kDenseThreads) {
    const int k = q / NBP, row = q - (q / NBP) * NBP;
    Bt[q] = row < nb ? B[(size_t)row * nb + k] : 0.0;
  }
  const int rg = tid & 31, eg = tid >> 5;  // rows 4rg..4rg+3, elements 4eg..4eg+3
  const int ntile = (ncells + kTE - 1) / kTE;
  const int per_tile = nt * kTE * npc;  // <= 128 * kTE = kPre * kDenseThreads
  // the next tile is gathered into registers while the current one is
  // computed (loads first, then the transposed shared stores)
  double pre[kPre];
  auto load_tile = [&](int tile) {
    const int e0 = tile * kTE, ne = min(kTE, ncells - e0);
#pragma unroll
    for (int c = 0; c < kPre; ++c) {
      const int q = tid + c * kDenseThreads;
      pre[c] = 0.0;
      if (q < per_tile) {
        const int t = q / (kTE * npc), r = q - t * (kTE * npc);
        if (r / npc < ne) pre[c] = __ldcs(in + t * ns + (long long)e0 * npc + r);
      }
    }
  };
  if (blockIdx.x < ntile) load_tile(blockIdx.x);
  for (int tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    const int e0 = tile * kTE;
    const int ne = min(kTE, ncells - e0);
    __syncthreads();  // Bt ready / previous tile's output drained
#pragma unroll
    for (int c = 0; c < kPre; ++c) {
      const int q = tid + c * kDenseThreads;
      if (q < per_tile) {
        const int t = q / (kTE * npc), r = q - t * (kTE * npc);
        const int e = r / npc, node = r - (r / npc) * npc;
        Xs[(t * npc + node) * kTEp + e] = pre[c];
      }
    }
    __syncthreads();
    if (tile + (int)gridDim.x < ntile) load_tile(tile + gridDim.x);
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    const double* bcol = Bt + 4 * rg;
    const double* xrow = Xs + 4 * eg;
#pragma unroll 5
    for (int k = 0; k < nb; ++k) {
      const double2 b01 = *reinterpret_cast<const double2*>(bcol + (size_t)k * NBP);
      const double2 b23 = *reinterpret_cast<const double2*>(bcol + (size_t)k * NBP + 2);
      const double x0 = xrow[k * kTEp + 0], x1 = xrow[k * kTEp + 1],
                   x2 = xrow[k * kTEp + 2], x3 = xrow[k * kTEp + 3];
      const double bb[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[i][0] = fma(bb[i], x0, acc[i][0]);
        acc[i][1] = fma(bb[i], x1, acc[i][1]);
        acc[i][2] = fma(bb[i], x2, acc[i][2]);
        acc[i][3] = fma(bb[i], x3, acc[i][3]);
      }
    }
    __syncthreads();  // every thread has read the input tile
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = 4 * rg + i;
      if (row < nb) {
#pragma unroll
        for (int j = 0; j < 4; ++j) Xs[row * kTEp + 4 * eg + j] = acc[i][j];
      }
    }
    __syncthreads();
    for (int t = 0; t < nt; ++t) {  // coalesced write-back
      double* dst = out + t * ns + (long long)e0 * npc;
      for (int q = tid; q < ne * npc; q += kDenseThreads) {
        const int e = q / npc, node = q - (q / npc) * npc;
        dst[q] = Xs[(t * npc + node) * kTEp + e];
      }
    }
  }
}

// ---- element blocks of the general (linear) models by coloured probing -----
// P = unit entry `col` in every cell of colour (cx0, cy0); after F = F(P) the
// cells of that colour read column `col` of their local Jacobian K_e off
// their own rows (same-colour cells are >= 3 apart: neighbour couplings never
// reach them).  Then B_e = T (x) I + S (x) K_e is inverted per element.
__global__ void k_probe_set(double* __restrict__ P, int ndl, int col, int nx, int ny, int sx,
                            int sy, int cx0, int cy0, int ncells) {
  pdl_entry();
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncells; c += gridDim.x * blockDim.x) {
    const int cx = c % nx, cy = c / nx;
    const bool on = (cx % sx) == cx0 && (cy % sy) == cy0;
    for (int k = 0; k < ndl; ++k) P[(long long)c * ndl + k] = (on && k == col) ? 1.0 : 0.0;
  }
}
__global__ void k_probe_extract(double* __restrict__ K, const double* __restrict__ F, int ndl,
                                int col, int nx, int sx, int sy, int cx0, int cy0, int ncells) {
  pdl_entry();
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncells; c += gridDim.x * blockDim.x) {
    const int cx = c % nx, cy = c / nx;
    if ((cx % sx) != cx0 || (cy % sy) != cy0) continue;
    for (int i = 0; i < ndl; ++i)
      K[((long long)c * ndl + i) * ndl + col] = F[(long long)c * ndl + i];
  }
}

// one warp per element: lane l < nb owns row l = (t, i) of [B_e | I];
// Gauss-Jordan with partial pivoting without row exchanges (see
// k_build_burgers_eblock); B_e = T(t,j) delta_ik + S(t,j) K_e(i,k)
__global__ void __launch_bounds__(128) k_gen_eblock(double* __restrict__ Binv,
                                                    const double* __restrict__ K,
                                                    const MixCoef mx, int nt, int ndl,
                                                    int ncells) {
  pdl_entry();
  constexpr int MAXB = 32;
  const int lane = threadIdx.x & 31;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= ncells) return;  // warp-uniform
  const int nb = nt * ndl;
  const bool act = lane < nb;
  const int t = act ? lane / ndl : 0, i = act ? lane - (lane / ndl) * ndl : 0;
  const double* Kc = K + (size_t)c * ndl * ndl;
  double row[MAXB], inv[MAXB];
#pragma unroll
  for (int q = 0; q < MAXB; ++q) {
    double v = 0.0;
    if (act && q < nb) {
      const int j = q / ndl, k = q - (q / ndl) * ndl;
      v = (i == k ? mx.T[t][j] : 0.0) + mx.S[t][j] * Kc[i * ndl + k];
    }
    row[q] = v;
    inv[q] = (q == lane && act) ? 1.0 : 0.0;
  }
  bool used = !act;
  int my_col = 0;
#pragma unroll
  for (int col = 0; col < MAXB; ++col) {
    if (col >= nb) break;  // uniform
    double v = used ? -1.0 : fabs(row[col]);
    int idx = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
      if (v2 > v || (v2 == v && i2 < idx)) {
        v = v2;
        idx = i2;
      }
    }
    const int p = idx;
    const double ip = 1.0 / __shfl_sync(0xffffffffu, row[col], p);
    if (lane == p) {
#pragma unroll
      for (int q = 0; q < MAXB; ++q) {
        row[q] *= ip;
        inv[q] *= ip;
      }
      used = true;
      my_col = col;
    }
    const double f = row[col];
#pragma unroll
    for (int q = 0; q < MAXB; ++q) {
      const double pr = __shfl_sync(0xffffffffu, row[q], p);
      const double pi = __shfl_sync(0xffffffffu, inv[q], p);
      if (lane != p) {
        row[q] = fma(-f, pr, row[q]);
        inv[q] = fma(-f, pi, inv[q]);
      }
    }
  }
  if (act) {
    double* M = Binv + (size_t)c * nb * nb + (size_t)my_col * nb;
#pragma unroll
    for (int q = 0; q < MAXB; ++q)
      if (q < nb) M[q] = inv[q];
  }
}

template <int N1>
bool build_nt(float* Binv, float* G, const double* U, const SlabArgs& a, cudaStream_t s) {
  const long long warps = ((long long)a.g.nx + 1) / 2;  // two elements per warp
  const int blocks = int((warps * 32 + 127) / 128);
  auto go = [&](auto nt_tag) {
    constexpr int NT = decltype(nt_tag)::value;
    if constexpr (N1 * NT <= 16 && (N1 * NT) % 2 == 0) {
      launch_ex(kPdlPrecond, k_build_burgers_eblock<N1, NT>, blocks, 128, 0, s, Binv, G, U, a);
      return true;
    } else {
      return false;  // the fp32 block apply takes n_tau * (N+1) <= 16, even
    }
  };
  switch (a.n_in) {
    case 2: return go(std::integral_constant<int, 2>{});
    case 3: return go(std::integral_constant<int, 3>{});
    case 4: return go(std::integral_constant<int, 4>{});
    case 5: return go(std::integral_constant<int, 5>{});
    case 6: return go(std::integral_constant<int, 6>{});
    default: return false;
  }
}


bool precond_eblock_dense(double* out, const double* in, const double* B, int nt, int npc,
                          int ncells, long long ns, cudaStream_t s, Skip skip) {
  const int nb = nt * npc;
  if (nb > kDenseMax) return false;
  const size_t smem = sizeof(double) * ((size_t)nb * 128 + (size_t)128 * kTEp);
  if (smem > 227 * 1024) return false;
  static size_t set_dev[kMaxDevices];
  size_t& set = set_dev[device_slot()];
  if (smem > set) {
    cudaFuncSetAttribute(k_eblock_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    set = smem;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ntile = (ncells + kTE - 1) / kTE;
  const int grid = ntile < sms ? ntile : sms;
  launch_ex(kPdlPrecond, k_eblock_dense, grid, kDenseThreads, smem, s, out, in, B, nb, npc, nt,
            ncells, ns, skip);
  return true;
}

void probe_set(double* P, int ndl, int col, int nx, int ny, int sx, int sy, int cx0, int cy0,
               int ncells, cudaStream_t s) {
  launch_ex(kPdlPrecond, k_probe_set, pgrid(ncells), kPB, 0, s, P, ndl, col, nx, ny, sx, sy, cx0, cy0, ncells);
}
void probe_extract(double* K, const double* F, int ndl, int col, int nx, int sx, int sy, int cx0,
                   int cy0, int ncells, cudaStream_t s) {
  launch_ex(kPdlPrecond, k_probe_extract, pgrid(ncells), kPB, 0, s, K, F, ndl, col, nx, sx, sy, cx0, cy0, ncells);
}
bool gen_eblock_invert(double* Binv, const double* K, const MixCoef& mx, int nt, int ndl,
                       int ncells, cudaStream_t s) {
  if (nt * ndl > 32) return false;
  const long long threads = (long long)ncells * 32;
  launch_ex(kPdlPrecond, k_gen_eblock, int((threads + 127) / 128), 128, 0, s, Binv, K, mx, nt, ndl, ncells);
  return true;
}

void precond_eblock_f32(double* out, const double* in, const float* B, int nt, int n1,
                        int ncells, long long ns, cudaStream_t s, Skip skip) {
  const int nb = nt * n1;
  long long g = ((ncells + 1) / 2 + 7) / 8;  // 8 warps per block, 2 elements per warp
  if (g > 148 * 16) g = 148 * 16;
  switch (nb) {
    case 4: launch_ex(kPdlPrecond, k_eblock2<4>, int(g), 256, 0, s, out, in, B, n1, ncells, ns, skip); return;
    case 6: launch_ex(kPdlPrecond, k_eblock2<6>, int(g), 256, 0, s, out, in, B, n1, ncells, ns, skip); return;
    case 8: launch_ex(kPdlPrecond, k_eblock2<8>, int(g), 256, 0, s, out, in, B, n1, ncells, ns, skip); return;
    case 10: launch_ex(kPdlPrecond, k_eblock2<10>, int(g), 256, 0, s, out, in, B, n1, ncells, ns, skip); return;
    case 12: launch_ex(kPdlPrecond, k_eblock2<12>, int(g), 256, 0, s, out, in, B, n1, ncells, ns, skip); return;
    case 14: launch_ex(kPdlPrecond, k_eblock2<14>, int(g), 256, 0, s, out, in, B, n1, ncells, ns, skip); return;
    case 16: launch_ex(kPdlPrecond, k_eblock2<16>, int(g), 256, 0, s, out, in, B, n1, ncells, ns, skip); return;
    default: break;
  }
}

bool sweep_supported(int nt, int n1) {
  return nt == 4 && (n1 == 2 || n1 == 4);
}

size_t sweep_work_doubles(int nt, int ncells, int n1) { return size_t(ncells) * n1 * nt; }

void precond_sweep(double* out, const double* in, const float* B, const float* G, double* work,
                   int nt, int n1, int ncells, long long ns, cudaStream_t s, Skip skip,
                   double* partial, double* vv) {
  long long g = ((ncells + 1) / 2 + 7) / 8;
  if (g > 148 * 16) g = 148 * 16;
  const int nch = (ncells + kSwCh - 1) / kSwCh;
  auto go = [&](auto n1_tag) {
    constexpr int N1 = decltype(n1_tag)::value;
    launch_ex(kPdlPrecond, k_eblock2<N1 * 4>, int(g), 256, 0, s, work, in, B, n1, ncells, ns, skip);
    constexpr size_t smem = sizeof(double) * ((kSwCh + kSwHalo) * (16 + 4) + kSwCh * 5);
    static bool set_dev[kMaxDevices];
    bool& set = set_dev[device_slot()];
    if (!set) {
      cudaFuncSetAttribute(k_sweep_win<N1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      set = true;
    }
    launch_ex(kPdlPrecond, k_sweep_win<N1, 4>, nch, kSwCh, smem, s, out, work, G, ncells, ns, skip,
              partial, vv, partial ? counter_of(partial) : nullptr);
  };
  if (nt != 4) return;
  if (n1 == 4) go(std::integral_constant<int, 4>{});
  else if (n1 == 2) go(std::integral_constant<int, 2>{});
}

bool offdiag_supported(const Geometry& g, int nt) {
  return (g.dim == 3 && ((g.n1 == 4 && nt == 4) || (g.n1 == 3 && nt == 3))) ||
         (g.dim == 2 && ((g.n1 == 5 && nt == 5) || (g.n1 == 4 && nt == 4) ||
                         (g.n1 == 3 && nt == 3))) ||
         (g.dim == 1 && g.n1 == 4 && nt == 4);
}

bool offdiag_residual(double* out, const double* r, const double* y, const SpatialCoef& sp,
                      const MixCoef& mx, const Geometry& g, int nt, cudaStream_t s, Skip skip) {
  const long long ns = g.n_sdof;
  long long blocks = (ns + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  const int gb = int(blocks);
  if (g.dim == 3 && g.n1 == 4 && nt == 4)
    launch_ex(kPdlPrecond, k_offdiag<3, 4, 4>, gb, 256, 0, s, out, r, y, sp, mx, g, skip);
  else if (g.dim == 3 && g.n1 == 3 && nt == 3)
    launch_ex(kPdlPrecond, k_offdiag<3, 3, 3>, gb, 256, 0, s, out, r, y, sp, mx, g, skip);
  else if (g.dim == 2 && g.n1 == 5 && nt == 5)
    launch_ex(kPdlPrecond, k_offdiag<2, 5, 5>, gb, 256, 0, s, out, r, y, sp, mx, g, skip);
  else if (g.dim == 2 && g.n1 == 4 && nt == 4)
    launch_ex(kPdlPrecond, k_offdiag<2, 4, 4>, gb, 256, 0, s, out, r, y, sp, mx, g, skip);
  else if (g.dim == 2 && g.n1 == 3 && nt == 3)
    launch_ex(kPdlPrecond, k_offdiag<2, 3, 3>, gb, 256, 0, s, out, r, y, sp, mx, g, skip);
  else if (g.dim == 1 && g.n1 == 4 && nt == 4)
    launch_ex(kPdlPrecond, k_offdiag<1, 4, 4>, gb, 256, 0, s, out, r, y, sp, mx, g, skip);
  else
    return false;
  return true;
}

bool eblock_f32_supported(int nt, int n1) {
  const int nb = nt * n1;
  return nb <= 16 && nb % 2 == 0;
}

bool build_burgers_eblock(float* Binv, float* G, const double* U, const SlabArgs& a,
                          cudaStream_t s) {
  switch (a.g.n1) {
    case 2: return build_nt<2>(Binv, G, U, a, s);
    case 3: return build_nt<3>(Binv, G, U, a, s);
    case 4: return build_nt<4>(Binv, G, U, a, s);
    default: return false;
  }
}

}  // namespace stg
