// Element-block Jacobi for the d = 3, N = 3, n_tau = 4 slab / stage
// Jacobians by fast diagonalisation (FDM).
//
// The element-local block of J = T (x) I + S (x) F (advection; F's
// neighbour couplings removed) is L_e = (S (x) I)(G (x) I + I (x) K) with
// G = S^-1 T and K = V_z (+) V_y (+) V_x (Kronecker sum of the per-axis 4x4
// element matrices, own-face terms included).  With G = Q Lt Q^-1 and
// V_a = P_a Th_a P_a^-1 (complex, host eig.hpp):
//   L_e^-1 = (Q (x) Pz (x) Py (x) Px) diag(1/(lt + thz + thy + thx))
//            (Q^-1 S^-1 (x) Pz^-1 (x) Py^-1 (x) Px^-1).
// The input is real, so the spectrum is conjugate-symmetric and only the
// x-eigen-indices {0, 2} (one of each conjugate pair) are kept: the data stays
// 256 doubles per cell and the last inverse mode is 2 Re(.).  Cost ~15k FMA
// per cell (a dense 256 x 256 inverse would be 65k) in three phases:
//   A : forward x and y modes on the (y,x) plane at (t, cell, z)
//   B : forward z, t modes, the 1/Lambda scaling, inverse t, z modes on the
//       (t,z) tile at (iy, j), split over two threads (columns, then rows)
//   A': inverse y and x modes, coalesced store
// The input tile arrives by TMA (the operator's 128B-swizzled 4-D box) in a
// 2-stage ring; coefficient matrices are kernel parameters read as
// constant-bank operands.  Exactness is tested against the dense inverse.
#include <cuda.h>

#include <cstdlib>

#include "kernels.hpp"
#include "ptx.cuh"

namespace stg {
namespace {

constexpr int E = 8;
constexpr int THREADS = 128;
constexpr int TILE = 16384;
constexpr int OFF_B1 = 2 * TILE;
constexpr int OFF_LI = 3 * TILE;
constexpr int OFF_BAR = OFF_LI + 2048;
constexpr int SMEM = OFF_BAR + 64 + 1024;

__device__ __forceinline__ int row_of(int t, int e, int z) { return (t * E + e) * 4 + z; }

// complex helpers on (re, im) pairs
struct C2 {
  double r, i;
};
__device__ __forceinline__ void cmac(C2& acc, double ar, double ai, const C2& b) {
  acc.r = fma(ar, b.r, fma(-ai, b.i, acc.r));
  acc.i = fma(ar, b.i, fma(ai, b.r, acc.i));
}

__device__ __forceinline__ double2* tile_at(double* B1, int t, int e, int z, int q) {
  const int row = row_of(t, e, z);
  return reinterpret_cast<double2*>(B1 + row * 16 + ((q ^ (row & 7)) << 1));
}

// Phase B, first part, for half H of the (t,z) tile of unit (e, q = (iy, j)):
// forward z for the z-eigen-columns iz = 2H, 2H+1, then the t modes
// (Q^-1 S^-1, 1/Lambda, Q) on those columns.  Templated so the coefficient
// indices stay compile-time constants (H is warp-uniform).
template <int H>
__device__ __forceinline__ void phase_b_cols(const FdmCoef& c, double* B1, const double* LI,
                                             int e, int q, C2 (&w)[4][2]) {
  const int iy = q >> 1, j = q & 1;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    C2 u[4];
#pragma unroll
    for (int z = 0; z < 4; ++z) {
      const double2 v = *tile_at(B1, t, e, z, q);
      u[z] = {v.x, v.y};
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      C2 s = {0.0, 0.0};
#pragma unroll
      for (int z = 0; z < 4; ++z) cmac(s, c.FZ[2 * H + k][z][0], c.FZ[2 * H + k][z][1], u[z]);
      w[t][k] = s;
    }
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int iz = 2 * H + k;
    C2 s[4];
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      C2 a = {0.0, 0.0};
#pragma unroll
      for (int t = 0; t < 4; ++t) cmac(a, c.FT[it][t][0], c.FT[it][t][1], w[t][k]);
      const double2 l =
          *reinterpret_cast<const double2*>(LI + ((((it * 4 + iz) * 4 + iy) * 2 + j) << 1));
      s[it] = {a.r * l.x - a.i * l.y, a.r * l.y + a.i * l.x};
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      C2 a = {0.0, 0.0};
#pragma unroll
      for (int it = 0; it < 4; ++it) cmac(a, c.IT[t][it][0], c.IT[t][it][1], s[it]);
      w[t][k] = a;
    }
  }
}

// ---- the three phases, shared by the standalone apply and the fused
// Arnoldi-update kernel.  Thread tid owns tile row rowA = tid = (t, e, z) in
// phases A / A' and the half hB of tile unit (eB, qB) in phase B.
// Phase A: forward x (kept eigen-indices j -> kx = 2j) and y modes of the
// thread's (y,x) plane r, into the complex tile B1.
__device__ __forceinline__ void fdm_phase_a(const FdmCoef& c, const double (&r)[16], double* B1,
                                            int rowA, int swA) {
  C2 a[4][2];
#pragma unroll
  for (int y = 0; y < 4; ++y)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        re = fma(c.FX[j][x][0], r[4 * y + x], re);
        im = fma(c.FX[j][x][1], r[4 * y + x], im);
      }
      a[y][j] = {re, im};
    }
#pragma unroll
  for (int iy = 0; iy < 4; ++iy)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      C2 b = {0.0, 0.0};
#pragma unroll
      for (int y = 0; y < 4; ++y) cmac(b, c.FY[iy][y][0], c.FY[iy][y][1], a[y][j]);
      const int q = iy * 2 + j;
      *reinterpret_cast<double2*>(B1 + rowA * 16 + ((q ^ swA) << 1)) = make_double2(b.r, b.i);
    }
}

// Phase B: (t,z) tile at (iy, j), two threads per tile: forward z and t
// modes, 1/Lambda, inverse t and z modes, in place in B1.  Contains CTA
// barriers: every thread calls it.
__device__ __forceinline__ void fdm_phase_b(const FdmCoef& c, double* B1, const double* LI,
                                            int hB, int eB, int qB) {
  C2 w[4][2];  // [t][k]: z-eigen-column 2 hB + k
  if (hB)
    phase_b_cols<1>(c, B1, LI, eB, qB, w);
  else
    phase_b_cols<0>(c, B1, LI, eB, qB, w);
  __syncthreads();  // both halves have read the tile
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int k = 0; k < 2; ++k)
      *tile_at(B1, t, eB, 2 * hB + k, qB) = make_double2(w[t][k].r, w[t][k].i);
  __syncthreads();
  // inverse z on rows t = 2 hB, 2 hB + 1 (all four columns)
  C2 o[2][4];
#pragma unroll
  for (int tt = 0; tt < 2; ++tt) {
    C2 m[4];
#pragma unroll
    for (int iz = 0; iz < 4; ++iz) {
      const double2 v = *tile_at(B1, 2 * hB + tt, eB, iz, qB);
      m[iz] = {v.x, v.y};
    }
#pragma unroll
    for (int z = 0; z < 4; ++z) {
      C2 s = {0.0, 0.0};
#pragma unroll
      for (int iz = 0; iz < 4; ++iz) cmac(s, c.IZ[z][iz][0], c.IZ[z][iz][1], m[iz]);
      o[tt][z] = s;
    }
  }
  __syncthreads();  // every column read before the results overwrite them
#pragma unroll
  for (int tt = 0; tt < 2; ++tt)
#pragma unroll
    for (int z = 0; z < 4; ++z)
      *tile_at(B1, 2 * hB + tt, eB, z, qB) = make_double2(o[tt][z].r, o[tt][z].i);
}

// Phase A': inverse y and x modes (2 Re) of the thread's row into o.
__device__ __forceinline__ void fdm_phase_a2(const FdmCoef& c, const double* B1, int rowA,
                                             int swA, double (&o)[16]) {
  C2 h[4][2];
#pragma unroll
  for (int iy = 0; iy < 4; ++iy)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int q = iy * 2 + j;
      const double2 v = *reinterpret_cast<const double2*>(B1 + rowA * 16 + ((q ^ swA) << 1));
      h[iy][j] = {v.x, v.y};
    }
#pragma unroll
  for (int y = 0; y < 4; ++y) {
    C2 m[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      C2 s = {0.0, 0.0};
#pragma unroll
      for (int iy = 0; iy < 4; ++iy) cmac(s, c.IY[y][iy][0], c.IY[y][iy][1], h[iy][j]);
      m[j] = s;
    }
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      double re = 0.0;
#pragma unroll
      for (int j = 0; j < 2; ++j)
        re = fma(c.IX[x][j][0], m[j].r, fma(-c.IX[x][j][1], m[j].i, re));
      o[4 * y + x] = 2.0 * re;
    }
  }
}

template <int MINB>
__global__ void __launch_bounds__(THREADS, MINB)
    fdm_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm_out,
               const __grid_constant__ FdmCoef c, const Geometry g, const Skip skip) {
  pdl_entry();
  if (skip_now(skip)) return;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (ptxh::smem_u32(smem_raw) & 1023u)) & 1023u);
  double* B1 = reinterpret_cast<double*>(base + OFF_B1);
  double* LI = reinterpret_cast<double*>(base + OFF_LI);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + OFF_BAR);
  const uint32_t bar0 = ptxh::smem_u32(bars), bar1 = ptxh::smem_u32(bars + 1);
  const int tid = threadIdx.x;
  const int nseg = g.n_cells / E;

  for (int q = tid; q < 4 * 4 * 4 * 2 * 2; q += THREADS)
    LI[q] = (&c.LI[0][0][0][0][0])[q];
  if (tid == 0) {
    ptxh::mbar_init(bar0, 1);
    ptxh::mbar_init(bar1, 1);
    ptxh::fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int seg, int st) {
    const uint32_t bar = st ? bar1 : bar0;
    ptxh::mbar_expect_tx(bar, TILE);
    ptxh::tma_load_4d(ptxh::smem_u32(base + st * TILE), &tm, bar, 0, 0, seg * E, 0);
  };
  int seg = blockIdx.x;
  if (tid == 0 && seg < nseg) issue(seg, 0);

  const int zA = tid & 3, eA = (tid >> 2) & (E - 1), tA = tid >> 5;
  const int rowA = row_of(tA, eA, zA), swA = rowA & 7;
  // phase B: tile unit = (cell, iy, j); the two halves of a unit sit in
  // different warps so the half index is warp-uniform
  const int hB = (tid >> 5) & 1, uB = (tid & 31) | ((tid >> 6) << 5);
  const int eB = uB >> 3, qB = uB & 7;

  for (int it = 0; seg < nseg; ++it, seg += gridDim.x) {
    const int st = it & 1;
    double* Xs = reinterpret_cast<double*>(base + st * TILE);
    if (tid == 0 && seg + (int)gridDim.x < nseg) {
      // stage st^1 last held the previous segment's result: its bulk store
      // must have read it before the next load overwrites it
      ptxh::bulk_wait_read0();
      ptxh::fence_proxy_async_smem();
      issue(seg + gridDim.x, st ^ 1);
    }
    while (!ptxh::mbar_try_wait(st ? bar1 : bar0, (it >> 1) & 1)) {
    }
    {
      double r[16];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double2 v = *reinterpret_cast<const double2*>(Xs + rowA * 16 + ((q ^ swA) << 1));
        r[2 * q] = v.x;
        r[2 * q + 1] = v.y;
      }
      fdm_phase_a(c, r, B1, rowA, swA);
    }
    __syncthreads();
    fdm_phase_b(c, B1, LI, hB, eB, qB);
    __syncthreads();
    {
      // the result row goes back into the (consumed) input stage, in the
      // same swizzled box layout, and leaves by one TMA tensor store: full
      // 128-byte lines instead of 16-byte stores 128 bytes apart (which made
      // the L2 fetch every output sector from DRAM before merging)
      double o[16];
      fdm_phase_a2(c, B1, rowA, swA, o);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<double2*>(Xs + rowA * 16 + ((q ^ swA) << 1)) =
            make_double2(o[2 * q], o[2 * q + 1]);
    }
    ptxh::fence_proxy_async_smem();
    __syncthreads();  // result tile complete; B1 free for reuse
    if (tid == 0) {
      ptxh::tma_store_4d(&tm_out, ptxh::smem_u32(Xs), 0, 0, seg * E, 0);
      ptxh::bulk_commit();
    }
  }
  if (tid == 0) ptxh::bulk_wait0();
}

// ---------------------------------------------------------------------------
// fdm3_kernel: the same element-block inverse with the temporal direction
// solved directly per spatial mode, M_theta = (T + theta S)^-1 (4 x 4
// complex), instead of Q^-1 S^-1, 1/Lambda and Q, and the y / z transforms
// by conjugate pairs: 9.2k FP64 ops per cell (12.3k with plain complex y / z
// transforms, 15k with the eigen-decomposed t direction).  E cells per segment (8, below) and one thread per (cell, iy, j) unit in
// phase B, so every phase is one pass over the tile: three CTA barriers per
// segment (the two-half phase B above needs six per 8 cells).  The complex tile
// lives in place of the real one (a (t, z) row of 16 reals becomes 8 complex
// (iy, j) values).  All factors (FdmCoef3, 9.5 KB) arrive with the first tile
// by one bulk copy and are read from shared memory: warp-uniform addresses
// (broadcast) for the spatial factors, one 128-byte wavefront per table read
// (q fastest) -- kernel-parameter operands had the compiler keep ~100 of them
// in uniform registers and spill those.
// cells per segment: 8 (64-thread CTAs, 4 per SM) measured best for the
// coupled apply that dominates the c4 / c5 solves (c4 slab solve 0.678 ->
// 0.652 ms against 16 cells x 3 CTAs/SM; the plain apply 31.9 -> 30.2 us):
// half the first-tile wait and last-tile drain per CTA, 8 warps per SM at up
// to 254 registers without spills.  4 cells (one-warp CTAs, 8 per SM) gives
// the plain apply 29.1 us but the coupled one less.
#ifndef STG_FDM3_E
#define STG_FDM3_E 8
#endif
namespace f3 {
constexpr int E = STG_FDM3_E;      // cells per segment
constexpr int THREADS = 8 * E;     // two tile rows per thread, one phase-B unit per thread
constexpr int TILE = E * 256 * 8;  // 32 KB at E = 16: [t][cell][z] rows of 16 doubles
constexpr int COEF = int(sizeof(FdmCoef3));
constexpr int OFF_C = 2 * TILE;
constexpr int OFF_BAR = OFF_C + COEF;
constexpr int SMEM = OFF_BAR + 64 + 1024;  // + 1024 B alignment slack
__device__ __forceinline__ int row_of(int t, int e, int z) { return (t * E + e) * 4 + z; }
__device__ __forceinline__ double2* at(double* X, int row, int q) {
  return reinterpret_cast<double2*>(X + row * 16 + ((q ^ (row & 7)) << 1));
}
__device__ __forceinline__ C2 ld(const double (&a)[2]) {
  const double2 v = *reinterpret_cast<const double2*>(a);
  return {v.x, v.y};
}
// a spatial factor: a kernel-parameter (constant bank) operand or a shared load
template <bool PARAM>
__device__ __forceinline__ C2 cf(const double (&a)[2]) {
  if constexpr (PARAM) return {a[0], a[1]};
  return ld(a);
}
__device__ __forceinline__ void mac(C2& acc, const C2& a, const C2& b) {
  acc.r = fma(a.r, b.r, fma(-a.i, b.i, acc.r));
  acc.i = fma(a.r, b.i, fma(a.i, b.r, acc.i));
}
}  // namespace f3

// The y and z transforms run on complex data by conjugate pairs (FdmCoef3):
// fwd_pair returns the pair members' coefficients of the complex 4-vector
// (ur, ui) from the member row (p + iq): 16 FMA + 4 adds for two modes
// instead of 32 FMA.
namespace f3 {
template <bool PARAM>
__device__ __forceinline__ void fwd_pair(const double (&row)[4][2], const double (&ur)[4],
                                         const double (&ui)[4], C2& m0, C2& m1) {
  double A = 0.0, B = 0.0, Cc = 0.0, D = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const C2 f = cf<PARAM>(row[k]);
    A = fma(f.r, ur[k], A);
    B = fma(f.i, ur[k], B);
    Cc = fma(f.r, ui[k], Cc);
    D = fma(f.i, ui[k], D);
  }
  m0 = {A - D, Cc + B};
  m1 = {A + D, Cc - B};
}
// the inverse side: out += (pc + i qc) m0 + (pc - i qc) m1 = pc s + i qc d,
// s = m0 + m1, d = m0 - m1 (formed once per pair by the caller)
__device__ __forceinline__ void inv_pair(const C2& col, const C2& s, const C2& d, C2& out) {
  out.r = fma(col.r, s.r, fma(-col.i, d.i, out.r));
  out.i = fma(col.r, s.i, fma(col.i, d.r, out.i));
}
}  // namespace f3

// OD: the row minus its neighbour couplings, -S(t,t) sum_a (cL_a y[c - e_a]
// trace + cR_a y[c + e_a] trace), before the transforms (FdmOffdiag).  The
// traces are loaded into registers at the top of the segment (both rows of
// the thread at once, ahead of the tile wait): the x / y face lines of the
// row itself, and a quarter of the z-face plane -- the four lanes of one
// (t, cell) hold the four rows z = 0..3 and each loads one line of the
// plane, which the z = 0 (cL) / z = 3 (cR) lane gathers by shuffles.
struct RowTr {
  double x[4], y[4], z[4];
};

__device__ __forceinline__ void ld4_nc(const double* p, double (&v)[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}
__device__ __forceinline__ void st4_g(double* p, double a0, double a1, double a2, double a3) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a0), "d"(a1), "d"(a2),
               "d"(a3)
               : "memory");
}

// both rows of the thread (tid and tid + THREADS: the same cell and z, temporal
// nodes t and t + 2): the neighbour cells once, six 32-byte loads
template <bool OD>
__device__ __forceinline__ void fdm3_rows_prefetch(RowTr& tr0, RowTr& tr1, const FdmOffdiag& od,
                                                   const Geometry& g, int seg, int row) {
  if constexpr (OD) {
    const int t = row / (f3::E * 4), e = (row >> 2) & (f3::E - 1), z = row & 3;
    const int cell = seg * f3::E + e;
    const int cxy = cell % (g.nx * g.ny);
    const int cx = cxy % g.nx, cy = cxy / g.nx, cz = cell / (g.nx * g.ny);
    const long long plane = (long long)4 * g.n_cells * 16;  // one axis' traces
    const long long tstep = 2LL * g.n_cells * 16;           // t -> t + 2
    const double* tt = od.tr_in + (long long)t * g.n_cells * 16;
#pragma unroll
    for (int q = 0; q < 4; ++q) tr0.x[q] = tr0.y[q] = tr0.z[q] = tr1.x[q] = tr1.y[q] = tr1.z[q] = 0.0;
    if (od.cL[0] != 0.0 || od.cR[0] != 0.0) {  // the x-neighbour's face line z: [z][iy]
      const bool L = od.cL[0] != 0.0;
      const int dc = L ? (cx == 0 ? g.nx - 1 : -1) : (cx == g.nx - 1 ? 1 - g.nx : 1);
      const double* p = tt + (long long)(cell + dc) * 16 + z * 4;
      ld4_nc(p, tr0.x);
      ld4_nc(p + tstep, tr1.x);
    }
    if (od.cL[1] != 0.0 || od.cR[1] != 0.0) {  // the y-neighbour's face line z: [z][ix]
      const bool L = od.cL[1] != 0.0;
      const int dc = L ? (cy == 0 ? (g.ny - 1) * g.nx : -g.nx)
                       : (cy == g.ny - 1 ? -(g.ny - 1) * g.nx : g.nx);
      const double* p = tt + plane + (long long)(cell + dc) * 16 + z * 4;
      ld4_nc(p, tr0.y);
      ld4_nc(p + tstep, tr1.y);
    }
    if (od.cL[2] != 0.0 || od.cR[2] != 0.0) {  // line iy = z of the z-neighbour's face
      const bool L = od.cL[2] != 0.0;
      const long long pl = (long long)g.nx * g.ny;
      const long long dc = L ? (cz == 0 ? (g.nz - 1) * pl : -pl) : (cz == g.nz - 1 ? -(g.nz - 1) * pl : pl);
      const double* p = tt + 2 * plane + (cell + dc) * 16 + z * 4;
      ld4_nc(p, tr0.z);
      ld4_nc(p + tstep, tr1.z);
    }
  }
}

// every lane calls it (the z-plane gather shuffles within the 4-lane group)
template <bool OD>
__device__ __forceinline__ void fdm3_row_offdiag(double (&r)[16], const RowTr& tr,
                                                 const FdmOffdiag& od, int row) {
  if constexpr (OD) {
    const int t = row / (f3::E * 4), z = row & 3;
    // (a select chain: a dynamic index into the parameter struct would copy
    // it to local memory)
    const double s = t == 0 ? od.S[0] : (t == 1 ? od.S[1] : (t == 2 ? od.S[2] : od.S[3]));
    if (od.cL[0] != 0.0 || od.cR[0] != 0.0) {
      const int ix = od.cL[0] != 0.0 ? 0 : 3;
      const double f = s * (od.cL[0] != 0.0 ? od.cL[0] : od.cR[0]);
#pragma unroll
      for (int iy = 0; iy < 4; ++iy) {
        if (ix == 0) r[4 * iy] = fma(-f, tr.x[iy], r[4 * iy]);
        else r[4 * iy + 3] = fma(-f, tr.x[iy], r[4 * iy + 3]);
      }
    }
    if (od.cL[1] != 0.0 || od.cR[1] != 0.0) {
      const int o = od.cL[1] != 0.0 ? 0 : 12;
      const double f = s * (od.cL[1] != 0.0 ? od.cL[1] : od.cR[1]);
#pragma unroll
      for (int ix = 0; ix < 4; ++ix) {
        if (o == 0) r[ix] = fma(-f, tr.y[ix], r[ix]);
        else r[12 + ix] = fma(-f, tr.y[ix], r[12 + ix]);
      }
    }
    if (od.cL[2] != 0.0 || od.cR[2] != 0.0) {
      const bool L = od.cL[2] != 0.0;
      const int owner = L ? 0 : 3;
      const double f = s * (L ? od.cL[2] : od.cR[2]);
      const int base = (threadIdx.x & 31) & ~3;
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double v = __shfl_sync(0xffffffffu, tr.z[k], base + q);
          if (z == owner) r[4 * q + k] = fma(-f, v, r[4 * q + k]);
        }
    }
  }
}

// phase A on one (t, cell, z) row: forward x (kept modes j) and y, in place
template <bool PARAM, bool OD>
__device__ __forceinline__ void fdm3_fwd_row(const FdmCoef3& c, double* X, int row,
                                             const FdmOffdiag& od, const RowTr& tr) {
  const int sw = row & 7;
  double r[16];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const double2 v = *reinterpret_cast<const double2*>(X + row * 16 + ((q ^ sw) << 1));
    r[2 * q] = v.x;
    r[2 * q + 1] = v.y;
  }
  fdm3_row_offdiag<OD>(r, tr, od, row);
  double ar[2][4], ai[2][4];  // [j][y]: x-mode j of line y
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    C2 fx[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) fx[x] = f3::cf<PARAM>(c.FX[j][x]);
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        re = fma(fx[x].r, r[4 * y + x], re);
        im = fma(fx[x].i, r[4 * y + x], im);
      }
      ar[j][y] = re;
      ai[j][y] = im;
    }
  }
#pragma unroll
  for (int pr = 0; pr < 2; ++pr)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      C2 m0, m1;
      f3::fwd_pair<PARAM>(c.FY[pr], ar[j], ai[j], m0, m1);
      *reinterpret_cast<double2*>(X + row * 16 + ((((2 * pr) * 2 + j) ^ sw) << 1)) =
          make_double2(m0.r, m0.i);
      *reinterpret_cast<double2*>(X + row * 16 + ((((2 * pr + 1) * 2 + j) ^ sw) << 1)) =
          make_double2(m1.r, m1.i);
    }
}

// phase A' on one row: inverse y and x (2 Re, the 2 folded into IX), in place
template <bool PARAM>
__device__ __forceinline__ void fdm3_inv_row(const FdmCoef3& c, double* X, int row,
                                             const FdmOffdiag& od, const Geometry& g, int seg,
                                             bool trace_out, bool full_out) {
  const int sw = row & 7;
  C2 s[2][2], d[2][2];  // [P][j]: sum and difference of the pair members
#pragma unroll
  for (int pr = 0; pr < 2; ++pr)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double2 v0 =
          *reinterpret_cast<const double2*>(X + row * 16 + ((((2 * pr) * 2 + j) ^ sw) << 1));
      const double2 v1 =
          *reinterpret_cast<const double2*>(X + row * 16 + ((((2 * pr + 1) * 2 + j) ^ sw) << 1));
      s[pr][j] = {v0.x + v1.x, v0.y + v1.y};
      d[pr][j] = {v0.x - v1.x, v0.y - v1.y};
    }
  double o[16];
#pragma unroll
  for (int y = 0; y < 4; ++y) {
    C2 m[2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
    for (int pr = 0; pr < 2; ++pr) {
      const C2 col = f3::cf<PARAM>(c.IY[y][pr]);
#pragma unroll
      for (int j = 0; j < 2; ++j) f3::inv_pair(col, s[pr][j], d[pr][j], m[j]);
    }
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      double re = 0.0;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const C2 ix = f3::cf<PARAM>(c.IX[x][j]);
        re = fma(ix.r, m[j].r, fma(-ix.i, m[j].i, re));
      }
      o[4 * y + x] = re;
    }
  }
  if (trace_out) {  // the faces the downstream neighbours read (FdmOffdiag)
    const int t = row / (f3::E * 4), e = (row >> 2) & (f3::E - 1), z = row & 3;
    const long long cell = (long long)seg * f3::E + e;
    const long long plane = (long long)4 * g.n_cells * 16;
    double* tt = od.tr_out + (long long)t * g.n_cells * 16 + cell * 16;
    auto st4 = [](double* p, double a0, double a1, double a2, double a3) {
      st4_g(p, a0, a1, a2, a3);
    };
    // (constant indices into o[] in both branches: a runtime index would put
    // o in local memory)
    if (od.cL[0] != 0.0)
      st4(tt + z * 4, o[3], o[7], o[11], o[15]);
    else if (od.cR[0] != 0.0)
      st4(tt + z * 4, o[0], o[4], o[8], o[12]);
    if (od.cL[1] != 0.0)
      st4(tt + plane + z * 4, o[12], o[13], o[14], o[15]);
    else if (od.cR[1] != 0.0)
      st4(tt + plane + z * 4, o[0], o[1], o[2], o[3]);
    if (od.cL[2] != 0.0 || od.cR[2] != 0.0) {
      if (z == (od.cL[2] != 0.0 ? 3 : 0)) {
#pragma unroll
        for (int iy = 0; iy < 4; ++iy)
          st4(tt + 2 * plane + iy * 4, o[4 * iy], o[4 * iy + 1], o[4 * iy + 2], o[4 * iy + 3]);
      }
    }
  }
  if (!full_out) return;
#pragma unroll
  for (int q = 0; q < 8; ++q)
    *reinterpret_cast<double2*>(X + row * 16 + ((q ^ sw) << 1)) = make_double2(o[2 * q], o[2 * q + 1]);
}

// phase B on unit (cell e, q = (iy, j)): forward z, the per-mode temporal
// solve, inverse z, in place on the unit's 16 complex (t, z) values
template <bool PARAM>
__device__ __forceinline__ void fdm3_unit(const FdmCoef3& c, const FdmCoef3& cs, double* X, int e,
                                          int q) {
  C2 v[4][4];  // [t][iz] -> [it][iz] -> [t][z], in place in registers
#pragma unroll
  for (int t = 0; t < 4; ++t) {  // loaded and forward z, row by row
    double ur[4], ui[4];
#pragma unroll
    for (int z = 0; z < 4; ++z) {
      const double2 d = *f3::at(X, f3::row_of(t, e, z), q);
      ur[z] = d.x;
      ui[z] = d.y;
    }
#pragma unroll
    for (int pr = 0; pr < 2; ++pr)
      f3::fwd_pair<PARAM>(c.FZ[pr], ur, ui, v[t][2 * pr], v[t][2 * pr + 1]);
  }
#pragma unroll
  for (int iz = 0; iz < 4; ++iz) {  // temporal solve of mode (iz, q), column by column
    C2 y[4];
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      C2 acc = {0.0, 0.0};
#pragma unroll
      for (int t = 0; t < 4; ++t) f3::mac(acc, f3::ld(cs.M[iz][it][t][q]), v[t][iz]);
      y[it] = acc;
    }
#pragma unroll
    for (int it = 0; it < 4; ++it) v[it][iz] = y[it];
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) {  // inverse z, stored
    C2 s[2], d[2];
#pragma unroll
    for (int pr = 0; pr < 2; ++pr) {
      s[pr] = {v[t][2 * pr].r + v[t][2 * pr + 1].r, v[t][2 * pr].i + v[t][2 * pr + 1].i};
      d[pr] = {v[t][2 * pr].r - v[t][2 * pr + 1].r, v[t][2 * pr].i - v[t][2 * pr + 1].i};
    }
#pragma unroll
    for (int z = 0; z < 4; ++z) {
      C2 acc = {0.0, 0.0};
#pragma unroll
      for (int pr = 0; pr < 2; ++pr) f3::inv_pair(f3::cf<PARAM>(c.IZ[z][pr]), s[pr], d[pr], acc);
      *f3::at(X, f3::row_of(t, e, z), q) = make_double2(acc.r, acc.i);
    }
  }
}

// PARAM: the spatial factors are read as kernel-parameter operands (cp is
// the FdmCoef3 by value); otherwise from the shared copy.  The temporal
// table is always read from shared memory (per-lane addresses).
#ifndef STG_FDM3_MINB
#define STG_FDM3_MINB (STG_FDM3_E >= 16 ? 3 : (STG_FDM3_E == 8 ? 4 : 8))
#endif
#ifndef STG_FDM3_ROW_UNROLL
#define STG_FDM3_ROW_UNROLL 1
#endif
namespace f3 {
constexpr int kRowUnroll = STG_FDM3_ROW_UNROLL;
}
template <bool PARAM, bool OD>
__global__ void __launch_bounds__(f3::THREADS, STG_FDM3_MINB)
    fdm3_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm_out,
                const FdmCoef3* __restrict__ coef, const __grid_constant__ FdmCoef3 cp,
                const Geometry g, const Skip skip, const FdmOffdiag od) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (ptxh::smem_u32(smem_raw) & 1023u)) & 1023u);
  const FdmCoef3& cs = *reinterpret_cast<const FdmCoef3*>(base + f3::OFF_C);
  const FdmCoef3& c = PARAM ? cp : cs;
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + f3::OFF_BAR);
  const uint32_t bar0 = ptxh::smem_u32(bars), bar1 = ptxh::smem_u32(bars + 1);
  const int tid = threadIdx.x;
  const int nseg = g.n_cells / f3::E;
  int seg = blockIdx.x;
  // prologue before the programmatic-dependency wait (it overlaps the
  // previous kernel's tail): the barriers and the factor block, which no
  // kernel of the stream writes (uploaded once per mix).  The factors ride
  // on the first tile's barrier phase (expect_tx without arrival; the tile
  // issue below arrives).
  if (tid == 0) {
    ptxh::mbar_init(bar0, 1);
    ptxh::mbar_init(bar1, 1);
    ptxh::fence_mbar_init();
    if (seg < nseg) {
      ptxh::mbar_expect_tx_only(bar0, f3::COEF);
      ptxh::bulk_g2s_1d(ptxh::smem_u32(base + f3::OFF_C), coef, f3::COEF, bar0);
    }
  }
  pdl_entry();
  __syncthreads();
  auto issue = [&](int sg, int st) {
    const uint32_t bar = st ? bar1 : bar0;
    ptxh::mbar_expect_tx(bar, f3::TILE);
    ptxh::tma_load_4d(ptxh::smem_u32(base + st * f3::TILE), &tm, bar, 0, 0, sg * f3::E, 0);
  };
  if (skip_now(skip)) {
    // the factor copy is in flight: it must land before the CTA exits
    if (seg < nseg) {
      if (tid == 0) ptxh::mbar_arrive(bar0);
      while (!ptxh::mbar_try_wait(bar0, 0)) {
      }
    }
    return;
  }
  if (tid == 0 && seg < nseg) issue(seg, 0);
  // phase B unit: q = (iy, j) fastest across the lanes (conflict-free tile
  // reads, one 128-byte wavefront per table read), 4 cells per warp
  const int qB = tid & 7, eB = tid >> 3;

  for (int it = 0; seg < nseg; ++it, seg += gridDim.x) {
    const int st = it & 1;
    double* X = reinterpret_cast<double*>(base + st * f3::TILE);
    if (tid == 0 && seg + (int)gridDim.x < nseg) {
      // stage st^1 last held the previous segment's result: its bulk store
      // must have read it before the next load overwrites it
      ptxh::bulk_wait_read0();
      ptxh::fence_proxy_async_smem();
      issue(seg + gridDim.x, st ^ 1);
    }
    RowTr tr0, tr1;
    fdm3_rows_prefetch<OD>(tr0, tr1, od, g, seg, tid);
    while (!ptxh::mbar_try_wait(st ? bar1 : bar0, (it >> 1) & 1)) {
    }
    fdm3_fwd_row<PARAM, OD>(c, X, tid, od, tr0);
    fdm3_fwd_row<PARAM, OD>(c, X, tid + f3::THREADS, od, tr1);
    __syncthreads();
    fdm3_unit<PARAM>(c, cs, X, eB, qB);
    __syncthreads();
    const bool tr_out = od.tr_out != nullptr, full = od.full_out != 0 || !od.tr_out;
#pragma unroll(f3::kRowUnroll)
    for (int k = 0; k < 2; ++k)
      fdm3_inv_row<PARAM>(c, X, tid + k * f3::THREADS, od, g, seg, tr_out, full);
    ptxh::fence_proxy_async_smem();
    __syncthreads();  // result tile complete
    if (full && tid == 0) {
      ptxh::tma_store_4d(&tm_out, ptxh::smem_u32(X), 0, 0, seg * f3::E, 0);
      ptxh::bulk_commit();
    }
  }
  if (tid == 0) ptxh::bulk_wait0();
}

// ---------------------------------------------------------------------------
// fdm2_kernel: the d = 2 element-block inverse (c2: n = 5, n_tau = 5) by the
// same fast diagonalisation, on the stage-major vectors directly (no
// element-major permutes).  A segment is 32 consecutive cells: n_tau bulk
// copies of 32 * n^2 contiguous doubles.  Phases (one thread per (t, cell)
// plane in A / A', lanes = cells; one warp per kept spatial mode in B):
//   A : forward x (NR real modes with real factors + NP pair members) and y
//   B : (T + theta_m S)^-1 on the n_tau values of each (cell, mode)
//   A': inverse y and x (2 Re for the pair members), in place, bulk store.
// ~5.3k FMA per cell at c2 (a dense 125 x 125 block is 15.6k).
namespace f2 {
constexpr int E = 32;
template <int N1, int NT, int NR, int NP>
struct Shape {
  static constexpr int NPC = N1 * N1;
  static constexpr int KX = NR + NP;         // kept x modes
  static constexpr int KM = N1 * KX;         // kept spatial modes
  static constexpr int THREADS = NT * E;
  static constexpr int NW = THREADS / 32;
  static constexpr int STAGE = NT * E * NPC;  // doubles
  static constexpr int OFF_C = 2 * STAGE * 8;
  static constexpr int OFF_M = OFF_C + NT * KM * E * 16;
  static constexpr int MBYTES = int(sizeof(((FdmCoef2*)nullptr)->M));
  static constexpr int OFF_BAR = OFF_M + MBYTES;
  static constexpr int SMEM = OFF_BAR + 64;
  static_assert(N1 <= kFdm2MaxN && NT <= kFdm2MaxN && NR + 2 * NP == N1, "shape");
  static_assert((E * NPC * 8) % 16 == 0, "bulk copy granularity");
};
}  // namespace f2

template <int N1, int NT, int NR, int NP>
__global__ void __launch_bounds__(f2::Shape<N1, NT, NR, NP>::THREADS)
    fdm2_kernel(const double* __restrict__ in, double* __restrict__ out,
                const FdmCoef2* __restrict__ coef, const __grid_constant__ FdmCoef2 c,
                const Geometry g, const Skip skip) {
  using S = f2::Shape<N1, NT, NR, NP>;
  constexpr int NPC = S::NPC, KX = S::KX, KM = S::KM, E = f2::E;
  extern __shared__ __align__(128) unsigned char smem2[];
  double* st0 = reinterpret_cast<double*>(smem2);
  double2* Ct = reinterpret_cast<double2*>(smem2 + S::OFF_C);  // [t][m][e]
  const double2* Ms = reinterpret_cast<const double2*>(smem2 + S::OFF_M);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem2 + S::OFF_BAR);
  const uint32_t bar0 = ptxh::smem_u32(bars), bar1 = ptxh::smem_u32(bars + 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tA = tid / E, eA = tid % E;
  const long long ns = g.n_sdof;
  const int nseg = g.n_cells / E;
  constexpr uint32_t PB = E * NPC * 8;  // bytes of one temporal block of a segment
  int seg = blockIdx.x;
  // prologue before the programmatic-dependency wait: the barriers and the
  // temporal table (uploaded once per mix, no kernel writes it), which rides
  // on the first segment's barrier phase (expect_tx without arrival)
  if (tid == 0) {
    ptxh::mbar_init(bar0, 1);
    ptxh::mbar_init(bar1, 1);
    ptxh::fence_mbar_init();
    if (seg < nseg) {
      ptxh::mbar_expect_tx_only(bar0, S::MBYTES);
      ptxh::bulk_g2s_1d(ptxh::smem_u32(Ms), coef->M, S::MBYTES, bar0);
    }
  }
  pdl_entry();
  __syncthreads();
  if (skip_now(skip)) {  // the table copy must land before the CTA exits
    if (seg < nseg) {
      if (tid == 0) ptxh::mbar_arrive(bar0);
      while (!ptxh::mbar_try_wait(bar0, 0)) {
      }
    }
    return;
  }
  auto issue = [&](int sg, int st) {
    const uint32_t bar = st ? bar1 : bar0;
    ptxh::mbar_expect_tx(bar, NT * PB);
    const uint32_t dst = ptxh::smem_u32(st0 + st * S::STAGE);
    const double* src = in + (long long)sg * E * NPC;
    for (int t = 0; t < NT; ++t) ptxh::bulk_g2s_1d(dst + t * PB, src + t * ns, PB, bar);
  };
  if (tid == 0 && seg < nseg) issue(seg, 0);

  for (int it = 0; seg < nseg; ++it, seg += gridDim.x) {
    const int st = it & 1;
    double* X = st0 + st * S::STAGE;
    if (tid == 0 && seg + (int)gridDim.x < nseg) {
      ptxh::bulk_wait_read0();  // stage st^1's previous result has been stored
      ptxh::fence_proxy_async_smem();
      issue(seg + gridDim.x, st ^ 1);
    }
    while (!ptxh::mbar_try_wait(st ? bar1 : bar0, (it >> 1) & 1)) {
    }
    // ---- phase A: forward x, y on plane (tA, eA) ---------------------------
    {
      const double* pl = X + (tA * E + eA) * NPC;
      double u[NPC];
#pragma unroll
      for (int k = 0; k < NPC; ++k) u[k] = pl[k];
      double ar[N1][NR > 0 ? NR : 1];
      C2 ac[N1][NP];
#pragma unroll
      for (int y = 0; y < N1; ++y) {
#pragma unroll
        for (int k = 0; k < NR; ++k) {
          double sacc = 0.0;
#pragma unroll
          for (int x = 0; x < N1; ++x) sacc = fma(c.FX[k][x][0], u[y * N1 + x], sacc);
          ar[y][k] = sacc;
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          double re = 0.0, im = 0.0;
#pragma unroll
          for (int x = 0; x < N1; ++x) {
            re = fma(c.FX[NR + p][x][0], u[y * N1 + x], re);
            im = fma(c.FX[NR + p][x][1], u[y * N1 + x], im);
          }
          ac[y][p] = {re, im};
        }
      }
#pragma unroll
      for (int iy = 0; iy < N1; ++iy) {
#pragma unroll
        for (int k = 0; k < NR; ++k) {
          double re = 0.0, im = 0.0;
#pragma unroll
          for (int y = 0; y < N1; ++y) {
            re = fma(c.FY[iy][y][0], ar[y][k], re);
            im = fma(c.FY[iy][y][1], ar[y][k], im);
          }
          Ct[(tA * KM + iy * KX + k) * E + eA] = make_double2(re, im);
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          C2 b = {0.0, 0.0};
#pragma unroll
          for (int y = 0; y < N1; ++y) cmac(b, c.FY[iy][y][0], c.FY[iy][y][1], ac[y][p]);
          Ct[(tA * KM + iy * KX + NR + p) * E + eA] = make_double2(b.r, b.i);
        }
      }
    }
    __syncthreads();
    // ---- phase B: temporal solve per (cell, mode); the mode is warp-uniform --
#pragma unroll 1
    for (int m = warp; m < KM; m += S::NW) {
      C2 v[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const double2 d = Ct[(t * KM + m) * E + lane];
        v[t] = {d.x, d.y};
      }
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        C2 acc = {0.0, 0.0};
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const double2 mm = Ms[(m * kFdm2MaxN + q) * kFdm2MaxN + t];
          cmac(acc, mm.x, mm.y, v[t]);
        }
        Ct[(q * KM + m) * E + lane] = make_double2(acc.r, acc.i);
      }
    }
    __syncthreads();
    // ---- phase A': inverse y, x, in place ----------------------------------
    {
      double* pl = X + (tA * E + eA) * NPC;
      C2 h[N1][KX];
#pragma unroll
      for (int iy = 0; iy < N1; ++iy)
#pragma unroll
        for (int k = 0; k < KX; ++k) {
          const double2 d = Ct[(tA * KM + iy * KX + k) * E + eA];
          h[iy][k] = {d.x, d.y};
        }
#pragma unroll
      for (int y = 0; y < N1; ++y) {
        double mr[NR > 0 ? NR : 1];
        C2 mc[NP];
#pragma unroll
        for (int k = 0; k < NR; ++k) {  // real x mode: the real part is the value
          double re = 0.0;
#pragma unroll
          for (int iy = 0; iy < N1; ++iy)
            re = fma(c.IY[y][iy][0], h[iy][k].r, fma(-c.IY[y][iy][1], h[iy][k].i, re));
          mr[k] = re;
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          C2 b = {0.0, 0.0};
#pragma unroll
          for (int iy = 0; iy < N1; ++iy) cmac(b, c.IY[y][iy][0], c.IY[y][iy][1], h[iy][NR + p]);
          mc[p] = b;
        }
#pragma unroll
        for (int x = 0; x < N1; ++x) {
          double o = 0.0;
#pragma unroll
          for (int k = 0; k < NR; ++k) o = fma(c.IX[x][k][0], mr[k], o);
#pragma unroll
          for (int p = 0; p < NP; ++p)
            o = fma(c.IX[x][NR + p][0], mc[p].r, fma(-c.IX[x][NR + p][1], mc[p].i, o));
          pl[y * N1 + x] = o;
        }
      }
    }
    ptxh::fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      const uint32_t src = ptxh::smem_u32(X);
      double* dst = out + (long long)seg * E * NPC;
      for (int t = 0; t < NT; ++t) ptxh::bulk_s2g_1d(dst + t * ns, src + t * PB, PB);
      ptxh::bulk_commit();
    }
  }
  if (tid == 0) ptxh::bulk_wait0();
}

// ---------------------------------------------------------------------------
// fdm2i_kernel: fdm2 in place (see FdmCoef2i in kernels.hpp).  Plane layout
// after phase A, per (t, cell): for each real x-mode j < NR: NR real y-mode
// values then NP complex y-pair values (n doubles); for each complex x-mode:
// n complex y-mode values (2n doubles).  A thread per (t, cell) plane in
// phases A / A' (lanes = cells: odd plane stride, conflict-free), one warp per
// spatial mode in phase B (table reads are broadcasts).
namespace f2i {
constexpr int E = 32;
template <int N1, int NT, int NR, int NP>
struct Shape {
  static constexpr int NPC = N1 * N1;
  static constexpr int KY = NR + NP;                 // stored y-modes of a real x-column
  static constexpr int NMODE = NR * KY + NP * N1;    // temporal solves per cell
  static constexpr int THREADS = NT * E;
  static constexpr int NW = THREADS / 32;
  static constexpr int STAGE = NT * E * NPC;         // doubles
  static constexpr int MBYTES = int(sizeof(((FdmCoef2i*)nullptr)->M));
  static constexpr int OFF_M = 2 * STAGE * 8;
  static constexpr int OFF_BAR = OFF_M + MBYTES;
  static constexpr int SMEM = OFF_BAR + 64;
  static_assert(NR + 2 * NP == N1 && (N1 & 1) && N1 <= kFdm2MaxN && NT <= kFdm2MaxN, "shape");
  // plane offset of phase-B mode m and whether it is a real value
  __host__ __device__ static constexpr int off(int m) {
    return m < NR * KY ? (m / KY) * N1 + ((m % KY) < NR ? (m % KY) : NR + 2 * ((m % KY) - NR))
                       : NR * N1 + 2 * (m - NR * KY);
  }
  __host__ __device__ static constexpr bool real(int m) { return m < NR * KY && (m % KY) < NR; }
};
}  // namespace f2i

// OD: P0^-1 (in - L y) with y's faces from od.tr_in (FdmOffdiag2); with
// od.tr_out the result's faces are written, with !od.full_out only those
template <int N1, int NT, int NR, int NP, bool OD>
__global__ void __launch_bounds__(f2i::Shape<N1, NT, NR, NP>::THREADS, 3)
    fdm2i_kernel(const double* __restrict__ in, double* __restrict__ out,
                 const FdmCoef2i* __restrict__ coef, const __grid_constant__ FdmCoef2i c,
                 const Geometry g, const Skip skip, const FdmOffdiag2 od) {
  using S = f2i::Shape<N1, NT, NR, NP>;
  constexpr int NPC = S::NPC, KY = S::KY, E = f2i::E;
  extern __shared__ __align__(128) unsigned char smem2i[];
  double* st0 = reinterpret_cast<double*>(smem2i);
  const double2* Ms = reinterpret_cast<const double2*>(smem2i + S::OFF_M);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem2i + S::OFF_BAR);
  const uint32_t bar0 = ptxh::smem_u32(bars), bar1 = ptxh::smem_u32(bars + 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tA = tid / E, eA = tid % E;
  const long long ns = g.n_sdof;
  const int nseg = g.n_cells / E;
  constexpr uint32_t PB = E * NPC * 8;
  int seg = blockIdx.x;
  if (tid == 0) {  // before the dependency wait: barriers, the temporal table
    ptxh::mbar_init(bar0, 1);
    ptxh::mbar_init(bar1, 1);
    ptxh::fence_mbar_init();
    if (seg < nseg) {
      ptxh::mbar_expect_tx_only(bar0, S::MBYTES);
      ptxh::bulk_g2s_1d(ptxh::smem_u32(Ms), coef->M, S::MBYTES, bar0);
    }
  }
  pdl_entry();
  __syncthreads();
  if (skip_now(skip)) {
    if (seg < nseg) {
      if (tid == 0) ptxh::mbar_arrive(bar0);
      while (!ptxh::mbar_try_wait(bar0, 0)) {
      }
    }
    return;
  }
  auto issue = [&](int sg, int st) {
    const uint32_t bar = st ? bar1 : bar0;
    ptxh::mbar_expect_tx(bar, NT * PB);
    const uint32_t dst = ptxh::smem_u32(st0 + st * S::STAGE);
    const double* src = in + (long long)sg * E * NPC;
    for (int t = 0; t < NT; ++t) ptxh::bulk_g2s_1d(dst + t * PB, src + t * ns, PB, bar);
  };
  if (tid == 0 && seg < nseg) issue(seg, 0);

  for (int it = 0; seg < nseg; ++it, seg += gridDim.x) {
    const int st = it & 1;
    double* X = st0 + st * S::STAGE;
    if (tid == 0 && seg + (int)gridDim.x < nseg) {
      ptxh::bulk_wait_read0();
      ptxh::fence_proxy_async_smem();
      issue(seg + gridDim.x, st ^ 1);
    }
    const int cell = seg * E + eA;
    double trx[N1], try_[N1];  // the upwind neighbours' face lines (OD)
    if constexpr (OD) {
      const int cx = cell % g.nx, cy = cell / g.nx;
      const double* tt = od.tr_in + (long long)tA * g.n_cells * N1;
      const long long plane = (long long)NT * g.n_cells * N1;
#pragma unroll
      for (int q = 0; q < N1; ++q) trx[q] = try_[q] = 0.0;
      if (od.cL[0] != 0.0 || od.cR[0] != 0.0) {
        const int dc = od.cL[0] != 0.0 ? (cx == 0 ? g.nx - 1 : -1) : (cx == g.nx - 1 ? 1 - g.nx : 1);
#pragma unroll
        for (int q = 0; q < N1; ++q) trx[q] = __ldg(tt + (long long)(cell + dc) * N1 + q);
      }
      if (od.cL[1] != 0.0 || od.cR[1] != 0.0) {
        const int dc = od.cL[1] != 0.0 ? (cy == 0 ? (g.ny - 1) * g.nx : -g.nx)
                                       : (cy == g.ny - 1 ? -(g.ny - 1) * g.nx : g.nx);
#pragma unroll
        for (int q = 0; q < N1; ++q) try_[q] = __ldg(tt + plane + (long long)(cell + dc) * N1 + q);
      }
    }
    while (!ptxh::mbar_try_wait(st ? bar1 : bar0, (it >> 1) & 1)) {
    }
    double* pl = X + (tA * E + eA) * NPC;
    // ---- phase A: forward x then y, in place -------------------------------
    {
      double u[NPC];
#pragma unroll
      for (int k = 0; k < NPC; ++k) u[k] = pl[k];
      if constexpr (OD) {  // minus the neighbour couplings: S(t,t) (cL / cR) face terms
        double sd = od.S[0];
#pragma unroll
        for (int q = 1; q < NT; ++q) sd = tA == q ? od.S[q] : sd;
        if (od.cL[0] != 0.0) {
#pragma unroll
          for (int y = 0; y < N1; ++y) u[y * N1] = fma(-sd * od.cL[0], trx[y], u[y * N1]);
        } else if (od.cR[0] != 0.0) {
#pragma unroll
          for (int y = 0; y < N1; ++y)
            u[y * N1 + N1 - 1] = fma(-sd * od.cR[0], trx[y], u[y * N1 + N1 - 1]);
        }
        if (od.cL[1] != 0.0) {
#pragma unroll
          for (int x = 0; x < N1; ++x) u[x] = fma(-sd * od.cL[1], try_[x], u[x]);
        } else if (od.cR[1] != 0.0) {
#pragma unroll
          for (int x = 0; x < N1; ++x)
            u[(N1 - 1) * N1 + x] = fma(-sd * od.cR[1], try_[x], u[(N1 - 1) * N1 + x]);
        }
      }
      double ar[NR][N1];  // real x-modes, per y
      C2 ac[NP][N1];      // complex x-modes, per y
#pragma unroll
      for (int y = 0; y < N1; ++y) {
#pragma unroll
        for (int k = 0; k < NR; ++k) {
          double a = 0.0;
#pragma unroll
          for (int x = 0; x < N1; ++x) a = fma(c.FX[k][x][0], u[y * N1 + x], a);
          ar[k][y] = a;
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          double re = 0.0, im = 0.0;
#pragma unroll
          for (int x = 0; x < N1; ++x) {
            re = fma(c.FX[NR + p][x][0], u[y * N1 + x], re);
            im = fma(c.FX[NR + p][x][1], u[y * N1 + x], im);
          }
          ac[p][y] = {re, im};
        }
      }
#pragma unroll
      for (int k = 0; k < NR; ++k) {  // real column: real y-modes, then pair members
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          double a = 0.0;
#pragma unroll
          for (int y = 0; y < N1; ++y) a = fma(c.FY[q][y][0], ar[k][y], a);
          pl[k * N1 + q] = a;
        }
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          double re = 0.0, im = 0.0;
#pragma unroll
          for (int y = 0; y < N1; ++y) {
            re = fma(c.FY[NR + q][y][0], ar[k][y], re);
            im = fma(c.FY[NR + q][y][1], ar[k][y], im);
          }
          pl[k * N1 + NR + 2 * q] = re;
          pl[k * N1 + NR + 2 * q + 1] = im;
        }
      }
#pragma unroll
      for (int p = 0; p < NP; ++p) {  // complex columns: every y-mode
#pragma unroll
        for (int ky = 0; ky < N1; ++ky) {
          C2 b = {0.0, 0.0};
#pragma unroll
          for (int y = 0; y < N1; ++y) cmac(b, c.FY[ky][y][0], c.FY[ky][y][1], ac[p][y]);
          pl[NR * N1 + 2 * (p * N1 + ky)] = b.r;
          pl[NR * N1 + 2 * (p * N1 + ky) + 1] = b.i;
        }
      }
    }
    __syncthreads();
    // ---- phase B: temporal solves, one warp per mode --------------------------
#pragma unroll 1
    for (int m = warp; m < S::NMODE; m += S::NW) {
      const int o = S::off(m);
      double* base = X + lane * NPC + o;
      if (S::real(m)) {
        double v[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) v[t] = base[t * E * NPC];
#pragma unroll
        for (int q = 0; q < NT; ++q) {
          double acc = 0.0;
#pragma unroll
          for (int t = 0; t < NT; ++t) acc = fma(Ms[(m * kFdm2MaxN + q) * kFdm2MaxN + t].x, v[t], acc);
          base[q * E * NPC] = acc;
        }
      } else {
        C2 v[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) v[t] = {base[t * E * NPC], base[t * E * NPC + 1]};
#pragma unroll
        for (int q = 0; q < NT; ++q) {
          C2 acc = {0.0, 0.0};
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const double2 mm = Ms[(m * kFdm2MaxN + q) * kFdm2MaxN + t];
            cmac(acc, mm.x, mm.y, v[t]);
          }
          base[q * E * NPC] = acc.r;
          base[q * E * NPC + 1] = acc.i;
        }
      }
    }
    __syncthreads();
    // ---- phase A': inverse y then x, in place -------------------------------
    const bool full = od.full_out != 0 || !od.tr_out;
    {
      double h[NPC];
#pragma unroll
      for (int k = 0; k < NPC; ++k) h[k] = pl[k];
#pragma unroll
      for (int y = 0; y < N1; ++y) {
        double mr[NR];
        C2 mc[NP];
#pragma unroll
        for (int k = 0; k < NR; ++k) {  // real column: the value is real
          double a = 0.0;
#pragma unroll
          for (int q = 0; q < NR; ++q) a = fma(c.IYW[y][q][0], h[k * N1 + q], a);
#pragma unroll
          for (int q = 0; q < NP; ++q)
            a = fma(c.IYW[y][NR + q][0], h[k * N1 + NR + 2 * q],
                    fma(-c.IYW[y][NR + q][1], h[k * N1 + NR + 2 * q + 1], a));
          mr[k] = a;
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          C2 b = {0.0, 0.0};
#pragma unroll
          for (int ky = 0; ky < N1; ++ky) {
            const C2 hv = {h[NR * N1 + 2 * (p * N1 + ky)], h[NR * N1 + 2 * (p * N1 + ky) + 1]};
            cmac(b, c.IY[y][ky][0], c.IY[y][ky][1], hv);
          }
          mc[p] = b;
        }
        double orow[N1];
#pragma unroll
        for (int x = 0; x < N1; ++x) {
          double o = 0.0;
#pragma unroll
          for (int k = 0; k < NR; ++k) o = fma(c.IX[x][k][0], mr[k], o);
#pragma unroll
          for (int p = 0; p < NP; ++p)
            o = fma(c.IX[x][NR + p][0], mc[p].r, fma(-c.IX[x][NR + p][1], mc[p].i, o));
          orow[x] = o;
          if (full) pl[y * N1 + x] = o;
        }
        if (od.tr_out) {  // the faces the downstream neighbours read
          double* tt = od.tr_out + ((long long)tA * g.n_cells + cell) * N1;
          const long long plane = (long long)NT * g.n_cells * N1;
          if (od.cL[0] != 0.0) tt[y] = orow[N1 - 1];
          else if (od.cR[0] != 0.0) tt[y] = orow[0];
          if ((od.cL[1] != 0.0 && y == N1 - 1) || (od.cR[1] != 0.0 && y == 0)) {
#pragma unroll
            for (int x = 0; x < N1; ++x) tt[plane + x] = orow[x];
          }
        }
      }
    }
    ptxh::fence_proxy_async_smem();
    __syncthreads();
    if (full && tid == 0) {
      const uint32_t src = ptxh::smem_u32(X);
      double* dst = out + (long long)seg * E * NPC;
      for (int t = 0; t < NT; ++t) ptxh::bulk_s2g_1d(dst + t * ns, src + t * PB, PB);
      ptxh::bulk_commit();
    }
  }
  if (tid == 0) ptxh::bulk_wait0();
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
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

bool fdm_supported(const Geometry& g, int n_tau) {
  return g.dim == 3 && g.n1 == 4 && n_tau == 4 && g.n_cells % E == 0 &&
         encode_fn() != nullptr;
}

int launch_precond_fdm(const FdmCoef& coef, const Geometry& g, const double* in, double* out,
                       cudaStream_t s, Skip skip) {
  EncodeFn enc = encode_fn();
  if (!enc || (reinterpret_cast<uintptr_t>(in) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return -1;
  CUtensorMap map;
  const cuuint64_t gdim[4] = {16, 4, cuuint64_t(g.n_cells), 4};
  const cuuint64_t gstride[3] = {128, 512, cuuint64_t(g.n_sdof) * 8};
  const cuuint32_t box[4] = {16, 4, E, 4};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(in), gdim, gstride, box,
          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;
  CUtensorMap map_out;
  if (enc(&map_out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, out, gdim, gstride, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;
  // 3 CTAs/SM (144 registers, no spills) by default; STG_FDM_MINB=4 trades a
  // small spill for a fourth CTA
  static const bool four = [] {
    const char* e = std::getenv("STG_FDM_MINB");
    return e && std::atoi(e) == 4;
  }();
  auto kern = four ? fdm_kernel<4> : fdm_kernel<3>;
  static int occ_dev[kMaxDevices];  // 0: not set up on that device yet
  int& occ = occ_dev[device_slot()];
  if (occ <= 0) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, THREADS, SMEM);
    if (occ < 1) occ = 1;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nseg = g.n_cells / E;
  int grid = occ * sms;
  if (grid > nseg) grid = nseg;
  launch_ex(kPdlFdm, kern, grid, THREADS, SMEM, s, map, map_out, coef, g, skip);
  return 1;
}

bool fdm3_supported(const Geometry& g, int n_tau) {
  return g.dim == 3 && g.n1 == 4 && n_tau == 4 && g.n_cells % f3::E == 0 &&
         encode_fn() != nullptr && !std::getenv("STG_FDM_V1");
}

int launch_precond_fdm3(const FdmCoef3* coef, const FdmCoef3& host_coef, const Geometry& g,
                        const double* in, double* out, cudaStream_t s, Skip skip,
                        const FdmOffdiag* od) {
  EncodeFn enc = encode_fn();
  if (!enc || (reinterpret_cast<uintptr_t>(in) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return -1;
  const cuuint64_t gdim[4] = {16, 4, cuuint64_t(g.n_cells), 4};
  const cuuint64_t gstride[3] = {128, 512, cuuint64_t(g.n_sdof) * 8};
  const cuuint32_t box[4] = {16, 4, f3::E, 4};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUtensorMap map, map_out;
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(in), gdim, gstride, box,
          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;
  if (enc(&map_out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, out, gdim, gstride, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;
  static const bool smem_coef = std::getenv("STG_FDM3_SMEMC") != nullptr;
  const bool coupled = od && od->tr_in;
  auto kern = coupled ? (smem_coef ? fdm3_kernel<false, true> : fdm3_kernel<true, true>)
                      : (smem_coef ? fdm3_kernel<false, false> : fdm3_kernel<true, false>);
  static int occ_dev[kMaxDevices];
  const int dev = device_slot();
  int& occ = occ_dev[dev];
  if (occ <= 0) {
    for (auto k : {fdm3_kernel<false, false>, fdm3_kernel<true, false>, fdm3_kernel<false, true>,
                   fdm3_kernel<true, true>})
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, f3::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, f3::THREADS, f3::SMEM);
    if (occ < 1) occ = 1;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nseg = g.n_cells / f3::E;
  int grid = occ * sms;
  if (grid > nseg) grid = nseg;
  launch_ex(kPdlFdm, kern, grid, f3::THREADS, f3::SMEM, s, map, map_out, coef, host_coef, g, skip,
            od ? *od : FdmOffdiag{});
  return 1;
}

namespace {
// (n1, n_tau, nr, np) instances: c2 (5, 5, 1, 2) and the n = 4 / 3 analogues
template <int N1, int NT, int NR, int NP>
int launch_fdm2_t(const FdmCoef2* coef, const FdmCoef2& hc, const Geometry& g, const double* in,
                  double* out, cudaStream_t s, Skip skip) {
  using S = f2::Shape<N1, NT, NR, NP>;
  static int occ_dev[kMaxDevices];
  const int dev = device_slot();
  int& occ = occ_dev[dev];
  if (occ <= 0) {
    cudaFuncSetAttribute(fdm2_kernel<N1, NT, NR, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         S::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fdm2_kernel<N1, NT, NR, NP>, S::THREADS,
                                                  S::SMEM);
    if (occ < 1) occ = 1;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nseg = g.n_cells / f2::E;
  int grid = occ * sms;
  if (grid > nseg) grid = nseg;
  launch_ex(kPdlFdm, fdm2_kernel<N1, NT, NR, NP>, grid, S::THREADS, S::SMEM, s, in, out, coef, hc,
            g, skip);
  return 1;
}
}  // namespace

bool fdm2_supported(const Geometry& g, int n_tau, int nr, int np) {
  if (g.dim != 2 || g.n_cells % f2::E != 0 || (g.n_sdof * 8) % 16 != 0 || std::getenv("STG_NO_FDM2"))
    return false;
  return (g.n1 == 5 && n_tau == 5 && nr == 1 && np == 2) ||
         (g.n1 == 4 && n_tau == 4 && nr == 0 && np == 2) ||
         (g.n1 == 3 && n_tau == 3 && nr == 1 && np == 1);
}

int launch_precond_fdm2(const FdmCoef2* coef, const FdmCoef2& hc, const Geometry& g, int n_tau,
                        int nr, int np, const double* in, double* out, cudaStream_t s, Skip skip) {
  if (!fdm2_supported(g, n_tau, nr, np) || (reinterpret_cast<uintptr_t>(in) & 15) ||
      (reinterpret_cast<uintptr_t>(out) & 15))
    return -1;
  if (g.n1 == 5) return launch_fdm2_t<5, 5, 1, 2>(coef, hc, g, in, out, s, skip);
  if (g.n1 == 4) return launch_fdm2_t<4, 4, 0, 2>(coef, hc, g, in, out, s, skip);
  return launch_fdm2_t<3, 3, 1, 1>(coef, hc, g, in, out, s, skip);
}

bool fdm2i_supported(const Geometry& g, int n_tau, int nr, int np) {
  if (g.dim != 2 || g.n_cells % f2i::E != 0 || (g.n_sdof * 8) % 16 != 0 ||
      std::getenv("STG_NO_FDM2") || std::getenv("STG_NO_FDM2I"))
    return false;
  return (g.n1 == 5 && n_tau == 5 && nr == 1 && np == 2) ||
         (g.n1 == 3 && n_tau == 3 && nr == 1 && np == 1);
}

namespace {
template <int N1, int NT, int NR, int NP>
int launch_fdm2i_t(const FdmCoef2i* coef, const FdmCoef2i& hc, const Geometry& g,
                   const double* in, double* out, cudaStream_t s, Skip skip,
                   const FdmOffdiag2* od) {
  using S = f2i::Shape<N1, NT, NR, NP>;
  static int occ_dev[kMaxDevices];
  const int dev = device_slot();
  int& occ = occ_dev[dev];
  if (occ <= 0) {
    for (auto k : {fdm2i_kernel<N1, NT, NR, NP, false>, fdm2i_kernel<N1, NT, NR, NP, true>})
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fdm2i_kernel<N1, NT, NR, NP, true>,
                                                  S::THREADS, S::SMEM);
    if (occ < 1) occ = 1;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nseg = g.n_cells / f2i::E;
  int grid = occ * sms;
  if (grid > nseg) grid = nseg;
  auto kern = od && od->tr_in ? fdm2i_kernel<N1, NT, NR, NP, true>
                              : fdm2i_kernel<N1, NT, NR, NP, false>;
  launch_ex(kPdlFdm, kern, grid, S::THREADS, S::SMEM, s, in, out, coef, hc, g, skip,
            od ? *od : FdmOffdiag2{});
  return 1;
}
}  // namespace

int launch_precond_fdm2i(const FdmCoef2i* coef, const FdmCoef2i& hc, const Geometry& g, int n_tau,
                         const double* in, double* out, cudaStream_t s, Skip skip,
                         const FdmOffdiag2* od) {
  if ((reinterpret_cast<uintptr_t>(in) & 15) || (reinterpret_cast<uintptr_t>(out) & 15)) return -1;
  if (g.n1 == 5 && n_tau == 5) return launch_fdm2i_t<5, 5, 1, 2>(coef, hc, g, in, out, s, skip, od);
  if (g.n1 == 3 && n_tau == 3) return launch_fdm2i_t<3, 3, 1, 1>(coef, hc, g, in, out, s, skip, od);
  return -1;
}

}  // namespace stg
