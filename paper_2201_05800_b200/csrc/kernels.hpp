// Device-side data structures and kernel launchers of the slab operator.
//
// Every slab-type apply of the reference is one fused kernel of the form
//
//   R_r = sum_j T(r,j) X_j + sum_j S(r,j) G_j + c_r W          (r < n_out)
//
// where X_j (j < n_in) are the input temporal blocks, G_j = F(X_j) is the
// DG-SEM spatial operator applied per block (spatial.hpp:107-266) -- or its
// Jacobian action J_F(U_j) X_j -- and W is an optional spatial vector.
// The reference callers map onto (T, S, c) as follows (built in stg.cpp):
//   st_residual   (stdg.hpp:56-76):  T = e e^T - D^T M, S = -(dt/2) M, c = -e_1, W = u_n
//   st_jacobian v (stdg.hpp:79-110): same T, S, c = 0
//   rk residual A-form   (lodg.hpp:111-114): T = I, S = -dt A, c = -1, W = u
//   rk residual A^-1-form (lodg.hpp:116-118): T = A^-1/dt, S = -I, c = -rowsum(A^-1)/dt
//   rk u_next (lodg.hpp:142-145): n_out = 1, T = 0, S = dt b^T, c = 1, W = u
//   SemiDiscreteSystem::rhs:          n_in = n_out = 1, T = 0, S = 1, c = 0
#pragma once

#include <cstdint>
#include <utility>

#include <cuda_runtime.h>

namespace stg {

constexpr int kMaxN = 6;  // max LGL nodes per axis (degree <= 5)
constexpr int kMaxT = 6;  // max temporal nodes / stages

// Spatial operator coefficients for constant-velocity advection, weak form
// divided by the diagonal mass (spatial.hpp:117-156, 158-208, 265):
//   F[.. i_a ..] += V[a][i][k] u[.. k ..]                 (volume + own traces)
//   F[.. i_a = 0 ..] += cL[a] * u_{c - e_a}[.. i_a = N ..] (upwind neighbour)
//   F[.. i_a = N ..] += cR[a] * u_{c + e_a}[.. i_a = 0 ..] (downwind neighbour)
// with V[a][i][k] = (2/h_a) b_a w_k D(k,i)/w_i plus the LLF own-trace terms
// -(2/h_a)/w_N * alpha_a at (N,N) and +(2/h_a)/w_0 * beta_a at (0,0),
// alpha = (b+|b|)/2, beta = (b-|b|)/2 (llf_flux, spatial.hpp:20-25).
struct SpatialCoef {
  double V[3][kMaxN][kMaxN];
  double cL[3];
  double cR[3];
  // Burgers (d = 1, EXTENSION): raw D(i,k), 2/h and 1/w_0, 1/w_N
  double Dm[kMaxN][kMaxN];
  double sc;
  double inv_w0;
  double inv_wN;
};

struct MixCoef {
  double T[kMaxT][kMaxT];
  double S[kMaxT][kMaxT];
  double c[kMaxT];
};

struct Geometry {
  int dim;
  int n1;      // LGL nodes per axis
  int npc;     // nodes per cell
  int nx, ny, nz;
  int n_cells;
  long long n_sdof;
};

enum class Model : int { advection = 0, burgers = 1 };

// Device-side cancellation of queued work.  The GMRES driver enqueues the
// next Arnoldi step before it has read the outcome of the current one; every
// kernel of a step carries a Skip and returns at entry unless *flag == run
// (flag null: always run).  The flag is written by an earlier kernel on the
// same stream, so stream order makes it visible.
struct Skip {
  const int* flag = nullptr;
  int run = 0;
};
#ifdef __CUDACC__
__device__ __forceinline__ bool skip_now(const Skip& s) {
  return s.flag != nullptr && *reinterpret_cast<const volatile int*>(s.flag) != s.run;
}

// Programmatic dependent launch.  The hot kernels are launched with
// programmatic stream serialisation (launch_pdl) and start with pdl_entry():
// wait until the preceding kernel has completed and its writes are visible
// (griddepcontrol.wait -- before ANY global read, the skip flag included),
// then let the next kernel be scheduled at once, so its launch and prologue
// overlap this kernel's tail instead of following it.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// kernel classes for STG_PDL_MASK (A/B measurements; default: all on;
// STG_NO_PDL: all off)
enum PdlClass : int { kPdlSlab = 1, kPdlFdm = 2, kPdlVec = 4, kPdlPrecond = 8 };
bool pdl_enabled(int cls);

// Per-device caches of launch attributes (occupancy, SM count, the max
// dynamic shared memory attribute) are indexed by the current device: a
// handle may be used on any GPU, and cudaFuncSetAttribute is per device.
constexpr int kMaxDevices = 64;
inline int device_slot() {
  int d = 0;
  cudaGetDevice(&d);
  return d >= 0 && d < kMaxDevices ? d : kMaxDevices - 1;
}

template <typename... KArgs, typename... Args>
inline void launch_ex(int pdl_cls, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                      cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled(pdl_cls) ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

#endif

// Device state of one GMRES(m) cycle (stg.cpp, gmres): the Hessenberg matrix
// reduced by Givens rotations, the rotations, the rotated right-hand side g,
// the inverse norms c_j = 1/||S_j|| of the stored basis vectors, and the
// cycle status: 0 running, 1 residual estimate <= tol_abs, 2 breakdown,
// 3 the last step needs a second Gram-Schmidt pass, 4 nothing to do (b = 0),
// 5 the initial residual norm is NaN / infinite (the solve fails).
constexpr int kGmresMaxRestart = 60;
struct GmresDev {
  double H[(kGmresMaxRestart + 1) * kGmresMaxRestart];  // H(i,j) at i*m + j
  double cs[kGmresMaxRestart], sn[kGmresMaxRestart];
  double g[kGmresMaxRestart + 1];
  double cn[kGmresMaxRestart + 1];
  double tol_abs, reorth_tol, est, bnorm;
  int m, status, k_done, pad;
};
// The Givens step of Arnoldi step k, run by the last block of the update
// pass: pass 0 after the first projection (raw dots d1 = <S_j, w>, j <= k,
// and d1[k+1] = <w,w>), pass 1 after a re-orthogonalisation (raw dots d2).
// The step's status is mirrored to host-mapped memory (host[k]).
struct GivensArgs {
  GmresDev* G = nullptr;
  int k = 0;
  int pass = 0;
  const double* d1 = nullptr;
  const double* sc1 = nullptr;  // scale applied by pass 0 (pass 1 reads it)
  int* host = nullptr;          // mapped pinned per-step status slots
  // a step that converges within kInlineBacksub columns also leaves the
  // cycle's update coefficients y_j c_j here (no k_gmres_backsub launch)
  double* ysol = nullptr;
};
constexpr int kInlineBacksub = 8;
// bb != null: beta = sqrt(*bb) on the device and tol is relative (first
// cycle from x = 0, no host round trip); else beta and tol_abs = tol given.
// beta = 0 sets status 4 ("no work") and writes it to every host slot.
// s0_sign != 0: S_0 is b itself, unnormalised (c_0 = 1/||b||, ||S_0||^2 =
// <b,b>), and the right-hand side's sign goes into g_0 = s0_sign ||b||
void gmres_init(GmresDev* G, int m, const double* bb, double beta, double tol, double reorth_tol,
                double* hn2_0, int* host, cudaStream_t s, double s0_sign = 0.0);
// out[j] = y_j c_j, y = R^-1 g over the first k columns (the cycle's update)
void gmres_backsub(const GmresDev* G, int k, double* out, cudaStream_t s);

struct SlabArgs {
  SpatialCoef sp;
  MixCoef mx;
  Geometry g;
  int n_in;     // input temporal blocks
  int n_out;    // output blocks
  int has_w;    // W term present
  int jvp;      // 0: G = F(X); 1: G = J_F(U) X (Burgers; advection ignores U)
  int full_s;   // S not diagonal
  int model;
  const double* X;  // n_in blocks
  // X holds ONE spatial block standing for all n_in (the initial guess
  // 1 (x) u_n of a slab solve, never written out): fast 3-D kernel only (its
  // tensor maps get a zero temporal stride); other launchers return -1
  int x_bcast;
  const double* U;  // linearisation point (jvp && burgers), n_in blocks
  const double* W;  // spatial vector or null
  double* R;        // n_out blocks
  // fast 3-D path only: process 8-cell segments [seg_begin, seg_end) of the
  // mesh (seg_end == 0: all).  Used by the pipelined host-buffer entry point.
  int seg_begin;
  int seg_end;
  // fused central-difference Jacobian action (d = 1 lane kernel): when fdv is
  // set, X is the linearisation point U and the kernel returns
  // T v + S [F(U + e v) - F(U - e v)] / (2e), e = fd_c / sqrt(*fd_vv)
  // (fd_vv = <v,v> on the device: no host round trip)
  const double* fdv;
  const double* fd_vv;
  double fd_c;
  // fd_uu != null: e = fd_c * sqrt(1 + sqrt(*fd_uu)) / sqrt(*fd_vv), with
  // fd_uu = <U,U> also on the device (fd_c then holds fd_eps)
  const double* fd_uu;
  Skip skip;
  // launch without programmatic serialisation (the launch follows a
  // cross-stream event wait, which PDL must not relax)
  int no_pdl;
  // fused reductions of R (fast 3-D kernel; red_done reports whether the
  // launched kernel produced them): *red_max = max |R_i| as the bit pattern
  // of a non-negative double (zeroed beforehand), *red_ss = <R,R> summed in
  // fixed order over per-CTA partials (red_part, with its completion counter
  // right after kPartialDoubles doubles)
  unsigned long long* red_max;
  double* red_ss;
  double* red_part;
};
// whether launch_slab_fast / launch_slab_generic compute the fused R
// reductions for these args (fast 3-D kernel / d = 2 plane kernel)
bool slab_fast_reduces(const SlabArgs& a);
bool slab_generic_reduces(const SlabArgs& a);
// true if the d = 1 lane kernel handles fused FD Jacobian actions for a
bool fd_fused_supported(const SlabArgs& a);

// ---- launchers (kernels_slab.cu) -------------------------------------------
// Returns the number of kernels launched (>= 1) or -1 if no kernel fits.
int launch_slab_generic(const SlabArgs& a, cudaStream_t s);
// Fast TMA path: d = 3, n = 4, n_in = n_out = 4, advection, nx % 8 == 0.
bool slab_fast_supported(const SlabArgs& a);
bool slab_fast_bcast_ok();
int launch_slab_fast(const SlabArgs& a, cudaStream_t s);

// ---- general flux models, d in {1, 2} (kernels_general.cu) -----------------
// r = 1: advdiff_model (constant / rotating velocity, eps >= 0, interior
// penalty eta); r = 4: euler_model(gamma).
struct GenCoef {
  int r;
  int field;      // 0 constant b, 1 rotating_field (models.hpp:79-85)
  double b[2];
  double eps, eta, gamma;
  double xi[kMaxN], w[kMaxN];
  double D[kMaxN][kMaxN];  // D[j][i] = D(j,i) = psi_i'(x_j)
  double h[2], lower[2];
  double vol_scale;        // prod(h) / 2^d (global_mass, mesh.hpp:125-141)
};
struct GenArgs {
  GenCoef c;
  Geometry g;     // n_sdof includes the r components
  MixCoef mx;
  int n_in, n_out;
  const double* X;     // n_in blocks: F_j = F(X_j)
  const double* Xmix;  // blocks of the T term (null: none)
  const double* W;     // spatial vector of the c term (null: none)
  double* F;           // workspace, n_in blocks
  double* R;           // n_out blocks (null: only F is computed)
  int* err;            // admissibility flag: 1 + first failing block
  Skip skip;
};
// Returns the number of kernels launched, or -1 if (d, n, r) is unsupported.
int launch_general(const GenArgs& a, cudaStream_t s);

// ---- fused small-problem Newton-GMRES (kernels_small.cu) -------------------
constexpr int kSmallMaxRestart = 30;
#define STG_MAX_HISTORY_DEV 64
struct SmallSolveOut {
  int status;  // 0 ok, 1 Newton did not converge, 2 GMRES did not converge
  int newton_iterations, linear_iterations, n_history;
  double final_residual, gmres_rel;
  double history[STG_MAX_HISTORY_DEV];
};
struct SmallSolveArgs {
  SpatialCoef sp;
  MixCoef mx_res, mx_jac, mx_next;  // residual (with W), Jacobian, rk u_next
  int n, K, nt, n1;                  // n = nt * ns
  long long ns, ld;                  // spatial size, basis leading dimension
  int restart, max_it, max_iter, rk;
  double tol, abs_tol, rel_tol;
  const double* W;    // u_n (stdg) or u (rk)
  const double* B;    // element-block inverse (nt*n1)^2 or null (no preconditioner)
  double* V;          // basis workspace, (restart + 1) * ld (vectors not held in smem)
  int basis_in_smem;  // set by the launcher
  double* U_out;      // n
  double* u_next;     // ns or null
  SmallSolveOut* out;
};
bool small_solve_supported(const Geometry& g, int nt, int model, int restart);
int launch_small_solve(SmallSolveArgs a, cudaStream_t s);

// ---- element-block Jacobi by fast diagonalisation, d = 3 N = 3 n_tau = 4
// (kernels_fdm.cu).  Complex entries are stored [re, im]; x eigen-indices are
// kept for one member of each conjugate pair (kx = 2j, j = 0, 1).
struct FdmCoef {
  double FX[2][4][2];        // rows 0, 2 of Px^-1
  double FY[4][4][2];        // Py^-1
  double FZ[4][4][2];        // Pz^-1
  double FT[4][4][2];        // Q^-1 S^-1
  double IT[4][4][2];        // Q
  double IZ[4][4][2];        // Pz
  double IY[4][4][2];        // Py
  double IX[4][2][2];        // columns 0, 2 of Px
  double LI[4][4][4][2][2];  // 1 / (lt[it] + thz[iz] + thy[iy] + thx[2j])
};
bool fdm_supported(const Geometry& g, int n_tau);
int launch_precond_fdm(const FdmCoef& c, const Geometry& g, const double* in, double* out,
                       cudaStream_t s, Skip skip = {});

// FDM with a direct temporal solve per spatial mode (kernels_fdm.cu,
// fdm3_kernel): L_e^-1 = (I (x) Pz (x) Py (x) Px) blockdiag_theta((T + theta S)^-1)
// (I (x) Pz^-1 (x) Py^-1 (x) Px^-1), theta = thz + thy + thx over the kept
// modes -- no eigen-decomposition of the temporal operator, and S need not be
// invertible.  The per-mode n_tau x n_tau complex inverses live in device
// memory, [iz][it][t][q] with q = iy * 2 + j fastest (M).
// One device block, copied to shared memory by one bulk copy per CTA:
// the spatial factors (complex [re, im]) followed by the temporal table.
// Every axis has two complex-conjugate eigenvalue pairs (2P, 2P + 1), whose
// eigenvector columns (rows of P^-1) are exact conjugates, so one member of a
// pair carries the pair: with a row p + iq of P^-1, the coefficients of the
// pair members of a complex vector u are (p.Re u - q.Im u) + i(p.Im u + q.Re u)
// and (p.Re u + q.Im u) + i(p.Im u - q.Re u), four real dots and four adds
// instead of two complex dots; the inverse side likewise.
struct FdmCoef3 {
  double FX[2][4][2];  // rows 0, 2 of Px^-1 (one of each conjugate pair)
  double FY[2][4][2];  // rows 0, 2 of Py^-1 ([P][y] = p + iq of row 2P)
  double FZ[2][4][2];  // rows 0, 2 of Pz^-1
  double IZ[4][2][2];  // columns 0, 2 of Pz ([z][P])
  double IY[4][2][2];  // columns 0, 2 of Py
  double IX[4][2][2];  // 2 x columns 0, 2 of Px (the factor 2 of 2 Re(.) folded in)
  double M[4][4][4][8][2];  // [iz][it][t][q]: (T + theta S)^-1, q = iy * 2 + j
};
static_assert(sizeof(FdmCoef3) % 16 == 0, "bulk-copied block");
bool fdm3_supported(const Geometry& g, int n_tau);
// coef: a device copy of host_coef (the kernel reads its spatial factors as
// parameters and bulk-copies the temporal table)
// The neighbour couplings of a Neumann step folded into the block apply:
// with od, fdm3_kernel computes out = P0^-1 (in - L y) (L: the upwind face
// terms cL / cR of the constant-velocity advection Jacobian, mixed by the
// diagonal S), reading y's neighbour traces while it stages each row.
// The neighbour traces travel between the chain's steps in a compact array
// instead of the full iterate: trace[a][t][cell][16] holds, per axis a, the
// face of the cell its downstream neighbour reads (i_a = N for cL_a != 0,
// i_a = 0 for cR_a != 0): x [z][iy], y [z][ix], z [iy][ix].
struct FdmOffdiag {
  const double* tr_in;  // traces of y_i (nullptr: no coupling, the plain block apply)
  double* tr_out;       // traces of the result (nullptr: none)
  int full_out;         // 0: the result itself is not stored (an intermediate term)
  double S[4];          // diagonal of the temporal mix S
  double cL[3], cR[3];  // SpatialCoef face coefficients
};
inline long long fdm_trace_doubles(const Geometry& g, int nt) {
  return 3LL * nt * g.n_cells * 16;
}
int launch_precond_fdm3(const FdmCoef3* coef, const FdmCoef3& host_coef, const Geometry& g,
                        const double* in, double* out, cudaStream_t s, Skip skip = {},
                        const FdmOffdiag* od = nullptr);

// d = 2 element-block inverse by fast diagonalisation (kernels_fdm.cu,
// fdm2_kernel): L_e^-1 = (I (x) Py (x) Px) blockdiag_theta((T + theta S)^-1)
// (I (x) Py^-1 (x) Px^-1) over the kept spatial modes theta = thy + thx, x
// modes: the NR real eigenvalues of V_x (real eigenvectors) then one member
// of each of the NP complex-conjugate pairs.  One device block per mix;
// complex entries [re, im]; sized for n <= 5, n_tau <= 5.
constexpr int kFdm2MaxN = 5;
struct FdmCoef2 {
  double FX[kFdm2MaxN][kFdm2MaxN][2];  // kept rows of Px^-1 ([kept k][x])
  double FY[kFdm2MaxN][kFdm2MaxN][2];  // Py^-1 ([iy][y])
  double IY[kFdm2MaxN][kFdm2MaxN][2];  // Py ([y][iy])
  double IX[kFdm2MaxN][kFdm2MaxN][2];  // kept columns of Px, x2 for pair members ([x][k])
  // [m = iy * KX + k][it][t]: (T + theta_m S)^-1
  double M[kFdm2MaxN * kFdm2MaxN][kFdm2MaxN][kFdm2MaxN][2];
};
static_assert(sizeof(FdmCoef2) % 16 == 0, "bulk-copied block");
// fdm2i_kernel (odd n: 3, 5): the same inverse computed IN PLACE in the
// input stage.  The y-transform of a real x-mode column is real data, so it
// keeps one member of each y conjugate pair too: per (t, cell) plane the
// transformed values take exactly n^2 doubles (NR real x-modes x (NR reals +
// NP complex) + NP complex x-modes x n complex), no separate complex tile,
// 3 CTAs/SM, and NR*NR + NR*NP + NP*n temporal solves per cell (13 at n = 5
// instead of 15).  y-modes are ordered [real (NR), pair members with
// Im > 0 (NP), their conjugates (NP)].
struct FdmCoef2i {
  double FX[kFdm2MaxN][kFdm2MaxN][2];   // kept x rows of Px^-1 ([k][x]; real modes: im 0)
  double FY[kFdm2MaxN][kFdm2MaxN][2];   // Py^-1 rows in y-mode order ([ky][y])
  double IY[kFdm2MaxN][kFdm2MaxN][2];   // Py columns in y-mode order ([y][ky])
  double IYW[kFdm2MaxN][kFdm2MaxN][2];  // real x-mode columns: IY x (1 real / 2 pair) ([y][ky < NR+NP])
  double IX[kFdm2MaxN][kFdm2MaxN][2];   // kept x columns of Px, x (1 / 2) ([x][k])
  // [m][it][t]: (T + theta_m S)^-1 in phase-B mode order: real x-modes
  // (j < NR) x y-modes ky < NR+NP, then complex x-modes x all n y-modes
  double M[kFdm2MaxN * kFdm2MaxN][kFdm2MaxN][kFdm2MaxN][2];
};
static_assert(sizeof(FdmCoef2i) % 16 == 0, "bulk-copied block");
bool fdm2i_supported(const Geometry& g, int n_tau, int nr, int np);
// d = 2 analogue of FdmOffdiag for fdm2i_kernel: trace[a][t][cell][n]
// holds the face line its downstream neighbour reads (x: [iy], y: [ix]).
struct FdmOffdiag2 {
  const double* tr_in;
  double* tr_out;
  int full_out;
  double S[kFdm2MaxN];
  double cL[2], cR[2];
};
inline long long fdm2_trace_doubles(const Geometry& g, int nt) {
  return 2LL * nt * g.n_cells * g.n1;
}
int launch_precond_fdm2i(const FdmCoef2i* coef, const FdmCoef2i& host_coef, const Geometry& g,
                         int n_tau, const double* in, double* out, cudaStream_t s,
                         Skip skip = {}, const FdmOffdiag2* od = nullptr);

// n1 / n_tau / (real, pair) x-mode counts the kernel is instantiated for
bool fdm2_supported(const Geometry& g, int n_tau, int nr, int np);
int launch_precond_fdm2(const FdmCoef2* coef, const FdmCoef2& host_coef, const Geometry& g,
                        int n_tau, int nr, int np, const double* in, double* out, cudaStream_t s,
                        Skip skip = {});

// ---- block-Jacobi preconditioners (kernels_precond.cu) ----------------------
// out[t][cell][k] = sum_j minv[k][t][j] in[j][cell][k]   (npc class tables)
void precond_tblock(double* out, const double* in, const double* minv, int nt, int npc,
                    long long ns, cudaStream_t s, Skip skip = {});
// out_e = B_e in_e, B_e = B + e * bstride (bstride 0: one shared block), d = 1
void precond_eblock(double* out, const double* in, const double* B, long long bstride, int nt,
                    int n1, int ncells, long long ns, cudaStream_t s, Skip skip = {});
// d = 2: out_e = B in_e with ONE shared dense block B ((n_tau*npc)^2, <= 128^2)
bool precond_eblock_dense(double* out, const double* in, const double* B, int nt, int npc,
                          int ncells, long long ns, cudaStream_t s, Skip skip = {});
// element blocks of the general linear models by coloured probing
// (ndl = element-local DOFs per temporal block = npc * r)
void probe_set(double* P, int ndl, int col, int nx, int ny, int sx, int sy, int cx0, int cy0,
               int ncells, cudaStream_t s);
void probe_extract(double* K, const double* F, int ndl, int col, int nx, int sx, int sy, int cx0,
                   int cy0, int ncells, cudaStream_t s);
// Binv_e = (T (x) I + S (x) K_e)^-1 per element (nt * ndl <= 32)
bool gen_eblock_invert(double* Binv, const double* K, const MixCoef& mx, int nt, int ndl,
                       int ncells, cudaStream_t s);
// per-element inverse blocks of the 1-D Burgers slab/stage Jacobian at U,
// stored in fp32 (a preconditioner; applied in fp64 arithmetic)
// G (may be null): the upwind-sweep inflow couplings B_e^-1 L_e (fp32)
bool build_burgers_eblock(float* Binv, float* G, const double* U, const SlabArgs& a,
                          cudaStream_t s);
// out_e = B_e in_e with per-element fp32 blocks, nt*n1 <= 16 and even
bool eblock_f32_supported(int nt, int n1);
// d = 1 upwind block sweep (kernels_precond.cu: k_eblock2, k_sweep_win): the
// element blocks B (fp32, build_burgers_eblock) plus the inflow couplings G;
// work: sweep_work_doubles(nt, ncells, n1) doubles (y = B^-1 in).
// n_tau = 4, N + 1 in {2, 4}.
bool offdiag_supported(const Geometry& g, int nt);
// out = r - L y, L the neighbour couplings of the constant-velocity advection
// Jacobian (mix mx); false (nothing launched) for an uninstantiated shape
bool offdiag_residual(double* out, const double* r, const double* y, const SpatialCoef& sp,
                      const MixCoef& mx, const Geometry& g, int nt, cudaStream_t s, Skip skip);
bool sweep_supported(int nt, int n1);
size_t sweep_work_doubles(int nt, int ncells, int n1);
// vv (with partial): also <out, out> into *vv
void precond_sweep(double* out, const double* in, const float* B, const float* G, double* work,
                   int nt, int n1, int ncells, long long ns, cudaStream_t s, Skip skip,
                   double* partial = nullptr, double* vv = nullptr);
unsigned* counter_of(double* partial);
void precond_eblock_f32(double* out, const double* in, const float* B, int nt, int n1,
                        int ncells, long long ns, cudaStream_t s, Skip skip = {});

// ---- vector kernels (kernels_vec.cu) ----------------------------------------
// All reductions are deterministic: fixed grid for a given n, fixed-order
// block and final reductions (the only atomic is the completion counter that
// elects the finishing block; the sum order never depends on it).
// `partial` buffers hold kPartialDoubles doubles followed by one zeroed
// 32-bit completion counter.
constexpr long long kPartialDoubles = 148LL * 8 * 80;
int reduce_grid(long long n);
void vec_fill(double* x, double v, long long n, cudaStream_t s);
void vec_copy(double* y, const double* x, long long n, cudaStream_t s);
void vec_axpy(double* y, double a, const double* x, long long n, cudaStream_t s);
// y = a*x + b*y
void vec_axpby(double* y, double a, const double* x, double b, long long n, cudaStream_t s);
// U_j = u for j < nb (1 (x) u, stdg.hpp:131)
void vec_broadcast(double* U, const double* u, int nb, long long n, cudaStream_t s);
// y = z + x - q (x may alias y; 16-byte aligned vectors), honouring skip
void vec_poly_step(double* y, const double* z, const double* x, const double* q, long long n,
                   cudaStream_t s, Skip skip);
// out[j] = <V_j, w>, j < k <= 64 (V_j = V + j*ldv); partial buffer >= grid*k doubles
void vec_multidot(const double* V, long long ldv, int k, const double* w, long long n,
                  double* partial, double* out, cudaStream_t s, Skip skip = {});
// w = (w - sum_{j<k} h[j] V_j) * s (h on device), then out2[k] = <w,w> and,
// if want_dots, out2[j] = <V_j, w> (an extra pass); partial buffer >= grid*(k+1).  s = 1 unless
// scale_src = [h_0..h_{k-1}, <w,w>] is given: then s = 1/sqrt(<w,w> - sum h^2)
// (Pythagorean norm of the projected vector), written to scale_out[0].
// norm_only: w_new is reduced (its exact norm, the Givens step) but not stored.
// hn2 (optional, device) = ||V_j||^2 for basis vectors stored unnormalised:
// the coefficients become h_j / hn2[j] and sum h^2 becomes sum h_j^2 / hn2[j].
void vec_update_dot(double* w, const double* V, long long ldv, int k, const double* h,
                    long long n, int want_dots, double* partial, double* out2, cudaStream_t s,
                    const double* scale_src = nullptr, double* scale_out = nullptr,
                    const double* hn2 = nullptr, Skip skip = {}, GivensArgs gv = {},
                    bool norm_only = false);
// y = sign * x / sqrt(*nrm2)  (nrm2 on device)
void vec_scale_invsqrt(double* y, const double* x, const double* nrm2, long long n,
                       cudaStream_t s, double sign = 1.0);
// x = (accumulate ? x : 0) + sum_{j<k} y[j] V_j (y on device), k <= 64.
// bsrc != null: the old x is bsrc repeated with period bper doubles (n a
// multiple of bper) and is not read from x: x = 1 (x) bsrc + sum y_j V_j.
void vec_combine(double* x, const double* V, long long ldv, int k, const double* y, long long n,
                 cudaStream_t s, bool accumulate = true, const double* bsrc = nullptr,
                 long long bper = 1);
// Central-difference Jacobian action on the device, no host scalars:
// e = c * sqrt(1 + sqrt(*uu)) / sqrt(*vv) (uu null: e = c / sqrt(*vv); e = 1
// if <v,v> = 0).  fd_pm: Up = U + e v, Um = U - e v.  fd_diff: Jv = (Jv - Fm) / 2e.
void vec_fd_pm(double* Up, double* Um, const double* U, const double* v, long long n,
               const double* vv, const double* uu, double c, cudaStream_t s, Skip skip = {});
void vec_fd_diff(double* Jv, const double* Fm, long long n, const double* vv, const double* uu,
                 double c, cudaStream_t s, Skip skip = {});
// *out = max |x_i|
void vec_maxabs(const double* x, long long n, double* partial, double* out, cudaStream_t s);
// *out = <x,y>
void vec_dot(const double* x, const double* y, long long n, double* partial, double* out,
             cudaStream_t s, Skip skip = {});

}  // namespace stg
