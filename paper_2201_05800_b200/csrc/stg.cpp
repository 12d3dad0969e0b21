// Host side of the C ABI (include/stg_cuda.h): handle, constants, operator
// dispatch, device-resident GMRES(m), Newton and the STDG / LoDG steps.
// Control flow follows the reference drivers (stdg.hpp:120-143,
// lodg.hpp:89-149, newton.hpp:102-130); all vector work is on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/stg_cuda.h"
#include "constants.hpp"
#include "eig.hpp"
#include "hostcopy.hpp"
#include "kernels.hpp"

namespace {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// AdmissibilityError (models.hpp:15-20), rethrown per temporal node (stdg.hpp:41-50)
struct AdmissibilityError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// NonconvergenceError (newton.hpp:40-48).  The last iterate stays in the
// caller's U (Newton updates it in place); the residual history and the
// linear-iteration count travel with the exception into stg_solve_info.
struct NonconvergenceError : std::runtime_error {
  std::vector<double> history;
  int linear_iterations = 0;
  NonconvergenceError(const std::string& w, std::vector<double> h, int lin = 0)
      : std::runtime_error(w), history(std::move(h)), linear_iterations(lin) {}
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

thread_local std::string g_create_error;

std::string fmt_short(double v) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "%.6g", v);
  return buf;
}

struct DevBuf {
  double* p = nullptr;
  size_t n = 0;
  void ensure(size_t count) {
    if (count <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    ck(cudaMalloc(&p, count * sizeof(double)), "cudaMalloc");
    n = count;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

// page-locked host mirror of a caller's pageable buffer (hostcopy.hpp)
struct PinBuf {
  double* p = nullptr;
  size_t n = 0;
  void ensure(size_t count) {
    if (count <= n) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
    ck(cudaHostAlloc(reinterpret_cast<void**>(&p), count * sizeof(double), cudaHostAllocDefault),
       "cudaHostAlloc");
    n = count;
  }
  ~PinBuf() {
    if (p) cudaFreeHost(p);
  }
};

// whether the driver would have to stage copies from / to p itself
bool pageable(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeUnregistered;
}

long long round_up(long long v, long long m) { return (v + m - 1) / m * m; }

bool general_model(int m) { return m == STG_MODEL_ADVDIFF || m == STG_MODEL_EULER; }
bool linear_model(int m) { return m == STG_MODEL_ADVECTION || m == STG_MODEL_ADVDIFF; }

}  // namespace

struct stg_handle {
  stg_desc desc{};
  stg::Geometry g{};
  int n1 = 0, nt = 0;
  long long n_sdof = 0, n_dof = 0;
  stg::SpatialCoef sp{};
  stg::GenCoef gc{};   // general flux models (advdiff / euler)
  int r = 1;           // components per node
  stg::LglRule rule, trule;
  std::vector<double> D, Dt;  // row-major D(j,i) at [j*n+i]
  stg::Tableau tab;
  std::vector<double> Ainv;
  cudaStream_t stream = nullptr;
  int kernel_pref = STG_KERNEL_AUTO;
  std::string err;
  long long launches = 0;
  long long reorth = 0;  // Arnoldi steps that needed a second Gram-Schmidt pass

  // workspace
  DevBuf small;    // device scalars / Hessenberg columns
  DevBuf partial;  // reduction partials
  DevBuf basis, wv, rv, res, res2, delta, tmp1, tmp2, Ustage, host_U, host_R, host_u, host_u2;
  DevBuf ptab;          // preconditioner block tables
  int ptab_kind = -1;   // TBLOCK / JACOBI table in ptab and its mix (-1: none)
  stg::MixCoef ptab_mix{};
  DevBuf zbasis;        // flexible GMRES: preconditioned basis Z_k = P^-1 S_k
  DevBuf genF, genFlag;  // general models: F(X_j) blocks; admissibility flag (int)
  DevBuf small_out;      // fused small-solve result record
  DevBuf march;          // integrate: ping-pong states
  // general linear models: element-local Jacobians K_e (probed once) and the
  // inverted element blocks for the last mix
  DevBuf gK, gProbe, gBinv;
  bool gK_valid = false, gB_valid = false;
  stg::MixCoef g_mix{};
  // Burgers element blocks: built at the first Newton iteration of a step and
  // reused for the rest of it (a lagged preconditioner; STG_PRECOND_REBUILD=1
  // rebuilds every iteration)
  bool eblock_valid = false;
  bool eblock_sweep = false;  // ... with the sweep's inflow couplings in sweepG
  // ... and across steps: the blocks of step n serve steps n+1.. while the mix
  // (dt) is the same, up to STG_PRECOND_LAG_STEPS steps (new_step())
  int eblock_age = 0;
  stg::MixCoef eblock_mix{};
  // set by the build, read by newton(): whether the blocks the current
  // Jacobian uses were built for it (else they are lagged), and the GMRES
  // count of the first solve after the build (lagged blocks that need clearly
  // more are rebuilt)
  bool eblock_built_now = false, eblock_in_use = false;
  int eblock_fresh_its = 0;
  DevBuf sweepG, sweepW;      // d = 1 upwind sweep: couplings (fp32), y = B^-1 r
  DevBuf polyZ, polyW, polyQ;  // polynomial preconditioner: P0^-1 r, J y, P0^-1 J y
  bool block_exact = false;    // the last make_precond built an exact element-block inverse
  // the vector whose <v, v> small[kVVSlot] holds (set by the preconditioner
  // that wrote it, consumed by the next FD Jacobian action; reset per call)
  const double* vv_of = nullptr;
  // d = 2 dense element block: the uploaded inverse and the mix it belongs to
  DevBuf etab;  // d = 1 advection element block (shared), keyed by mix
  stg::MixCoef etab_mix{};
  bool etab_valid = false;
  DevBuf dtab;  // d = 2 dense block (fallback of the d = 2 FDM)
  stg::MixCoef dense_mix{};
  bool dense_valid = false;
  DevBuf fdm2M;  // device copy of the fdm2_kernel factors (stg::FdmCoef2)
  std::unique_ptr<stg::FdmCoef2> fdm2_host;
  stg::MixCoef fdm2_mix{};
  bool fdm2_valid = false;
  int fdm2_nr = 0, fdm2_np = 0;
  DevBuf fdm2iM;  // in-place d = 2 FDM (fdm2i_kernel)
  std::unique_ptr<stg::FdmCoef2i> fdm2i_host;
  stg::MixCoef fdm2i_mix{};
  bool fdm2i_valid = false;
  // d = 3 fast-diagonalisation factors and the mix they belong to
  stg::FdmCoef fdm{};
  stg::MixCoef fdm_mix{};
  bool fdm_valid = false;
  stg::MixCoef fdm3_mix{};
  bool fdm3_valid = false;
  DevBuf fdm3M;  // device copy of the fdm3_kernel factors (stg::FdmCoef3)
  std::unique_ptr<stg::FdmCoef3> fdm3_host;  // and the host copy (kernel parameters)
  double* pinned = nullptr;  // pinned host mirror of `small`
  static constexpr int kSmall = 1024;
  // GMRES cycle state on the device, its pinned host copy, the host-mapped
  // [status, k_done] word pair the Givens step publishes, and the skip flag
  // the operator / preconditioner launchers attach to their kernels while an
  // Arnoldi step is being enqueued speculatively
  DevBuf gstate;
  stg::GmresDev* gpin = nullptr;
  int* mapped = nullptr;
  cudaEvent_t ev_step[2] = {}, ev_re = nullptr;
  stg::Skip skip{};
  // Euler admissibility: a flag may be set on the device (pending) and the
  // check is deferred while a Newton solve runs (apply_general)
  bool adm_pending = false, adm_defer = false;
  // fused residual reductions (fast 3-D kernel): requested by newton() for
  // its residual applies; red_done: the last apply produced them
  bool red = false, red_done = false;
  // pipelined host-buffer path: copy-in / copy-out streams and chunk events
  static constexpr int kChunks = 8;
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev_start = nullptr, ev_in[kChunks] = {}, ev_c[kChunks] = {};
  // Lazy initial guess of a slab / stage solve: lazy_dst (the solve's U) is
  // notionally 1 (x) lazy_src but has not been written; the fast 3-D kernel
  // reads lazy_src through zero-stride tensor maps and the first Newton
  // update writes U = 1 (x) lazy_src + correction.  materialise() writes it
  // out for any other reader.
  const double* lazy_src = nullptr;
  double* lazy_dst = nullptr;
  // GMRES speculation: the iteration count of the last converged solve, per
  // Newton-iteration index of the enclosing newton() call (slot 0 outside
  // one); the driver does not enqueue a speculative Arnoldi step past it
  static constexpr int kPredSlots = 8;
  int gmres_pred[kPredSlots] = {};
  int pred_slot = 0;
  // pageable callers: page-locked mirrors and the events of their D2H chunks
  PinBuf pin_U, pin_R, pin_u, pin_u2;
  std::vector<cudaEvent_t> ev_stage;

  ~stg_handle() {
    for (cudaEvent_t e : ev_stage) cudaEventDestroy(e);
    if (pinned) cudaFreeHost(pinned);
    if (gpin) cudaFreeHost(gpin);
    if (mapped) cudaFreeHost(mapped);
    for (cudaEvent_t e : ev_step)
      if (e) cudaEventDestroy(e);
    if (ev_re) cudaEventDestroy(ev_re);
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
    if (ev_start) cudaEventDestroy(ev_start);
    for (int k = 0; k < kChunks; ++k) {
      if (ev_in[k]) cudaEventDestroy(ev_in[k]);
      if (ev_c[k]) cudaEventDestroy(ev_c[k]);
    }
  }
};

namespace {

using Op = std::function<void(const double* x, double* y)>;

void check_launch(stg_handle* h) {
  ck(cudaGetLastError(), "kernel launch");
}

// ---- operator dispatch ----------------------------------------------------
// slots of `small` for the fused residual reductions (clear of the GMRES
// step data; kRedSsSlot is where the deferred first GMRES cycle reads <b,b>)
constexpr int kRedMaxSlot = 1010;
constexpr int kRedSsSlot = 200;
constexpr int kVVSlot = 1000;  // <v, v> of the FD Jacobian action's direction
// Euler's admissibility flag (1 + first failing temporal block, set by the
// rhs kernel) is raised as AdmissibilityError naming the temporal node
// (stdg.hpp:41-50).  Outside a solve every apply checks it (one sync); inside
// newton() the check is deferred to the Newton step's own sync points, so no
// Arnoldi step waits on the host (the step that went nonphysical still throws,
// a few kernels later).
void check_admissibility(stg_handle* h) {
  if (!h->adm_pending) return;
  h->adm_pending = false;
  int* hp = reinterpret_cast<int*>(h->pinned + 1000);
  int* flag = reinterpret_cast<int*>(h->genFlag.p);
  ck(cudaMemcpyAsync(hp, flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream), "memcpy");
  ck(cudaStreamSynchronize(h->stream), "sync");
  if (*hp != 0) {
    const int node = *hp - 1;
    ck(cudaMemsetAsync(flag, 0, sizeof(int), h->stream), "memset");
    throw AdmissibilityError("temporal node " + std::to_string(node) +
                             ": euler_model: nonphysical state");
  }
}

// while in scope, admissibility checks wait for check_admissibility()
struct AdmDefer {
  stg_handle* h;
  bool prev;
  explicit AdmDefer(stg_handle* hh) : h(hh), prev(hh->adm_defer) { h->adm_defer = true; }
  ~AdmDefer() { h->adm_defer = prev; }
};

// General flux models: F(X_j) for every input block, then the mix.
void apply_general(stg_handle* h, const stg::MixCoef& mx, int n_in, int n_out, const double* X,
                   const double* W, double* R) {
  if (h->kernel_pref == STG_KERNEL_FAST)
    throw std::invalid_argument("fast kernel requested but not applicable to this problem");
  stg::GenArgs a{};
  a.c = h->gc;
  a.g = h->g;
  a.mx = mx;
  a.n_in = n_in;
  a.n_out = n_out;
  a.X = X;
  a.Xmix = X;
  a.W = W;
  h->genF.ensure(size_t(n_in) * size_t(h->n_sdof));
  a.F = h->genF.p;
  a.R = R;
  a.err = reinterpret_cast<int*>(h->genFlag.p);
  a.skip = h->skip;
  const int launched = stg::launch_general(a, h->stream);
  if (launched < 0) throw std::invalid_argument("no kernel for this (dim, degree, model)");
  h->launches += launched;
  check_launch(h);
  if (h->desc.model == STG_MODEL_EULER) {
    h->adm_pending = true;
    if (!h->adm_defer) check_admissibility(h);
  }
}

// write the lazy initial guess out (no-op when there is none)
void materialise(stg_handle* h) {
  if (!h->lazy_src) return;
  stg::vec_broadcast(h->lazy_dst, h->lazy_src, h->nt, h->n_sdof, h->stream);
  h->launches++;
  h->lazy_src = nullptr;
}

void apply(stg_handle* h, const stg::MixCoef& mx, int n_in, int n_out, const double* X,
           const double* U, const double* W, double* R, bool jvp, bool full_s,
           int seg_begin = 0, int seg_end = 0) {
  h->red_done = false;
  stg::SlabArgs a{};
  // the lazy initial guess as X: the fast 3-D kernel and the d = 2 plane
  // kernel read the one block it stands for; every other reader needs it in
  // memory
  bool lazy_x = false;
  if (h->lazy_src && (X == h->lazy_dst || U == h->lazy_dst || W == h->lazy_dst)) {
    lazy_x = X == h->lazy_dst && U != h->lazy_dst && W != h->lazy_dst && !jvp &&
             n_in == h->nt && seg_end == 0 && !general_model(h->desc.model);
    if (!lazy_x) materialise(h);
  }
  a.seg_begin = seg_begin;
  a.seg_end = seg_end;
  a.sp = h->sp;
  a.mx = mx;
  a.g = h->g;
  a.n_in = n_in;
  a.n_out = n_out;
  a.has_w = W != nullptr;
  a.jvp = jvp ? 1 : 0;
  a.full_s = full_s ? 1 : 0;
  a.model = h->desc.model;
  a.X = lazy_x ? h->lazy_src : X;
  a.x_bcast = lazy_x ? 1 : 0;
  a.U = U;
  a.W = W;
  a.R = R;
  a.skip = h->skip;
  if (h->red) {  // max |R| and <R,R> from the apply itself (fast 3-D kernel)
    a.red_max = reinterpret_cast<unsigned long long*>(h->small.p + kRedMaxSlot);
    a.red_ss = h->small.p + kRedSsSlot;
    a.red_part = h->partial.p;
  }
  if (general_model(h->desc.model)) {
    apply_general(h, mx, n_in, n_out, X, W, R);
    return;
  }
  int launched = -1;
  auto launch = [&] {
    if (h->kernel_pref != STG_KERNEL_GENERIC && stg::slab_fast_supported(a)) {
      launched = stg::launch_slab_fast(a, h->stream);
      if (launched >= 0) h->red_done = h->red && stg::slab_fast_reduces(a);
    } else if (h->kernel_pref == STG_KERNEL_FAST) {
      throw std::invalid_argument("fast kernel requested but not applicable to this problem");
    }
    if (launched < 0) {
      launched = stg::launch_slab_generic(a, h->stream);
      h->red_done = h->red && launched >= 0 && stg::slab_generic_reduces(a);
    }
  };
  launch();
  if (launched < 0 && a.x_bcast) {  // no kernel reads the one-block X here: write it out
    materialise(h);
    a.X = X;
    a.x_bcast = 0;
    launch();
  }
  if (launched < 0) throw std::invalid_argument("no kernel for this (dim, degree, model)");
  h->launches += launched;
  check_launch(h);
}

stg::MixCoef zero_mix() {
  stg::MixCoef m;
  std::memset(&m, 0, sizeof m);
  return m;
}

// st_residual (stdg.hpp:56-76): T = e e^T - D^T M, S = -(dt/2) M, c = -e_1.
stg::MixCoef st_mix(const stg_handle* h, double dt, bool with_un) {
  stg::MixCoef m = zero_mix();
  const int n = h->nt;
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      double v = -(h->Dt[size_t(j) * n + i] * h->trule.w[j]);
      if (i == n - 1 && j == n - 1) v += 1.0;
      m.T[i][j] = v;
    }
    m.S[i][i] = -(0.5 * dt * h->trule.w[i]);
  }
  if (with_un) m.c[0] = -1.0;
  return m;
}

// rk_step residual (lodg.hpp:104-122)
stg::MixCoef stage_mix(const stg_handle* h, int form, double dt, bool with_u) {
  stg::MixCoef m = zero_mix();
  const int s = h->nt;
  if (form == STG_FORM_A) {
    for (int i = 0; i < s; ++i) {
      m.T[i][i] = 1.0;
      for (int j = 0; j < s; ++j) m.S[i][j] = -(dt * h->tab.A[size_t(i) * s + j]);
      if (with_u) m.c[i] = -1.0;
    }
  } else {
    for (int i = 0; i < s; ++i) {
      double rs = 0.0;
      for (int j = 0; j < s; ++j) {
        m.T[i][j] = h->Ainv[size_t(i) * s + j] / dt;
        rs += m.T[i][j];
      }
      m.S[i][i] = -1.0;
      if (with_u) m.c[i] = -rs;
    }
  }
  return m;
}

void validate_desc(const stg_desc* d) {
  if (!d) throw std::invalid_argument("stg_create: null descriptor");
  if (d->dim < 1 || d->dim > 3) throw std::invalid_argument("uniform_mesh: d in {1,2,3}");
  if (d->degree < 1 || d->degree + 1 > stg::kMaxN)
    throw std::invalid_argument("dg_space: degree must be in [1, 5]");
  if (d->n_tau < 2 || d->n_tau > stg::kMaxT)
    throw std::invalid_argument("sbp_operators: n_tau must be in [2, 6]");
  if (d->model < STG_MODEL_ADVECTION || d->model > STG_MODEL_EULER)
    throw std::invalid_argument("unknown model");
  if (d->model == STG_MODEL_BURGERS && d->dim != 1)
    throw std::invalid_argument("burgers model: d = 1 only");
  if (d->model == STG_MODEL_ADVDIFF) {  // advdiff_model (models.hpp:68-76)
    if (d->dim > 2) throw std::invalid_argument("advdiff_model: d in {1, 2}");
    if (!(d->eps >= 0.0)) throw std::invalid_argument("advdiff_model: need eps >= 0");
    if (d->velocity_field != STG_FIELD_CONSTANT && d->velocity_field != STG_FIELD_ROTATING)
      throw std::invalid_argument("advdiff_model: unknown velocity field");
    if (d->velocity_field == STG_FIELD_ROTATING && d->dim != 2)
      throw std::invalid_argument("rotating_field: d = 2");
  }
  if (d->model == STG_MODEL_EULER) {  // euler_model (models.hpp:118-124)
    if (d->dim != 2) throw std::invalid_argument("assemble_semidiscrete: dimension mismatch");
    if (d->gamma > 0.0 && !(d->gamma > 1.0)) throw std::invalid_argument("euler_model: gamma > 1");
  }
  if (d->dim == 3 && d->degree + 1 > 5)
    throw std::invalid_argument("d = 3 supports degree <= 4");
  long long cells = 1;
  for (int a = 0; a < d->dim; ++a) {
    if (d->cells[a] < 1) throw std::invalid_argument("uniform_mesh: need cells >= 1");
    if (!(d->upper[a] > d->lower[a]))
      throw std::invalid_argument("uniform_mesh: need upper > lower");
    cells *= d->cells[a];
  }
  if (cells > (1LL << 30)) throw std::invalid_argument("too many cells");
  long long npc = 1;
  for (int a = 0; a < d->dim; ++a) npc *= d->degree + 1;
  if (d->model == STG_MODEL_EULER) npc *= 4;
  if (cells * npc >= (1LL << 31))
    throw std::invalid_argument("mesh too large: n_sdof must stay below 2^31");
}

void build_constants(stg_handle* h) {
  const stg_desc& d = h->desc;
  h->n1 = d.degree + 1;
  h->nt = d.n_tau;
  h->rule = stg::lgl(h->n1);
  h->D = stg::diff_matrix(h->rule);
  h->trule = stg::lgl(h->nt);
  h->Dt = stg::diff_matrix(h->trule);
  h->tab = stg::lobatto(h->nt);
  h->Ainv = stg::inverse(h->tab.A, h->nt);

  stg::Geometry& g = h->g;
  g.dim = d.dim;
  g.n1 = h->n1;
  g.npc = 1;
  for (int a = 0; a < d.dim; ++a) g.npc *= h->n1;
  g.nx = d.cells[0];
  g.ny = d.dim >= 2 ? d.cells[1] : 1;
  g.nz = d.dim >= 3 ? d.cells[2] : 1;
  g.n_cells = g.nx * g.ny * g.nz;
  h->r = d.model == STG_MODEL_EULER ? 4 : 1;
  g.n_sdof = (long long)g.n_cells * g.npc * h->r;
  h->n_sdof = g.n_sdof;
  h->n_dof = g.n_sdof * h->nt;

  stg::SpatialCoef& sp = h->sp;
  std::memset(&sp, 0, sizeof sp);
  const int n = h->n1;
  const auto& w = h->rule.w;
  for (int a = 0; a < d.dim; ++a) {
    const double hsp = (d.upper[a] - d.lower[a]) / double(d.cells[a]);
    const double s = 2.0 / hsp;
    if (d.model == STG_MODEL_ADVECTION) {
      const double b = d.velocity[a];
      const double alpha = 0.5 * (b + std::abs(b)), beta = 0.5 * (b - std::abs(b));
      for (int i = 0; i < n; ++i)
        for (int k = 0; k < n; ++k)
          sp.V[a][i][k] = s * b * (w[k] * h->D[size_t(k) * n + i]) / w[i];
      sp.V[a][n - 1][n - 1] += -(s / w[n - 1]) * alpha;
      sp.V[a][0][0] += (s / w[0]) * beta;
      sp.cL[a] = (s / w[0]) * alpha;
      sp.cR[a] = -(s / w[n - 1]) * beta;
    }
    if (a == 0) {
      sp.sc = s;
      sp.inv_w0 = 1.0 / w[0];
      sp.inv_wN = 1.0 / w[n - 1];
      for (int i = 0; i < n; ++i)
        for (int k = 0; k < n; ++k) sp.Dm[i][k] = h->D[size_t(i) * n + k];
    }
  }
  if (general_model(d.model)) {
    stg::GenCoef& c = h->gc;
    std::memset(&c, 0, sizeof c);
    c.r = h->r;
    c.field = d.velocity_field;
    c.b[0] = d.velocity[0];
    c.b[1] = d.velocity[1];
    c.eps = d.model == STG_MODEL_ADVDIFF ? d.eps : 0.0;
    c.eta = d.eta > 0.0 ? d.eta : 10.0 * d.degree * d.degree;  // spatial.hpp:366
    c.gamma = d.gamma > 0.0 ? d.gamma : 1.4;
    double hprod = 1.0;
    for (int a = 0; a < d.dim; ++a) {
      c.h[a] = (d.upper[a] - d.lower[a]) / double(d.cells[a]);
      c.lower[a] = d.lower[a];
      hprod *= c.h[a];
    }
    c.vol_scale = hprod / std::pow(2.0, d.dim);
    for (int i = 0; i < n; ++i) {
      c.xi[i] = h->rule.x[size_t(i)];
      c.w[i] = w[size_t(i)];
      for (int k = 0; k < n; ++k) c.D[i][k] = h->D[size_t(i) * n + k];
    }
  }
}

void ensure_workspace(stg_handle* h) {
  if (!h->pinned) {
    ck(cudaMallocHost(&h->pinned, sizeof(double) * stg_handle::kSmall), "cudaMallocHost");
    h->small.ensure(stg_handle::kSmall);
    // reduction partials + the zeroed completion counter (kernels.hpp)
    h->partial.ensure(size_t(stg::kPartialDoubles) + 1);
    ck(cudaMemset(h->partial.p, 0, sizeof(double) * (size_t(stg::kPartialDoubles) + 1)),
       "cudaMemset");
  }
}

// ---- device reductions returning to the host --------------------------------
// Slot of `small` / `pinned` for these scalars: clear of the GMRES step data
// ([0, 320): dots, norms, scales, y), which an operator that reduces (the FD
// Jacobian action) must not overwrite while a step is in flight.
constexpr int kScalarSlot = 960;
double dev_maxabs(stg_handle* h, const double* x, long long n) {
  stg::vec_maxabs(x, n, h->partial.p, h->small.p + kScalarSlot, h->stream);
  h->launches += 1;  // fused last-block reduction
  ck(cudaMemcpyAsync(h->pinned + kScalarSlot, h->small.p + kScalarSlot, sizeof(double),
                     cudaMemcpyDeviceToHost, h->stream), "memcpy");
  ck(cudaStreamSynchronize(h->stream), "sync");
  return h->pinned[kScalarSlot];
}

double dev_dot(stg_handle* h, const double* x, const double* y, long long n) {
  stg::vec_dot(x, y, n, h->partial.p, h->small.p + kScalarSlot, h->stream);
  h->launches += 1;
  ck(cudaMemcpyAsync(h->pinned + kScalarSlot, h->small.p + kScalarSlot, sizeof(double),
                     cudaMemcpyDeviceToHost, h->stream), "memcpy");
  ck(cudaStreamSynchronize(h->stream), "sync");
  return h->pinned[kScalarSlot];
}

// attaches a skip flag to every kernel the operator / preconditioner
// launchers enqueue while in scope
struct SkipScope {
  stg_handle* h;
  SkipScope(stg_handle* hh, stg::Skip s) : h(hh) { h->skip = s; }
  ~SkipScope() { h->skip = stg::Skip{}; }
};

struct GmresStats {
  int iterations = 0;
  double rel_residual = 0.0;
  bool converged = false;
  bool added = false;  // the solution was added into add_to instead of written to x
  bool aborted = false;  // early_stop() said the solve is not needed: x / add_to untouched
};

// Restarted GMRES(m), right-preconditioned (A P^-1 y = b, x = P^-1 y; P null:
// unpreconditioned), classical Gram-Schmidt in two fused passes per Arnoldi
// step (multidot incl. <w,w>; project + Pythagorean normalise) with a second
// pass only on heavy cancellation (DGKS-style).  Stopping test
// ||b - A x||_2 <= tol ||b||_2 (Eigen's criterion at newton.hpp:68-77) on the
// Arnoldi residual estimate, which with right preconditioning is the
// unpreconditioned residual; the true residual is recomputed at each restart.
// x holds the initial guess (x_zero: known 0).
//
// The Hessenberg column, the Givens rotations and the stopping test of each
// step run on the device (the last block of the update pass, kernels_vec.cu
// gmres_givens), so the host never waits inside a step: it enqueues step k+1
// before reading step k's outcome (lag 1).  Every kernel of a step carries a
// skip flag (the cycle status), so the speculative step is a string of empty
// launches once step k has converged or broken down, or needs a second
// Gram-Schmidt pass -- which the host then enqueues before re-enqueueing step
// k+1.  lag 0 (pipelined = false, or STG_GMRES_SYNC=1) waits after every step.
// The speculation stops at the iteration count the previous solve in the same
// position (the same Newton-iteration index) converged at: slab after slab
// the counts repeat, so the step that would only be a row of empty launches
// (2-4 us each: 11 of them per c4 step) is not enqueued; a solve that needs
// more pays one host round trip there and speculates on
// (STG_GMRES_NO_PREDICT=1: always speculate).
GmresStats gmres(stg_handle* h, const Op& A, const double* b, double* x, long long n, int m,
                 double tol, int max_it, const Op* P = nullptr, bool x_zero = false,
                 bool pipelined = true, double b_sign = 1.0, bool want_rel = true,
                 bool bb_ready = false, double* add_to = nullptr,
                 const std::function<bool()>* early_stop = nullptr) {
  ensure_workspace(h);
  if (m < 1) throw std::invalid_argument("gmres: restart >= 1");
  if (m > stg::kGmresMaxRestart) throw std::invalid_argument("gmres: restart <= 60");
  GmresStats st;
  const long long ld = round_up(n, 32);
  h->basis.ensure(size_t(ld) * (m + 1));
  h->wv.ensure(size_t(n));
  // flexible GMRES: Z_k = P^-1 S_k is kept, x += sum y_j c_j Z_j (no final
  // preconditioner apply, and P need not be the same linear map every step)
  if (P) h->zbasis.ensure(size_t(ld) * m);
  double* Z = P ? h->zbasis.p : nullptr;
  if (!h->gpin) {
    h->gstate.ensure((sizeof(stg::GmresDev) + 7) / 8);
    ck(cudaMallocHost(&h->gpin, sizeof(stg::GmresDev)), "cudaMallocHost");
    ck(cudaHostAlloc(&h->mapped, (stg::kGmresMaxRestart + 2) * sizeof(int), cudaHostAllocMapped),
       "cudaHostAlloc");
    for (cudaEvent_t& e : h->ev_step)
      ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&h->ev_re, cudaEventDisableTiming), "event");
  }
  stg::GmresDev* G = reinterpret_cast<stg::GmresDev*>(h->gstate.p);
  int* mapped_dev = nullptr;
  ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&mapped_dev), h->mapped, 0),
     "cudaHostGetDevicePointer");
  volatile int* mapped = h->mapped;
  double* V = h->basis.p;
  double* w = h->wv.p;
  double* dsm = h->small.p;  // [0..m+1] raw dots, [64..] ||S_j||^2, [128..] 2nd-pass dots,
                             // [190] / [191] pass scales, [200] <b,b> / <r,r>, [256..] y
  double* hp = h->pinned;
  cudaStream_t s = h->stream;
  static const bool force_sync = std::getenv("STG_GMRES_SYNC") != nullptr;
  const int lag = (pipelined && !force_sync) ? 1 : 0;
  // re-orthogonalise when ||w - V h||^2 <= reorth_tol ||w||^2 (orthogonality
  // loss of the single pass ~ eps * sqrt(1 / reorth_tol) = 2e-12 at 1e-8)
  static const double reorth_tol = [] {
    const char* e = std::getenv("STG_GMRES_REORTH_TOL");
    return e ? std::atof(e) : 1e-8;
  }();

  // The right-hand side is b_sign * b.  From x = 0 with tol < 1, ||b|| stays
  // on the device for the first cycle (S_0 = b / ||b|| and the stopping
  // threshold are formed there): no host round trip before the first step.
  // Otherwise it is read back here.
  const bool defer = x_zero && tol < 1.0;
  double bnorm = -1.0;  // < 0: not known on the host yet
  if (defer) {
    if (!bb_ready) {  // else the residual kernel left <b,b> in dsm[200] (kRedSsSlot)
      stg::vec_dot(b, b, n, h->partial.p, dsm + 200, s);
      h->launches++;
    }
  } else {
    const double bb = dev_dot(h, b, b, n);  // leaves <b,b> in small[kScalarSlot]
    bnorm = std::sqrt(bb);
    ck(cudaMemcpyAsync(h->small.p + 200, h->small.p + kScalarSlot, sizeof(double),
                       cudaMemcpyDeviceToDevice, h->stream), "memcpy");
    if (!std::isfinite(bnorm)) {  // NaN / inf right-hand side: not converged
      st.rel_residual = bnorm;
      return st;
    }
    if (bnorm == 0.0) {
      stg::vec_fill(x, 0.0, n, s);
      h->launches++;
      st.converged = true;
      return st;
    }
  }
  const stg::Skip run0{&G->status, 0}, run_re{&G->status, 3};
  static const bool no_predict = std::getenv("STG_GMRES_NO_PREDICT") != nullptr;
  const int pred = no_predict ? 0 : h->gmres_pred[h->pred_slot];  // 0: none yet
  std::vector<char> norm_only(size_t(m) + 1, 0);
  int total = 0;
  // Arnoldi step k: S_{k+1} <- A P^-1 S_k, then the two fused passes; the
  // update pass's last block runs the Givens step and publishes the status
  auto enqueue_step = [&](int k) {
    double* vn = V + size_t(k + 1) * ld;
    {
      SkipScope scope(h, run0);
      if (P) {
        double* zk = Z + size_t(k) * ld;
        (*P)(V + size_t(k) * ld, zk);  // Z_k = P^-1 S_k
        A(zk, vn);
      } else {
        A(V + size_t(k) * ld, vn);
      }
    }
    const int kk = k + 1;  // vectors S_0..S_k
    stg::GivensArgs gv;
    gv.G = G;
    gv.k = k;
    gv.pass = 0;
    gv.d1 = dsm;
    gv.host = mapped_dev;
    gv.ysol = want_rel ? nullptr : dsm + 256;
    stg::vec_multidot(V, ld, kk + 1, vn, n, h->partial.p, dsm, s, run0);  // [d_0..d_k, <w,w>]
    // the step the previous solve converged at: reduce the new vector's norm
    // (the convergence decision) without storing it; store_step() writes it
    // if the solve goes on after all
    norm_only[k] = !no_predict && pred > 0 && total + k + 1 == pred;
    stg::vec_update_dot(vn, V, ld, kk, dsm, n, 0, h->partial.p, dsm + 64, s, dsm, dsm + 190,
                        dsm + 64, run0, gv, norm_only[k]);
    h->launches += 2;
    ck(cudaEventRecord(h->ev_step[k & 1], s), "event");
  };
  // the projected, scaled S_{k+1} of a norm-only step, written after the fact
  // (same dots, same scale; no reduction and no Givens step)
  auto store_step = [&](int k) {
    double* vn = V + size_t(k + 1) * ld;
    stg::vec_update_dot(vn, V, ld, k + 1, dsm, n, 0, nullptr, dsm + 64, s, dsm, dsm + 190,
                        dsm + 64, stg::Skip{}, stg::GivensArgs{});
    h->launches++;
    norm_only[k] = false;
  };
  // second classical pass on S_{k+1}: [g2, <S,S>] = [V, S]^T S, then
  // S' = (S - sum g2_j / ||S_j||^2 S_j) * Pythagorean scale; runs only while
  // the status says "re-orthogonalise" (3)
  auto enqueue_reorth = [&](int k) {
    double* vn = V + size_t(k + 1) * ld;
    const int kk = k + 1;
    stg::GivensArgs gv;
    gv.G = G;
    gv.k = k;
    gv.pass = 1;
    gv.d1 = dsm;
    gv.sc1 = dsm + 190;
    gv.host = mapped_dev;
    gv.ysol = want_rel ? nullptr : dsm + 256;
    stg::vec_multidot(V, ld, kk + 1, vn, n, h->partial.p, dsm + 128, s, run_re);
    stg::vec_update_dot(vn, V, ld, kk, dsm + 128, n, 0, h->partial.p, dsm + 64, s, dsm + 128,
                        dsm + 191, dsm + 64, run_re, gv);
    h->launches += 2;
    ck(cudaEventRecord(h->ev_re, s), "event");
  };

  std::vector<double> y(static_cast<size_t>(m), 0.0);
  bool first = true;
  bool x_set = !x_zero;  // x_zero: x is written (not accumulated) by the first update
  // b may be the basis' first slot itself (Newton writes its residual there):
  // then the first cycle from x = 0 keeps S_0 = b unnormalised (no scaling
  // pass), and a restart first moves b out of the slot it would overwrite
  bool s0_is_b = false;
  while (true) {
    double beta = -1.0;  // < 0: on the device only (deferred first cycle)
    s0_is_b = false;
    if (first && x_zero) {  // x = 0: r = b and ||r|| = ||b|| (no operator apply, no sync)
      if (b == V) {
        s0_is_b = true;
      } else {
        stg::vec_scale_invsqrt(V, b, dsm + 200, n, s, b_sign);  // S_0 = b / ||b|| (dsm[200] = <b,b>)
        h->launches++;
      }
      if (!defer) beta = bnorm;
    } else {
      if (b == V) {  // keep b for this and later restarts
        h->res2.ensure(size_t(n));
        stg::vec_copy(h->res2.p, b, n, s);
        h->launches++;
        b = h->res2.p;
      }
      A(x, w);                                   // w = A x
      stg::vec_axpby(w, b_sign, b, -1.0, n, s);  // w = b - A x
      h->launches++;
      stg::vec_multidot(w, 0, 1, w, n, h->partial.p, dsm + 200, s);
      h->launches += 1;
      ck(cudaMemcpyAsync(hp + 200, dsm + 200, sizeof(double), cudaMemcpyDeviceToHost, s),
         "memcpy");
      stg::vec_scale_invsqrt(V, w, dsm + 200, n, s);  // S_0 = r / ||r||
      h->launches++;
      ck(cudaStreamSynchronize(s), "sync");
      beta = std::sqrt(hp[200]);
    }
    first = false;
    if (beta >= 0.0) {
      st.rel_residual = beta / bnorm;
      if (st.rel_residual <= tol) {
        st.converged = true;
        break;
      }
    }
    if (total >= max_it) break;
    for (int j = 0; j <= m; ++j) mapped[j] = -1;  // per-step status slots
    const double s0 = s0_is_b ? b_sign : 0.0;
    if (beta >= 0.0)
      stg::gmres_init(G, m, nullptr, beta, tol * bnorm, reorth_tol, dsm + 64, mapped_dev, s, s0);
    else
      stg::gmres_init(G, m, dsm + 200, 0.0, tol, reorth_tol, dsm + 64, mapped_dev, s, s0);
    h->launches++;
    auto can_enqueue = [&](int j) { return j < m && total + j < max_it; };
    int k = 0, enq = 0, status = 0;
    // a speculative step (e > k) that would be iteration pred + 1 waits for
    // step pred's outcome
    auto worth = [&](int e) { return e <= k || total + e != pred; };
    while (true) {
      while (enq <= k + lag && can_enqueue(enq) && worth(enq)) {  // step k and, speculatively, k + lag
        enqueue_step(enq);
        ++enq;
      }
      if (k >= enq) break;  // end of the cycle (restart length or max_it)
      ck(cudaEventSynchronize(h->ev_step[k & 1]), "sync");  // step k done
      // the caller's deferred check (newton: the residual norm it enqueued the
      // read-back of before this solve has arrived with this first wait): the
      // solve may turn out not to be needed; nothing has touched x or add_to
      if (early_stop && total == 0 && k == 0) {
        const bool stop = (*early_stop)();
        early_stop = nullptr;
        if (stop) {
          st.aborted = true;
          ck(cudaStreamSynchronize(s), "sync");  // drain the speculative launches
          return st;
        }
      }
      status = mapped[k];
      if (status == 4) break;  // b = 0 (deferred norm): no step ran
      if (status == 5) {       // ||r|| NaN / inf: no step ran, the solve failed
        st.iterations = total;
        st.rel_residual = std::numeric_limits<double>::quiet_NaN();
        return st;
      }
      if (norm_only[k] && (status == 0 || status == 3)) store_step(k);  // the solve goes on
      if (status == 3) {  // step k needs a second Gram-Schmidt pass
        enqueue_reorth(k);
        h->reorth++;
        ck(cudaEventSynchronize(h->ev_re), "sync");
        status = mapped[k];
        if (status == 0) enq = k + 1;  // a speculative step k+1 was skipped: enqueue it again
      }
      if (status < 0 || status > 2) throw std::runtime_error("gmres: Arnoldi step status lost");
      ++k;
      if (status != 0) break;  // converged (1) or breakdown (2) at step k - 1
    }
    // stream order: any speculative launches after step k - 1 are no-ops
    total += k;
    if (status == 1 && !want_rel) {
      // converged and the caller does not read the residual estimate: the
      // back substitution and the update run on the device, no round trip.
      // add_to (first cycle from x = 0): the solution goes straight into the
      // caller's vector (Newton's u += du without du)
      // (a step that converged within kInlineBacksub columns left the
      // coefficients in dsm + 256 itself)
      if (k > stg::kInlineBacksub) {
        stg::gmres_backsub(G, k, dsm + 256, s);
        h->launches++;
      }
      if (add_to && !x_set) {
        if (h->lazy_src && add_to == h->lazy_dst) {  // u = 1 (x) lazy_src + correction
          stg::vec_combine(add_to, P ? Z : V, ld, k, dsm + 256, n, s, true, h->lazy_src,
                           h->n_sdof);
          h->lazy_src = nullptr;
        } else {
          stg::vec_combine(add_to, P ? Z : V, ld, k, dsm + 256, n, s, true);
        }
        st.added = true;
      } else {
        stg::vec_combine(x, P ? Z : V, ld, k, dsm + 256, n, s, x_set);
      }
      h->launches += 1;
      x_set = true;
      st.converged = true;
      st.rel_residual = -1.0;  // not read back
      break;
    }
    ck(cudaMemcpyAsync(h->gpin, G, sizeof(stg::GmresDev), cudaMemcpyDeviceToHost, s), "memcpy");
    ck(cudaStreamSynchronize(s), "sync");
    check_admissibility(h);  // a nonphysical Euler state stops the solve here
    const stg::GmresDev& Gh = *h->gpin;
    if (bnorm < 0.0) bnorm = Gh.bnorm;  // deferred first cycle
    if (status == 4 || bnorm == 0.0) {   // b = 0: x = 0
      st.converged = true;
      st.rel_residual = 0.0;
      break;
    }
    if (Gh.k_done != k) throw std::runtime_error("gmres: device step count mismatch");
    for (int i = k - 1; i >= 0; --i) {
      double acc = Gh.g[i];
      for (int j = i + 1; j < k; ++j) acc -= Gh.H[size_t(i) * m + j] * y[size_t(j)];
      y[size_t(i)] = acc / Gh.H[size_t(i) * m + i];
    }
    for (int j = 0; j < k; ++j) hp[256 + j] = y[size_t(j)] * Gh.cn[j];  // x += sum y_j c_j S_j
    ck(cudaMemcpyAsync(dsm + 256, hp + 256, sizeof(double) * k, cudaMemcpyHostToDevice, s),
       "memcpy");
    // x (+)= sum y_j c_j Z_j (flexible) or sum y_j c_j S_j
    stg::vec_combine(x, P ? Z : V, ld, k, dsm + 256, n, s, x_set);
    h->launches++;
    x_set = true;
    if (status == 1) {
      // stop on the Arnoldi residual estimate, as Eigen's GMRES does; the
      // basis orthogonality keeps it close to the true residual (the Newton
      // residual that follows is computed exactly)
      st.converged = true;
      st.rel_residual = Gh.est / bnorm;
      break;
    }
    // no sync here: hp+256 is rewritten only after the next cycle's first
    // host read, which follows this H2D in stream order
  }
  if (!x_set) {  // no Arnoldi step ran (max_it = 0 or r = 0): x = 0
    stg::vec_fill(x, 0.0, n, s);
    h->launches++;
  }
  st.iterations = total;
  if (st.converged) h->gmres_pred[h->pred_slot] = total;
  check_launch(h);
  return st;
}

struct NewtonOut {
  int iterations = 0;
  int linear_iterations = 0;
  double final_residual = 0.0;
  std::vector<double> history;
};

// The linear system of one Newton iteration: the Jacobian action and an
// optional right preconditioner (empty function: none).
struct LinSys {
  Op A;
  Op P;
};

// newton_solve (newton.hpp:102-130) on device vectors; u holds u0 on entry.
NewtonOut newton(stg_handle* h, const Op& residual,
                 const std::function<LinSys(const double*)>& jacobian, double* u, long long n,
                 const stg_newton_config& cfg) {
  ensure_workspace(h);
  h->delta.ensure(size_t(n));
  // the residual is written straight into the first Krylov basis slot: the
  // GMRES that follows starts from it unnormalised (no copy or scaling pass)
  h->basis.ensure(size_t(round_up(n, 32)) * (cfg.gmres_restart + 1));
  double* r = h->basis.p;
  double* du = h->delta.p;
  NewtonOut out;
  AdmDefer defer(h);
  // the residual apply computes max |r| and <r,r> itself where it can
  // (fast 3-D kernel); otherwise a reduction pass reads r back
  auto residual_norm = [&]() -> double {
    h->red = true;
    try {
      residual(u, r);
    } catch (...) {
      h->red = false;
      throw;
    }
    h->red = false;
    if (!h->red_done) return dev_maxabs(h, r, n);
    ck(cudaMemcpyAsync(h->pinned + kRedMaxSlot, h->small.p + kRedMaxSlot, sizeof(double),
                       cudaMemcpyDeviceToHost, h->stream), "memcpy");
    ck(cudaStreamSynchronize(h->stream), "sync");
    return h->pinned[kRedMaxSlot];  // the bits of a non-negative double
  };
  // The first residual's norm is not waited for where the apply reduced it
  // itself: its read-back is enqueued, the first linear solve is enqueued
  // behind it, and the convergence test at the initial guess runs at that
  // solve's first host wait (gmres: early_stop), so the device does not idle
  // through a host round trip and the Jacobian / preconditioner set-up
  // between the residual and the solve (c4: ~45 us).  If the guess turns out
  // converged, the solve is abandoned before it touches u.
  // STG_NEWTON_SYNC_FIRST=1 waits for the norm first.
  static const bool sync_first = std::getenv("STG_NEWTON_SYNC_FIRST") != nullptr;
  double norm = 0.0, norm0 = 0.0;
  bool deferred = false;
  if (!sync_first && cfg.max_iter > 0 && cfg.gmres_tol < 1.0) {
    h->red = true;
    try {
      residual(u, r);
    } catch (...) {
      h->red = false;
      throw;
    }
    h->red = false;
    if (h->red_done) {
      ck(cudaMemcpyAsync(h->pinned + kRedMaxSlot, h->small.p + kRedMaxSlot, sizeof(double),
                         cudaMemcpyDeviceToHost, h->stream), "memcpy");
      deferred = true;
    } else {
      norm = dev_maxabs(h, r, n);
    }
  } else {
    norm = residual_norm();
  }
  auto converged = [&](double v) { return v <= cfg.abs_tol || v <= cfg.rel_tol * norm0; };
  if (!deferred) {
    check_admissibility(h);
    norm0 = norm;
    out.history.push_back(norm);
  }
  while (deferred || !converged(norm)) {
    if (!deferred && out.iterations >= cfg.max_iter)
      throw NonconvergenceError("newton_solve: no convergence in " +
                                    std::to_string(cfg.max_iter) + " iterations, residual " +
                                    fmt_short(norm),
                                out.history, out.linear_iterations);
    const bool red_r = h->red_done;  // <r,r> already in small[kRedSsSlot]
    h->eblock_built_now = h->eblock_in_use = false;
    LinSys J = jacobian(u);
    // (an operator apply inside jacobian() clears red_done; nothing there
    // writes small[kRedSsSlot])
    bool bb_ready = red_r && h->red_done;
    // J du = -r: the sign is folded into GMRES (b_sign = -1); du needs no
    // zero fill (gmres with x_zero writes it)
    GmresStats gs;
    // deferred first norm: read when the solve first waits on the device
    bool norm_read = false, stop = false;
    const std::function<bool()> first_norm = [&] {
      norm_read = true;
      norm = norm0 = h->pinned[kRedMaxSlot];  // the bits of a non-negative double
      out.history.push_back(norm);
      stop = converged(norm);
      return stop;
    };
    auto solve = [&] {
      h->pred_slot = std::min(out.iterations, stg_handle::kPredSlots - 1);
      gs = gmres(h, J.A, r, du, n, cfg.gmres_restart, cfg.gmres_tol, cfg.gmres_max_it,
                 J.P ? &J.P : nullptr, /*x_zero=*/true, /*pipelined=*/true,
                 /*b_sign=*/-1.0, /*want_rel=*/false, /*bb_ready=*/bb_ready, /*add_to=*/u,
                 deferred ? &first_norm : nullptr);
      out.linear_iterations += gs.iterations;
    };
    solve();
    if (deferred) {
      deferred = false;
      if (!norm_read) {  // the solve never waited (no step was enqueued)
        ck(cudaStreamSynchronize(h->stream), "sync");
        first_norm();
      }
      check_admissibility(h);
      if (stop) break;  // converged at the initial guess: u untouched
    }
    // Lagged Burgers element blocks (built for an earlier step's state): if
    // the solve failed with them, rebuild at u and solve again (the residual
    // slot was overwritten by the restarts: recompute it); if it merely took
    // clearly more steps than the solve right after the build, rebuild for
    // the next Newton iteration.
    if (h->eblock_in_use) {
      if (h->eblock_built_now) {
        h->eblock_fresh_its = gs.iterations;
      } else if (!gs.converged) {
        h->eblock_valid = false;
        residual_norm();
        const bool red_r2 = h->red_done;
        h->eblock_built_now = false;
        J = jacobian(u);
        bb_ready = red_r2 && h->red_done;
        solve();
        if (h->eblock_built_now) h->eblock_fresh_its = gs.iterations;
      } else if (gs.iterations > h->eblock_fresh_its + std::max(2, h->eblock_fresh_its / 2)) {
        h->eblock_valid = false;
      }
    }
    check_admissibility(h);
    if (!gs.converged)
      throw std::runtime_error("linear_solve: GMRES did not converge, error " +
                               fmt_short(gs.rel_residual));
    if (!gs.added) {  // (gmres added the correction into u itself otherwise)
      if (u == h->lazy_dst) materialise(h);
      stg::vec_axpy(u, 1.0, du, n, h->stream);
      h->launches++;
    }
    ++out.iterations;
    norm = residual_norm();
    check_admissibility(h);
    out.history.push_back(norm);
  }
  out.final_residual = norm;
  return out;
}

// stg_solve_info of a solve that stopped with NonconvergenceError: the
// iterations done so far and the residual history (newton.hpp:116-120)
NewtonOut partial_out(const NonconvergenceError& e) {
  NewtonOut p;
  p.history = e.history;
  p.iterations = e.history.empty() ? 0 : int(e.history.size()) - 1;
  p.linear_iterations = e.linear_iterations;
  p.final_residual = e.history.empty() ? 0.0 : e.history.back();
  return p;
}

void fill_info(stg_solve_info* info, const NewtonOut& o) {
  if (!info) return;
  info->failed_step = -1;
  info->newton_iterations = o.iterations;
  info->linear_iterations = o.linear_iterations;
  info->final_residual = o.final_residual;
  info->n_history = int(std::min<size_t>(o.history.size(), STG_MAX_HISTORY));
  for (int i = 0; i < info->n_history; ++i) info->residual_history[i] = o.history[size_t(i)];
}

// ---- operators as closures ---------------------------------------------------
void st_residual(stg_handle* h, double dt, const double* un, const double* U, double* R) {
  apply(h, st_mix(h, dt, un != nullptr), h->nt, h->nt, U, nullptr, un, R, false, false);
}

// Central-difference Jacobian action of the slab / stage residual without its
// constant (u_n / u) coupling, which cancels: [R0(U + h v) - R0(U - h v)] / 2h with
// h = fd_eps * sqrt(1 + ||U||_2) / ||v||_2 (the Walker-Pernice differencing
// parameter, as in PETSc's MFFD "wp"), so the perturbation is relative to the
// state regardless of the scaling of the Krylov vector v.
// un2 >= 0: ||U||_2 already known (U is fixed during a Newton linear solve);
// un2 == kUUOnDevice: <U,U> sits in small[kUUSlot] (fused path only)
constexpr double kUUOnDevice = -2.0;
constexpr int kUUSlot = 1001;
void fd_jvp(stg_handle* h, const stg::MixCoef& mix, bool full, const double* U, const double* v,
            double* Jv, double fd_eps, double un2 = -1.0) {
  const long long n = h->n_dof;
  if (h->desc.model == STG_MODEL_BURGERS && h->kernel_pref == STG_KERNEL_AUTO) {
    // fused: <v,v> on the device, then ONE kernel forms U +- e v per lane
    stg::SlabArgs a{};
    a.sp = h->sp;
    a.mx = mix;
    a.g = h->g;
    a.n_in = a.n_out = h->nt;
    a.full_s = full ? 1 : 0;
    a.model = h->desc.model;
    a.X = U;
    a.R = Jv;
    a.fdv = v;
    a.skip = h->skip;
    if (stg::fd_fused_supported(a)) {
      double* vv = h->small.p + kVVSlot;
      if (un2 == kUUOnDevice) {
        a.fd_uu = h->small.p + kUUSlot;
        a.fd_c = fd_eps;
      } else {
        const double un = un2 >= 0.0 ? un2 : std::sqrt(dev_dot(h, U, U, n));
        a.fd_c = fd_eps * std::sqrt(1.0 + un);
      }
      if (v != h->vv_of)  // (else the preconditioner that produced v reduced it)
        stg::vec_dot(v, v, n, h->partial.p, vv, h->stream, h->skip);
      h->vv_of = nullptr;
      a.fd_vv = vv;
      if (stg::launch_slab_generic(a, h->stream) < 0)
        throw std::runtime_error("fused FD Jacobian launch failed");
      h->launches += 2;
      check_launch(h);
      return;
    }
  }
  // central difference, the same two applies as a forward difference, O(h^2);
  // the step h is formed on the device from <v,v> (and <U,U>): no host sync
  double* vv = h->small.p + kVVSlot;
  if (v != h->vv_of) stg::vec_dot(v, v, n, h->partial.p, vv, h->stream, h->skip);
  h->vv_of = nullptr;
  const double* uu = nullptr;
  double c = fd_eps;
  if (un2 == kUUOnDevice) {
    uu = h->small.p + kUUSlot;
  } else {
    const double un = un2 >= 0.0 ? un2 : std::sqrt(dev_dot(h, U, U, n));
    c = fd_eps * std::sqrt(1.0 + un);
  }
  h->tmp1.ensure(size_t(n));
  h->tmp2.ensure(size_t(n));
  stg::vec_fd_pm(h->tmp1.p, h->tmp2.p, U, v, n, vv, uu, c, h->stream, h->skip);
  h->launches += 2;
  apply(h, mix, h->nt, h->nt, h->tmp1.p, nullptr, nullptr, Jv, false, full);
  apply(h, mix, h->nt, h->nt, h->tmp2.p, nullptr, nullptr, h->tmp1.p, false, full);
  stg::vec_fd_diff(Jv, h->tmp1.p, n, vv, uu, c, h->stream, h->skip);
  h->launches++;
}

// Host-buffer R(U) with the transfers pipelined against the compute (fast
// 3-D path): the mesh is cut into K z-chunks; chunk k's H2D (U's n_tau
// blocks and u_n) runs on s_in, its fast-kernel launch on the compute
// stream once chunk k (and the periodic z-neighbour layer it reads) has
// arrived, and its D2H on s_out right after.  PCIe is full duplex, so
// in-bound, out-bound and compute overlap.  Returns false when the fast
// kernel does not apply (the caller then runs the plain path).
bool st_residual_host_pipelined(stg_handle* h, double dt, const double* un_host,
                                const double* U_host, double* R_host) {
  const stg::Geometry& g = h->g;
  if (h->kernel_pref == STG_KERNEL_GENERIC || g.dim != 3 || g.nz < 2) return false;
  static const int kenv = [] {
    const char* e = std::getenv("STG_PIPE_K");
    return e ? std::atoi(e) : 0;
  }();
  int K = kenv > 0 && kenv <= stg_handle::kChunks ? kenv : stg_handle::kChunks;
  if (K > g.nz) K = g.nz;
  if (K < 2) return false;
  // chunk sizes in z-layers: a geometric ramp up and down (1, 2, 4, 8, 8, 4,
  // 2, 1 relative) so the first H2D before any compute and the last D2H after
  // it are small; STG_PIPE_UNIFORM=1 uses equal chunks
  static const bool uniform = std::getenv("STG_PIPE_UNIFORM") != nullptr;
  int zb[stg_handle::kChunks + 1];
  {
    double wsum = 0.0, w[stg_handle::kChunks];
    for (int k = 0; k < K; ++k) {
      const int d = std::min(k, K - 1 - k);
      w[k] = uniform ? 1.0 : double(1 << std::min(d, 3));
      wsum += w[k];
    }
    int acc = 0;
    double cw = 0.0;
    zb[0] = 0;
    for (int k = 0; k < K; ++k) {
      cw += w[k];
      int b = k + 1 == K ? g.nz : int(std::lround(g.nz * cw / wsum));
      b = std::max(b, acc + 1);                // every chunk has a layer
      b = std::min(b, g.nz - (K - 1 - k));     // and leaves one for each later chunk
      zb[k + 1] = acc = b;
    }
  }
  const long long ns = h->n_sdof, nd = h->n_dof;
  h->host_U.ensure(size_t(nd));
  h->host_R.ensure(size_t(nd));
  h->host_u.ensure(size_t(ns));
  stg::SlabArgs a{};
  a.sp = h->sp;
  a.mx = st_mix(h, dt, true);
  a.g = g;
  a.n_in = a.n_out = h->nt;
  a.has_w = 1;
  a.model = h->desc.model;
  a.X = h->host_U.p;
  a.W = h->host_u.p;
  a.R = h->host_R.p;
  a.no_pdl = 1;  // each chunk's launch follows an H2D event wait
  if (!stg::slab_fast_supported(a)) return false;
  if (!h->s_in) {
    ck(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming), "event");
    for (int k = 0; k < stg_handle::kChunks; ++k) {
      ck(cudaEventCreateWithFlags(&h->ev_in[k], cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&h->ev_c[k], cudaEventDisableTiming), "event");
    }
  }
  const long long layer = (long long)g.nx * g.ny * g.npc;  // doubles per layer per block
  const int seg_per_layer = g.nx * g.ny / 8;
  const bool needL = h->sp.cL[2] != 0.0, needR = h->sp.cR[2] != 0.0;
  // earlier work on the compute stream may still read the device buffers
  ck(cudaEventRecord(h->ev_start, h->stream), "event");
  ck(cudaStreamWaitEvent(h->s_in, h->ev_start, 0), "wait");
  const size_t pitch = sizeof(double) * size_t(ns);  // one temporal block
  static const bool one_d = std::getenv("STG_PIPE_1D") != nullptr;
  auto copy_layers = [&](int z0, int nl) {
    const long long off = z0 * layer, cnt = nl * layer;
    if (one_d) {  // one contiguous copy per temporal block
      for (int t = 0; t < h->nt; ++t)
        ck(cudaMemcpyAsync(h->host_U.p + t * ns + off, U_host + t * ns + off,
                           sizeof(double) * cnt, cudaMemcpyHostToDevice, h->s_in), "H2D");
    } else {  // one strided copy moves the chunk's slice of all n_tau blocks
      ck(cudaMemcpy2DAsync(h->host_U.p + off, pitch, U_host + off, pitch, sizeof(double) * cnt,
                           size_t(h->nt), cudaMemcpyHostToDevice, h->s_in), "H2D");
    }
    ck(cudaMemcpyAsync(h->host_u.p + off, un_host + off, sizeof(double) * cnt,
                       cudaMemcpyHostToDevice, h->s_in), "H2D");
  };
  // STG_PIPE_TRACE=1: time-stamp every chunk's H2D / kernel / D2H (stderr)
  static const bool trace = std::getenv("STG_PIPE_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  auto stamp = [&](cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tev.push_back(e);
  };
  stamp(h->s_in);
  if (needL) copy_layers(g.nz - 1, 1);  // periodic z- neighbour of chunk 0
  for (int k = 0; k < K; ++k) {
    copy_layers(zb[k], zb[k + 1] - zb[k]);
    ck(cudaEventRecord(h->ev_in[k], h->s_in), "event");
    stamp(h->s_in);
  }
  for (int k = 0; k < K; ++k) {
    ck(cudaStreamWaitEvent(h->stream, h->ev_in[needR ? std::min(k + 1, K - 1) : k], 0), "wait");
    a.seg_begin = zb[k] * seg_per_layer;
    a.seg_end = zb[k + 1] * seg_per_layer;
    if (stg::launch_slab_fast(a, h->stream) < 0)
      throw std::runtime_error("fast kernel launch failed in the pipelined path");
    h->launches++;
    check_launch(h);
    ck(cudaEventRecord(h->ev_c[k], h->stream), "event");
    stamp(h->stream);
    ck(cudaStreamWaitEvent(h->s_out, h->ev_c[k], 0), "wait");
    const long long off = zb[k] * layer, cnt = (zb[k + 1] - zb[k]) * layer;
    if (one_d) {
      for (int t = 0; t < h->nt; ++t)
        ck(cudaMemcpyAsync(R_host + t * ns + off, h->host_R.p + t * ns + off,
                           sizeof(double) * cnt, cudaMemcpyDeviceToHost, h->s_out), "D2H");
    } else {
      ck(cudaMemcpy2DAsync(R_host + off, pitch, h->host_R.p + off, pitch, sizeof(double) * cnt,
                           size_t(h->nt), cudaMemcpyDeviceToHost, h->s_out), "D2H");
    }
    stamp(h->s_out);
  }
  ck(cudaStreamSynchronize(h->s_out), "sync");
  if (trace) {
    cudaDeviceSynchronize();
    // order: start, in[0..K-1], then (kernel k, out k) pairs
    std::fprintf(stderr, "pipe K=%d in:", K);
    float ms = 0.f;
    for (int k = 0; k < K; ++k) {
      cudaEventElapsedTime(&ms, tev[0], tev[size_t(1 + k)]);
      std::fprintf(stderr, " %.3f", ms);
    }
    std::fprintf(stderr, " | kern/out:");
    for (int k = 0; k < K; ++k) {
      float a = 0.f, b = 0.f;
      cudaEventElapsedTime(&a, tev[0], tev[size_t(1 + K + 2 * k)]);
      cudaEventElapsedTime(&b, tev[0], tev[size_t(2 + K + 2 * k)]);
      std::fprintf(stderr, " %.3f/%.3f", a, b);
    }
    std::fprintf(stderr, "\n");
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
  }
  return true;
}

// ---- pageable callers (hostcopy.hpp) ----------------------------------------
constexpr size_t kStageChunk = size_t(1) << 20;  // doubles per staged chunk (8 MiB)

cudaEvent_t stage_event(stg_handle* h, size_t i) {
  while (h->ev_stage.size() <= i) {
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    h->ev_stage.push_back(e);
  }
  return h->ev_stage[i];
}

// n doubles from pageable host memory to the device on stream s: worker
// threads fill the page-locked mirror chunk by chunk while the copy engine
// moves the previous chunk
void staged_h2d(stg_handle* h, double* dev, const double* host, size_t n, PinBuf& pin,
                cudaStream_t s) {
  pin.ensure(n);
  stg::HostCopyPool& pool = stg::HostCopyPool::get();
  for (size_t off = 0; off < n; off += kStageChunk) {
    const size_t cnt = std::min(kStageChunk, n - off);
    const stg::CopyItem it{pin.p + off, host + off, cnt * sizeof(double)};
    pool.par_copy(&it, 1);
    ck(cudaMemcpyAsync(dev + off, pin.p + off, cnt * sizeof(double), cudaMemcpyHostToDevice, s),
       "H2D");
  }
  (void)h;
}

// n doubles from the device to pageable host memory, in two halves: enqueue
// every chunk's D2H into the mirror on s (an event after each), then drain:
// the workers copy chunk i out to `host` while the copy engine moves chunk
// i + 1.  ev_base: first index into the handle's staging events (two
// transfers of one call do not share events).
void staged_d2h_enqueue(stg_handle* h, const double* dev, size_t n, PinBuf& pin, cudaStream_t s,
                        size_t ev_base) {
  pin.ensure(n);
  size_t i = 0;
  for (size_t off = 0; off < n; off += kStageChunk, ++i) {
    const size_t cnt = std::min(kStageChunk, n - off);
    ck(cudaMemcpyAsync(pin.p + off, dev + off, cnt * sizeof(double), cudaMemcpyDeviceToHost, s),
       "D2H");
    ck(cudaEventRecord(stage_event(h, ev_base + i), s), "event");
  }
}

void staged_d2h_drain(stg_handle* h, double* host, size_t n, PinBuf& pin, size_t ev_base) {
  stg::HostCopyPool& pool = stg::HostCopyPool::get();
  size_t i = 0;
  for (size_t off = 0; off < n; off += kStageChunk, ++i) {
    const size_t cnt = std::min(kStageChunk, n - off);
    ck(cudaEventSynchronize(h->ev_stage[ev_base + i]), "sync");
    const stg::CopyItem it{host + off, pin.p + off, cnt * sizeof(double)};
    pool.par_copy(&it, 1);
  }
}

void staged_d2h(stg_handle* h, double* host, const double* dev, size_t n, PinBuf& pin,
                cudaStream_t s) {
  staged_d2h_enqueue(h, dev, n, pin, s, 0);
  staged_d2h_drain(h, host, n, pin, 0);
}

// The pipelined host-buffer R(U) (st_residual_host_pipelined) for pageable
// caller memory: K equal z-chunks; the workers gather chunk k (its slice of
// every temporal block of U, and of u_n) into the page-locked mirrors, its
// H2D, kernel launch and D2H (into the mirror of R) are enqueued, and while
// those run the workers gather chunk k + 1; finished chunks of R are copied
// out to the caller as their D2H events complete.  Returns false when the
// fast kernel does not apply.
bool st_residual_host_staged(stg_handle* h, double dt, const double* un_host,
                             const double* U_host, double* R_host) {
  const stg::Geometry& g = h->g;
  if (h->kernel_pref == STG_KERNEL_GENERIC || g.dim != 3 || g.nz < 2) return false;
  int K = std::min<int>(stg_handle::kChunks, g.nz);
  if (K < 2) return false;
  const long long ns = h->n_sdof, nd = h->n_dof;
  h->host_U.ensure(size_t(nd));
  h->host_R.ensure(size_t(nd));
  h->host_u.ensure(size_t(ns));
  stg::SlabArgs a{};
  a.sp = h->sp;
  a.mx = st_mix(h, dt, true);
  a.g = g;
  a.n_in = a.n_out = h->nt;
  a.has_w = 1;
  a.model = h->desc.model;
  a.X = h->host_U.p;
  a.W = h->host_u.p;
  a.R = h->host_R.p;
  a.no_pdl = 1;
  if (!stg::slab_fast_supported(a)) return false;
  h->pin_U.ensure(size_t(nd));
  h->pin_R.ensure(size_t(nd));
  h->pin_u.ensure(size_t(ns));
  if (!h->s_in) {
    ck(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming), "event");
    for (int k = 0; k < stg_handle::kChunks; ++k) {
      ck(cudaEventCreateWithFlags(&h->ev_in[k], cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&h->ev_c[k], cudaEventDisableTiming), "event");
    }
  }
  stage_event(h, size_t(K));
  int zb[stg_handle::kChunks + 1];
  for (int k = 0; k <= K; ++k) zb[k] = int((long long)g.nz * k / K);
  const long long layer = (long long)g.nx * g.ny * g.npc;
  const int seg_per_layer = g.nx * g.ny / 8;
  const bool needL = h->sp.cL[2] != 0.0, needR = h->sp.cR[2] != 0.0;
  const size_t pitch = sizeof(double) * size_t(ns);
  const int nt = h->nt;
  stg::HostCopyPool& pool = stg::HostCopyPool::get();
  ck(cudaEventRecord(h->ev_start, h->stream), "event");
  ck(cudaStreamWaitEvent(h->s_in, h->ev_start, 0), "wait");
  // gather layers [z0, z0 + nl) into the mirrors and enqueue their H2D
  auto in_layers = [&](int z0, int nl) {
    const long long off = z0 * layer, cnt = nl * layer;
    stg::CopyItem items[8];
    int ni = 0;
    for (int t = 0; t < nt; ++t)
      items[ni++] = {h->pin_U.p + t * ns + off, U_host + t * ns + off, sizeof(double) * size_t(cnt)};
    items[ni++] = {h->pin_u.p + off, un_host + off, sizeof(double) * size_t(cnt)};
    pool.par_copy(items, ni);
    ck(cudaMemcpy2DAsync(h->host_U.p + off, pitch, h->pin_U.p + off, pitch, sizeof(double) * cnt,
                         size_t(nt), cudaMemcpyHostToDevice, h->s_in), "H2D");
    ck(cudaMemcpyAsync(h->host_u.p + off, h->pin_u.p + off, sizeof(double) * cnt,
                       cudaMemcpyHostToDevice, h->s_in), "H2D");
  };
  // launch chunk j (its inputs' events recorded) and enqueue its D2H
  auto run_chunk = [&](int j) {
    ck(cudaStreamWaitEvent(h->stream, h->ev_in[needR ? std::min(j + 1, K - 1) : j], 0), "wait");
    a.seg_begin = zb[j] * seg_per_layer;
    a.seg_end = zb[j + 1] * seg_per_layer;
    if (stg::launch_slab_fast(a, h->stream) < 0)
      throw std::runtime_error("fast kernel launch failed in the staged host path");
    h->launches++;
    check_launch(h);
    ck(cudaEventRecord(h->ev_c[j], h->stream), "event");
    ck(cudaStreamWaitEvent(h->s_out, h->ev_c[j], 0), "wait");
    const long long off = zb[j] * layer, cnt = (zb[j + 1] - zb[j]) * layer;
    ck(cudaMemcpy2DAsync(h->pin_R.p + off, pitch, h->host_R.p + off, pitch, sizeof(double) * cnt,
                         size_t(nt), cudaMemcpyDeviceToHost, h->s_out), "D2H");
    ck(cudaEventRecord(h->ev_stage[size_t(j)], h->s_out), "event");
  };
  int copied_out = 0;  // chunks of R already handed to the caller
  auto out_chunk = [&](int j) {
    const long long off = zb[j] * layer, cnt = (zb[j + 1] - zb[j]) * layer;
    stg::CopyItem items[8];
    int ni = 0;
    for (int t = 0; t < nt; ++t)
      items[ni++] = {R_host + t * ns + off, h->pin_R.p + t * ns + off, sizeof(double) * size_t(cnt)};
    pool.par_copy(items, ni);
  };
  if (needL) in_layers(g.nz - 1, 1);  // periodic z- neighbour of chunk 0
  for (int k = 0; k < K; ++k) {
    in_layers(zb[k], zb[k + 1] - zb[k]);
    ck(cudaEventRecord(h->ev_in[k], h->s_in), "event");
    if (!needR) run_chunk(k);
    else if (k > 0) run_chunk(k - 1);
    // hand finished chunks out between gathers (keeps the tail short)
    while (copied_out < k && cudaEventQuery(h->ev_stage[size_t(copied_out)]) == cudaSuccess)
      out_chunk(copied_out++);
  }
  if (needR) run_chunk(K - 1);
  for (; copied_out < K; ++copied_out) {
    ck(cudaEventSynchronize(h->ev_stage[size_t(copied_out)]), "sync");
    out_chunk(copied_out);
  }
  return true;
}

// whether this handle's vectors are worth the worker threads (below 1 MiB the
// driver's own staging is as fast) and staging is not switched off
bool stage_large(const stg_handle* h) {
  static const bool off = std::getenv("STG_HOST_NO_STAGING") != nullptr;
  return !off && size_t(h->n_dof) * sizeof(double) >= (size_t(1) << 20);
}

// copy-in / copy-out of the host-buffer slab steps (stg_stdg_step_host,
// stg_rk_step_host): plain async copies for page-locked caller memory, the
// staged ones for pageable memory
void step_host_in(stg_handle* h, const double* u) {
  cudaStream_t s = h->stream;
  if (stage_large(h) && pageable(u))
    staged_h2d(h, h->host_u.p, u, size_t(h->n_sdof), h->pin_u, s);
  else
    ck(cudaMemcpyAsync(h->host_u.p, u, sizeof(double) * h->n_sdof, cudaMemcpyHostToDevice, s),
       "H2D");
}

void step_host_out(stg_handle* h, double* U, double* u_next) {
  cudaStream_t s = h->stream;
  const bool stU = stage_large(h) && pageable(U);
  const bool stu = u_next && stage_large(h) && pageable(u_next);
  // page-locked destinations first: their DMA runs while the workers copy
  if (!stU)
    ck(cudaMemcpyAsync(U, h->host_U.p, sizeof(double) * h->n_dof, cudaMemcpyDeviceToHost, s), "D2H");
  if (u_next && !stu)
    ck(cudaMemcpyAsync(u_next, h->host_u2.p, sizeof(double) * h->n_sdof, cudaMemcpyDeviceToHost,
                       s), "D2H");
  const size_t nU = (size_t(h->n_dof) + kStageChunk - 1) / kStageChunk;
  if (stU) staged_d2h_enqueue(h, h->host_U.p, size_t(h->n_dof), h->pin_U, s, 0);
  if (stu) staged_d2h_enqueue(h, h->host_u2.p, size_t(h->n_sdof), h->pin_u2, s, nU);
  if (stU) staged_d2h_drain(h, U, size_t(h->n_dof), h->pin_U, 0);
  if (stu) staged_d2h_drain(h, u_next, size_t(h->n_sdof), h->pin_u2, nU);
  ck(cudaStreamSynchronize(s), "sync");
}

// Euler has no exact linearisation here: a finite-difference step is always used
// (the reference differences too, spatial.hpp:299-320).  Default fd_eps 1e-5:
// the central difference's truncation (h^2) and rounding (eps_mach / h) errors
// balance near h ~ eps_mach^(1/3) per entry.
constexpr double kEulerFdEps = 1e-5;
double effective_fd_eps(const stg_handle* h, double fd_eps) {
  return h->desc.model == STG_MODEL_EULER && fd_eps <= 0.0 ? kEulerFdEps : fd_eps;
}

// whether the Jacobian action of this handle differences (Burgers with
// fd_eps > 0, Euler always)
bool uses_fd(const stg_handle* h, double fd_eps) {
  return !linear_model(h->desc.model) && effective_fd_eps(h, fd_eps) > 0.0;
}

// <U,U> for the FD Jacobian action at U, left on the device: both FD
// actions form their step there (no host round trip inside GMRES)
double fd_norm(stg_handle* h, double fd_eps, const double* U, long long n) {
  if (!uses_fd(h, fd_eps)) return -1.0;
  stg::vec_dot(U, U, n, h->partial.p, h->small.p + kUUSlot, h->stream);
  h->launches++;
  return kUUOnDevice;
}


void st_jvp(stg_handle* h, double dt, const double* U, const double* v, double* Jv,
            double fd_eps, double un2 = -1.0) {
  fd_eps = effective_fd_eps(h, fd_eps);
  if (linear_model(h->desc.model)) {
    // linear: J v = R(v) with the u_n coupling removed (stdg.hpp:79-110)
    apply(h, st_mix(h, dt, false), h->nt, h->nt, v, nullptr, nullptr, Jv, false, false);
  } else if (fd_eps <= 0.0) {
    apply(h, st_mix(h, dt, false), h->nt, h->nt, v, U, nullptr, Jv, true, false);
  } else {
    fd_jvp(h, st_mix(h, dt, false), false, U, v, Jv, fd_eps, un2);
  }
}

void stage_residual(stg_handle* h, int form, double dt, const double* u, const double* U,
                    double* R) {
  apply(h, stage_mix(h, form, dt, true), h->nt, h->nt, U, nullptr, u, R, false,
        form == STG_FORM_A);
}

void stage_jvp(stg_handle* h, int form, double dt, const double* U, const double* v, double* Jv,
               double fd_eps, double un2 = -1.0) {
  const bool full = form == STG_FORM_A;
  fd_eps = effective_fd_eps(h, fd_eps);
  if (linear_model(h->desc.model)) {
    apply(h, stage_mix(h, form, dt, false), h->nt, h->nt, v, nullptr, nullptr, Jv, false, full);
  } else if (fd_eps <= 0.0) {
    apply(h, stage_mix(h, form, dt, false), h->nt, h->nt, v, U, nullptr, Jv, true, full);
  } else {
    fd_jvp(h, stage_mix(h, form, dt, false), full, U, v, Jv, fd_eps, un2);
  }
}

// Fast-diagonalisation factors of the d = 3 element-local Jacobian block
// L_e = T (x) I + S (x) (V_z (+) V_y (+) V_x) (kernels_fdm.cu).  False when
// S is singular or a factor has no accurate eigen-decomposition of the form
// the kernel assumes (V_x: two complex-conjugate pairs).
bool build_fdm(const stg::SpatialCoef& sp, const stg::MixCoef& mx, stg::FdmCoef& c) {
  using stg::cplx;
  constexpr int n = 4;
  try {
    std::vector<double> S(n * n), T(n * n);
    for (int r = 0; r < n; ++r)
      for (int j = 0; j < n; ++j) {
        S[size_t(r) * n + j] = mx.S[r][j];
        T[size_t(r) * n + j] = mx.T[r][j];
      }
    const std::vector<double> Si = stg::inverse(S, n);
    std::vector<double> G(n * n, 0.0);
    for (int r = 0; r < n; ++r)
      for (int j = 0; j < n; ++j)
        for (int q = 0; q < n; ++q) G[size_t(r) * n + j] += Si[size_t(r) * n + q] * T[size_t(q) * n + j];
    std::vector<cplx> lt, Q, Qi, th[3], P[3], Pi[3];
    if (!stg::eig_real(G, n, lt, Q, Qi)) return false;
    for (int a = 0; a < 3; ++a) {
      std::vector<double> V(n * n);
      for (int i = 0; i < n; ++i)
        for (int k = 0; k < n; ++k) V[size_t(i) * n + k] = sp.V[a][i][k];
      if (!stg::eig_real(V, n, th[a], P[a], Pi[a])) return false;
    }
    // x modes: keep one member of each conjugate pair (0, 2)
    for (int j = 0; j < 2; ++j)
      if (!(th[0][size_t(2 * j)].imag() > 0.0) ||
          th[0][size_t(2 * j + 1)] != std::conj(th[0][size_t(2 * j)]))
        return false;
    auto put = [](double* dst, cplx z) {
      dst[0] = z.real();
      dst[1] = z.imag();
    };
    for (int r = 0; r < n; ++r)
      for (int q = 0; q < n; ++q) {
        cplx ft = 0.0;
        for (int m = 0; m < n; ++m) ft += Qi[size_t(r) * n + m] * Si[size_t(m) * n + q];
        put(c.FT[r][q], ft);
        put(c.IT[r][q], Q[size_t(r) * n + q]);
        put(c.FZ[r][q], Pi[2][size_t(r) * n + q]);
        put(c.IZ[r][q], P[2][size_t(r) * n + q]);
        put(c.FY[r][q], Pi[1][size_t(r) * n + q]);
        put(c.IY[r][q], P[1][size_t(r) * n + q]);
      }
    for (int j = 0; j < 2; ++j)
      for (int x = 0; x < n; ++x) {
        put(c.FX[j][x], Pi[0][size_t(2 * j) * n + x]);
        put(c.IX[x][j], P[0][size_t(x) * n + 2 * j]);
      }
    for (int it = 0; it < n; ++it)
      for (int iz = 0; iz < n; ++iz)
        for (int iy = 0; iy < n; ++iy)
          for (int j = 0; j < 2; ++j) {
            const cplx lam = lt[size_t(it)] + th[2][size_t(iz)] + th[1][size_t(iy)] + th[0][size_t(2 * j)];
            if (std::abs(lam) < 1e-300) return false;
            put(c.LI[it][iz][iy][j], 1.0 / lam);
          }
    return true;
  } catch (const std::exception&) {
    return false;
  }
}

// Factors of fdm3_kernel (kernels_fdm.cu): the complex eigen-decompositions
// of the per-axis element matrices V_a = P_a Th_a P_a^-1 and, per kept spatial
// mode theta = thz + thy + thx, the temporal inverse (T + theta S)^-1, written
// to M ([iz][it][t][q] complex, q = iy * 2 + j).  False when V_x does not have
// two complex-conjugate pairs, an eigen-decomposition is inaccurate or a
// temporal block is singular.
bool build_fdm3(const stg::SpatialCoef& sp, const stg::MixCoef& mx, stg::FdmCoef3& c) {
  using stg::cplx;
  constexpr int n = 4;
  try {
    std::vector<cplx> th[3], P[3], Pi[3];
    for (int a = 0; a < 3; ++a) {
      std::vector<double> V(n * n);
      for (int i = 0; i < n; ++i)
        for (int k = 0; k < n; ++k) V[size_t(i) * n + k] = sp.V[a][i][k];
      if (!stg::eig_real(V, n, th[a], P[a], Pi[a])) return false;
    }
    // every axis: two conjugate pairs (2P, 2P + 1) with conjugate eigenvector
    // columns and P^-1 rows (the kernel forms the partner from the member)
    for (int a = 0; a < 3; ++a)
      for (int pr = 0; pr < 2; ++pr) {
        const size_t m0 = size_t(2 * pr), m1 = m0 + 1;
        if (!(th[a][m0].imag() > 0.0) || th[a][m1] != std::conj(th[a][m0])) return false;
        for (int k = 0; k < n; ++k) {
          if (P[a][size_t(k) * n + m1] != std::conj(P[a][size_t(k) * n + m0])) return false;
          const cplx d = Pi[a][m1 * n + size_t(k)] - std::conj(Pi[a][m0 * n + size_t(k)]);
          if (std::abs(d) > 1e-12 * (1.0 + std::abs(Pi[a][m0 * n + size_t(k)]))) return false;
        }
      }
    auto put = [](double* dst, cplx z) {
      dst[0] = z.real();
      dst[1] = z.imag();
    };
    for (int pr = 0; pr < 2; ++pr)
      for (int q = 0; q < n; ++q) {
        put(c.FZ[pr][q], Pi[2][size_t(2 * pr) * n + q]);
        put(c.IZ[q][pr], P[2][size_t(q) * n + 2 * pr]);
        put(c.FY[pr][q], Pi[1][size_t(2 * pr) * n + q]);
        put(c.IY[q][pr], P[1][size_t(q) * n + 2 * pr]);
      }
    for (int j = 0; j < 2; ++j)
      for (int x = 0; x < n; ++x) {
        put(c.FX[j][x], Pi[0][size_t(2 * j) * n + x]);
        put(c.IX[x][j], 2.0 * P[0][size_t(x) * n + 2 * j]);  // 2 Re(.) of the kept half
      }
    std::vector<cplx> A(n * n), Ai;
    for (int iz = 0; iz < n; ++iz)
      for (int iy = 0; iy < n; ++iy)
        for (int j = 0; j < 2; ++j) {
          const cplx theta = th[2][size_t(iz)] + th[1][size_t(iy)] + th[0][size_t(2 * j)];
          for (int r = 0; r < n; ++r)
            for (int t = 0; t < n; ++t) A[size_t(r) * n + t] = mx.T[r][t] + theta * mx.S[r][t];
          if (!stg::cinverse(A, Ai, n)) return false;
          const int q = iy * 2 + j;
          for (int it = 0; it < n; ++it)
            for (int t = 0; t < n; ++t) put(c.M[iz][it][t][q], Ai[size_t(it) * n + t]);
        }
    return true;
  } catch (const std::exception&) {
    return false;
  }
}

// d = 2 advection: one shared dense element block, n_tau * n^2 <= 128
bool dense2d_ok(const stg_handle* h) {
  return h->desc.dim == 2 && h->desc.model == STG_MODEL_ADVECTION &&
         h->nt * h->g.npc <= 128;
}

bool fdm_ok(const stg_handle* h) {
  return h->desc.dim == 3 && h->desc.model == STG_MODEL_ADVECTION &&
         (stg::fdm3_supported(h->g, h->nt) || stg::fdm_supported(h->g, h->nt));
}

// general linear models (advdiff): element blocks n_tau * npc * r <= 32
bool gen_eblock_ok(const stg_handle* h) {
  return h->desc.model == STG_MODEL_ADVDIFF && h->nt * h->g.npc * h->r <= 32;
}

// Neumann terms of STG_PRECOND_POLY (env STG_POLY_TERMS, default 7).  With
// the couplings fused into the block apply a term costs ~50 us at c4 size
// against ~100 us for a GMRES step's operator apply and Gram-Schmidt passes:
// m = 7 converges c4, c2 and c5 in one GMRES step at 1e-10 (c4 / c2 / c5
// slab solves 0.72 / 0.68 / 0.82 ms; m = 3: two steps, 0.81 / 0.78 / 0.91;
// m = 6 takes c4 alone to one step, 0.67 ms, but c2 and c5 to two)
int poly_terms() {
  static const int m = [] {
    const char* e = std::getenv("STG_POLY_TERMS");
    const int v = e ? std::atoi(e) : 7;
    return v < 0 ? 0 : v;
  }();
  return m;
}

// the base block preconditioner P0 of STG_PRECOND_POLY
int poly_base(const stg_handle* h) {
  if (h->desc.dim == 1 && h->desc.model == STG_MODEL_BURGERS &&
      stg::sweep_supported(h->nt, h->n1))
    return STG_PRECOND_SWEEP;
  return STG_PRECOND_EBLOCK;
}

int resolve_precond(const stg_handle* h, int kind) {
  if (kind == STG_PRECOND_POLY) {
    resolve_precond(h, poly_base(h));  // throws where the base block does not exist
    return STG_PRECOND_POLY;
  }
  if (general_model(h->desc.model)) {
    if (kind == STG_PRECOND_NONE) return STG_PRECOND_NONE;
    if (kind == STG_PRECOND_JACOBI)
      throw std::invalid_argument("diagonal (Jacobi) preconditioner: advection only");
    if (kind == STG_PRECOND_AUTO) return gen_eblock_ok(h) ? STG_PRECOND_EBLOCK : STG_PRECOND_NONE;
    if (kind == STG_PRECOND_EBLOCK && gen_eblock_ok(h)) return STG_PRECOND_EBLOCK;
    throw std::invalid_argument(
        "block-Jacobi preconditioners for the general models: element blocks of the linear "
        "advdiff model with n_tau * (N+1)^d <= 32 only");
  }
  if (kind == STG_PRECOND_AUTO && h->desc.dim == 1 && h->desc.model == STG_MODEL_BURGERS)
    return stg::eblock_f32_supported(h->nt, h->n1)
               ? (stg::sweep_supported(h->nt, h->n1) ? STG_PRECOND_SWEEP : STG_PRECOND_EBLOCK)
               : STG_PRECOND_NONE;
  if (kind == STG_PRECOND_SWEEP &&
      !(h->desc.dim == 1 && h->desc.model == STG_MODEL_BURGERS &&
        stg::eblock_f32_supported(h->nt, h->n1) && stg::sweep_supported(h->nt, h->n1)))
    throw std::invalid_argument("upwind block sweep: d = 1 Burgers, n_tau = 4, degree 1 or 3");
  // d >= 2 advection with an exact element-block inverse: the polynomial
  // preconditioner around it (c4 slab solve 1.57 -> 1.08 ms, c2 1.65 ->
  // 1.15 ms: 7 GMRES steps -> 2); d = 1 keeps the element blocks (the fused
  // small solve takes c1)
  static const bool no_poly = std::getenv("STG_AUTO_NO_POLY") != nullptr;
  if (kind == STG_PRECOND_AUTO && h->desc.dim >= 2 && (fdm_ok(h) || dense2d_ok(h)) && !no_poly &&
      poly_terms() > 0 && stg::offdiag_supported(h->g, h->nt))
    return STG_PRECOND_POLY;
  if (kind == STG_PRECOND_AUTO)
    return (h->desc.dim == 1 || fdm_ok(h) || dense2d_ok(h))
               ? STG_PRECOND_EBLOCK
               : (h->desc.model == STG_MODEL_ADVECTION ? STG_PRECOND_TBLOCK : STG_PRECOND_NONE);
  if (kind == STG_PRECOND_EBLOCK && h->desc.dim != 1 && !fdm_ok(h) && !dense2d_ok(h))
    throw std::invalid_argument(
        "element-block Jacobi: d = 1, or d = 3 advection with degree 3, n_tau = 4 and a cell "
        "count divisible by 8");
  if (kind == STG_PRECOND_TBLOCK && h->desc.model != STG_MODEL_ADVECTION)
    throw std::invalid_argument("temporal-block Jacobi: advection only");
  if (kind == STG_PRECOND_JACOBI && h->desc.model != STG_MODEL_ADVECTION)
    throw std::invalid_argument("diagonal (Jacobi) preconditioner: advection only");
  if (kind < STG_PRECOND_NONE || kind > STG_PRECOND_POLY)
    throw std::invalid_argument("unknown preconditioner");
  return kind;
}

// Complex eigen-decomposition V = P diag(th) P^-1 of a real element matrix
// with the real eigenvalues' eigenvectors made real (phase of the largest
// entry removed) and the mode order [real, pair members with Im > 0, their
// conjugates]: ord[i] indexes th / the columns of P.  False when the
// factorisation does not reproduce V to 1e-11.
bool eig_ordered(const double (&Vm)[stg::kMaxN][stg::kMaxN], int n, std::vector<stg::cplx>& th,
                 std::vector<stg::cplx>& P, std::vector<stg::cplx>& Pi, std::vector<int>& ord,
                 int& nr, int& np) {
  using stg::cplx;
  std::vector<double> V(size_t(n) * n);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) V[size_t(i) * n + k] = Vm[i][k];
  if (!stg::eig_real(V, n, th, P, Pi)) return false;
  ord.clear();
  nr = np = 0;
  for (int k = 0; k < n; ++k)
    if (th[size_t(k)].imag() == 0.0) {
      cplx big = 0.0;
      for (int r = 0; r < n; ++r)
        if (std::abs(P[size_t(r) * n + k]) > std::abs(big)) big = P[size_t(r) * n + k];
      const cplx ph = std::conj(big) / std::abs(big);
      for (int r = 0; r < n; ++r)
        P[size_t(r) * n + k] = cplx((P[size_t(r) * n + k] * ph).real(), 0.0);
      ord.push_back(k);
      ++nr;
    }
  std::vector<int> conj_of;
  for (int k = 0; k < n; ++k)
    if (th[size_t(k)].imag() > 0.0) {
      ord.push_back(k);
      ++np;
      int best = -1;
      for (int q = 0; q < n; ++q)
        if (q != k && th[size_t(q)] == std::conj(th[size_t(k)])) best = q;
      if (best < 0) return false;
      conj_of.push_back(best);
    }
  for (int q : conj_of) ord.push_back(q);
  if (nr + 2 * np != n || int(ord.size()) != n) return false;
  if (!stg::cinverse(P, Pi, n)) return false;
  double err = 0.0, mxv = 0.0;
  for (int r = 0; r < n; ++r)
    for (int q = 0; q < n; ++q) {
      cplx acc = 0.0;
      for (int k = 0; k < n; ++k) acc += P[size_t(r) * n + k] * th[size_t(k)] * Pi[size_t(k) * n + q];
      err = std::max(err, std::abs(acc - Vm[r][q]));
      mxv = std::max(mxv, std::abs(Vm[r][q]));
    }
  return err <= 1e-11 * std::max(mxv, 1e-300);
}

// Factors of fdm2i_kernel (kernels_fdm.cu, FdmCoef2i in kernels.hpp).
bool build_fdm2i(const stg::SpatialCoef& sp, const stg::MixCoef& mx, int n, int nt,
                 stg::FdmCoef2i& c, int& nr, int& np) {
  using stg::cplx;
  try {
    std::vector<cplx> thx, Px, Pix, thy, Py, Piy;
    std::vector<int> ox, oy;
    int nry = 0, npy = 0;
    if (!eig_ordered(sp.V[0], n, thx, Px, Pix, ox, nr, np)) return false;
    if (!eig_ordered(sp.V[1], n, thy, Py, Piy, oy, nry, npy)) return false;
    if (nry != nr || npy != np) return false;
    std::memset(&c, 0, sizeof c);
    auto put = [](double* dst, cplx z) {
      dst[0] = z.real();
      dst[1] = z.imag();
    };
    const int kx = nr + np;
    for (int j = 0; j < kx; ++j)
      for (int x = 0; x < n; ++x) {
        cplx f = Pix[size_t(ox[size_t(j)]) * n + x];
        if (j < nr) f = cplx(f.real(), 0.0);
        put(c.FX[j][x], f);
        put(c.IX[x][j], (j < nr ? 1.0 : 2.0) * Px[size_t(x) * n + ox[size_t(j)]]);
      }
    for (int q = 0; q < n; ++q)
      for (int y = 0; y < n; ++y) {
        cplx f = Piy[size_t(oy[size_t(q)]) * n + y];
        if (q < nr) f = cplx(f.real(), 0.0);
        put(c.FY[q][y], f);
        put(c.IY[y][q], Py[size_t(y) * n + oy[size_t(q)]]);
        if (q < kx) put(c.IYW[y][q], (q < nr ? 1.0 : 2.0) * Py[size_t(y) * n + oy[size_t(q)]]);
      }
    std::vector<cplx> A(size_t(nt) * nt), Ai;
    int m = 0;
    auto add_mode = [&](cplx theta) {
      for (int r = 0; r < nt; ++r)
        for (int t = 0; t < nt; ++t) A[size_t(r) * nt + t] = mx.T[r][t] + theta * mx.S[r][t];
      if (!stg::cinverse(A, Ai, nt)) return false;
      for (int it = 0; it < nt; ++it)
        for (int t = 0; t < nt; ++t) put(c.M[m][it][t], Ai[size_t(it) * nt + t]);
      ++m;
      return true;
    };
    for (int j = 0; j < nr; ++j)
      for (int q = 0; q < kx; ++q)
        if (!add_mode(thx[size_t(ox[size_t(j)])] + thy[size_t(oy[size_t(q)])])) return false;
    for (int p = 0; p < np; ++p)
      for (int ky = 0; ky < n; ++ky)
        if (!add_mode(thx[size_t(ox[size_t(nr + p)])] + thy[size_t(oy[size_t(ky)])])) return false;
    return true;
  } catch (const std::exception&) {
    return false;
  }
}

// d = 2 dense element block (the fallback of the d = 2 FDM: meshes whose cell
// count is not a multiple of 32, other (n, n_tau)): out = B in for every
// element, hand-written shared-memory-tiled kernel (kernels_precond.cu)
Op dense_op(stg_handle* h, const double* tab, int nt, int npc, int ncells, long long ns) {
  return [h, tab, nt, npc, ncells, ns](const double* in, double* out) {
    if (!stg::precond_eblock_dense(out, in, tab, nt, npc, ncells, ns, h->stream, h->skip))
      throw std::runtime_error("element-block preconditioner launch failed");
    h->launches++;
  };
}

// Factors of fdm2_kernel (kernels_fdm.cu) for the d = 2 element-local block
// L_e = T (x) I + S (x) (V_y (+) V_x): complex eigen-decompositions of V_x
// (its real eigenvectors made real) and V_y, and per kept spatial mode
// theta = thy + thx the temporal inverse (T + theta S)^-1.  nr / np: real x
// eigenvalues and complex-conjugate pairs.  False when an eigen-
// decomposition is inaccurate or a temporal block singular.
bool build_fdm2(const stg::SpatialCoef& sp, const stg::MixCoef& mx, int n, int nt,
                stg::FdmCoef2& c, int& nr, int& np) {
  using stg::cplx;
  try {
    std::vector<cplx> th[2], P[2], Pi[2];
    for (int a = 0; a < 2; ++a) {
      std::vector<double> V(size_t(n) * n);
      for (int i = 0; i < n; ++i)
        for (int k = 0; k < n; ++k) V[size_t(i) * n + k] = sp.V[a][i][k];
      if (!stg::eig_real(V, n, th[a], P[a], Pi[a])) return false;
    }
    // x: real eigenvalues (made-real eigenvectors) first, then one member
    // (Im > 0) of each conjugate pair
    std::vector<int> kept;
    nr = np = 0;
    for (int k = 0; k < n; ++k)
      if (th[0][size_t(k)].imag() == 0.0) {
        cplx big = 0.0;
        for (int r = 0; r < n; ++r)
          if (std::abs(P[0][size_t(r) * n + k]) > std::abs(big)) big = P[0][size_t(r) * n + k];
        const cplx ph = std::conj(big) / std::abs(big);
        for (int r = 0; r < n; ++r)
          P[0][size_t(r) * n + k] = cplx((P[0][size_t(r) * n + k] * ph).real(), 0.0);
        kept.push_back(k);
        ++nr;
      }
    for (int k = 0; k < n; ++k)
      if (th[0][size_t(k)].imag() > 0.0) {
        kept.push_back(k);
        ++np;
      }
    if (nr + 2 * np != n) return false;
    if (!stg::cinverse(P[0], Pi[0], n)) return false;
    double err = 0.0, mxv = 0.0;  // the rephased factorisation still reproduces V_x
    for (int r = 0; r < n; ++r)
      for (int q = 0; q < n; ++q) {
        cplx acc = 0.0;
        for (int k = 0; k < n; ++k)
          acc += P[0][size_t(r) * n + k] * th[0][size_t(k)] * Pi[0][size_t(k) * n + q];
        err = std::max(err, std::abs(acc - sp.V[0][r][q]));
        mxv = std::max(mxv, std::abs(sp.V[0][r][q]));
      }
    if (!(err <= 1e-11 * std::max(mxv, 1e-300))) return false;
    std::memset(&c, 0, sizeof c);
    auto put = [](double* dst, cplx z) {
      dst[0] = z.real();
      dst[1] = z.imag();
    };
    const int kx = nr + np;
    for (int j = 0; j < kx; ++j) {
      const int k = kept[size_t(j)];
      const bool real_mode = j < nr;
      for (int x = 0; x < n; ++x) {
        cplx f = Pi[0][size_t(k) * n + x];
        if (real_mode) f = cplx(f.real(), 0.0);
        put(c.FX[j][x], f);
        put(c.IX[x][j], (real_mode ? 1.0 : 2.0) * P[0][size_t(x) * n + k]);
      }
    }
    for (int r = 0; r < n; ++r)
      for (int q = 0; q < n; ++q) {
        put(c.FY[r][q], Pi[1][size_t(r) * n + q]);
        put(c.IY[r][q], P[1][size_t(r) * n + q]);
      }
    std::vector<cplx> A(size_t(nt) * nt), Ai;
    for (int iy = 0; iy < n; ++iy)
      for (int j = 0; j < kx; ++j) {
        const cplx theta = th[1][size_t(iy)] + th[0][size_t(kept[size_t(j)])];
        for (int r = 0; r < nt; ++r)
          for (int t = 0; t < nt; ++t) A[size_t(r) * nt + t] = mx.T[r][t] + theta * mx.S[r][t];
        if (!stg::cinverse(A, Ai, nt)) return false;
        const int m = iy * kx + j;
        for (int it = 0; it < nt; ++it)
          for (int t = 0; t < nt; ++t) put(c.M[m][it][t], Ai[size_t(it) * nt + t]);
      }
    return true;
  } catch (const std::exception&) {
    return false;
  }
}

// Inverse of the (shared) element block of the d = 1 advection Jacobian with
// temporal mixing (T, S): rows / columns (r, i), (j, q) of the element-local
// block T (x) I + S (x) V.  Uploaded to h->ptab; returns the device pointer.
const double* eblock_table_1d(stg_handle* h, const stg::MixCoef& mx) {
  const int nt = h->nt, n1 = h->n1, nb = nt * n1;
  if (h->etab_valid && std::memcmp(&h->etab_mix, &mx, sizeof mx) == 0) return h->etab.p;
  std::vector<double> B(size_t(nb) * nb);
  for (int r = 0; r < nt; ++r)
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < nt; ++j)
        for (int q = 0; q < n1; ++q)
          B[size_t(r * n1 + i) * nb + size_t(j * n1 + q)] =
              (i == q ? mx.T[r][j] : 0.0) + mx.S[r][j] * h->sp.V[0][i][q];
  const std::vector<double> Bi = stg::inverse(B, nb);
  h->etab.ensure(Bi.size());
  ck(cudaMemcpyAsync(h->etab.p, Bi.data(), sizeof(double) * Bi.size(), cudaMemcpyHostToDevice,
                     h->stream), "H2D");
  ck(cudaStreamSynchronize(h->stream), "sync");
  h->etab_mix = mx;
  h->etab_valid = true;
  return h->etab.p;
}

// Right preconditioner for the Jacobian with temporal mixing (T, S) at the
// linearisation point U (used by the Burgers element blocks only).
// smallest divisor >= 3 of n (n itself when n <= 2 or prime): same-coloured
// cells on the periodic lattice are >= 3 apart (spatial.hpp color_stride)
int color_stride(int n) {
  if (n <= 2) return n;
  for (int m = 3; m < n; ++m)
    if (n % m == 0) return m;
  return n;
}

// element-block Jacobi of a general linear model: K_e by coloured probing of
// the spatial operator (once per handle: linear, time independent), then the
// blocks T (x) I + S (x) K_e inverted on the device (once per mix)
Op general_eblock(stg_handle* h, const stg::MixCoef& mx) {
  const stg::Geometry& g = h->g;
  const int ndl = g.npc * h->r, nt = h->nt, nb = nt * ndl, nc = g.n_cells;
  const long long ns = h->n_sdof;
  if (!h->gK_valid) {
    h->gK.ensure(size_t(nc) * ndl * ndl);
    h->gProbe.ensure(size_t(ns));
    h->genF.ensure(size_t(ns));
    const int sx = color_stride(g.nx), sy = g.dim == 2 ? color_stride(g.ny) : 1;
    stg::GenArgs a{};
    a.c = h->gc;
    a.g = g;
    a.n_in = 1;
    a.X = h->gProbe.p;
    a.F = h->genF.p;
    a.R = nullptr;
    a.err = reinterpret_cast<int*>(h->genFlag.p);
    for (int cy0 = 0; cy0 < sy; ++cy0)
      for (int cx0 = 0; cx0 < sx; ++cx0)
        for (int col = 0; col < ndl; ++col) {
          stg::probe_set(h->gProbe.p, ndl, col, g.nx, g.ny, sx, sy, cx0, cy0, nc, h->stream);
          if (stg::launch_general(a, h->stream) < 0)
            throw std::invalid_argument("no kernel for this (dim, degree, model)");
          stg::probe_extract(h->gK.p, h->genF.p, ndl, col, g.nx, sx, sy, cx0, cy0, nc,
                             h->stream);
          h->launches += 3;
        }
    check_launch(h);
    h->gK_valid = true;
  }
  if (!h->gB_valid || std::memcmp(&h->g_mix, &mx, sizeof mx) != 0) {
    h->gBinv.ensure(size_t(nc) * nb * nb);
    if (!stg::gen_eblock_invert(h->gBinv.p, h->gK.p, mx, nt, ndl, nc, h->stream))
      throw std::invalid_argument("element block too large");
    h->launches++;
    check_launch(h);
    h->g_mix = mx;
    h->gB_valid = true;
  }
  const double* tab = h->gBinv.p;
  return [h, tab, nb, nt, ndl, nc, ns](const double* in, double* out) {
    stg::precond_eblock(out, in, tab, (long long)nb * nb, nt, ndl, nc, ns, h->stream, h->skip);
    h->launches++;
  };
}

Op make_precond(stg_handle* h, int kind, const stg::MixCoef& mx, const double* U) {
  kind = resolve_precond(h, kind);
  if (kind == STG_PRECOND_POLY) kind = poly_base(h);  // the block part (precond_for wraps it)
  // an exact element-block inverse of an advection Jacobian unless a
  // fallback below says otherwise
  h->block_exact = kind == STG_PRECOND_EBLOCK && h->desc.model == STG_MODEL_ADVECTION;
  if (kind == STG_PRECOND_NONE) return Op();
  if (general_model(h->desc.model)) return general_eblock(h, mx);
  const int nt = h->nt, n1 = h->n1, npc = h->g.npc, d = h->desc.dim;
  const long long ns = h->n_sdof;
  if ((kind == STG_PRECOND_TBLOCK || kind == STG_PRECOND_JACOBI) && h->ptab_kind == kind &&
      std::memcmp(&h->ptab_mix, &mx, sizeof mx) == 0) {  // the table of this mix is uploaded
    const double* dt = h->ptab.p;
    return [h, dt, nt, npc, ns](const double* in, double* out) {
      stg::precond_tblock(out, in, dt, nt, npc, ns, h->stream, h->skip);
      h->launches++;
    };
  }
  if (kind == STG_PRECOND_TBLOCK || kind == STG_PRECOND_JACOBI) {
    // block of node class k: T + v_k S with v_k = sum_a V_a(i_a, i_a); the
    // diagonal preconditioner keeps its diagonal, inverted entry by entry
    // with Eigen's DiagonalPreconditioner rule (a zero entry -> 1)
    std::vector<double> tab(size_t(npc) * nt * nt, 0.0), B(size_t(nt) * nt);
    for (int k = 0; k < npc; ++k) {
      const int idx[3] = {k % n1, (k / n1) % n1, k / (n1 * n1)};
      double v = 0.0;
      for (int a = 0; a < d; ++a) v += h->sp.V[a][idx[a]][idx[a]];
      for (int r = 0; r < nt; ++r)
        for (int j = 0; j < nt; ++j) B[size_t(r) * nt + j] = mx.T[r][j] + v * mx.S[r][j];
      if (kind == STG_PRECOND_JACOBI) {
        for (int r = 0; r < nt; ++r) {
          const double dr = B[size_t(r) * nt + r];
          tab[size_t(k) * nt * nt + size_t(r) * nt + r] = dr != 0.0 ? 1.0 / dr : 1.0;
        }
        continue;
      }
      const std::vector<double> Bi = stg::inverse(B, nt);
      std::copy(Bi.begin(), Bi.end(), tab.begin() + long(size_t(k) * nt * nt));
    }
    h->ptab.ensure(tab.size());
    ck(cudaMemcpyAsync(h->ptab.p, tab.data(), sizeof(double) * tab.size(),
                       cudaMemcpyHostToDevice, h->stream), "H2D");
    ck(cudaStreamSynchronize(h->stream), "sync");
    h->ptab_kind = kind;
    h->ptab_mix = mx;
    h->eblock_valid = false;  // (ptab held Burgers blocks)
    const double* dt = h->ptab.p;
    return [h, dt, nt, npc, ns](const double* in, double* out) {
      stg::precond_tblock(out, in, dt, nt, npc, ns, h->stream, h->skip);
      h->launches++;
    };
  }
  if (d == 2 && n1 <= stg::kFdm2MaxN && nt <= stg::kFdm2MaxN) {  // d = 2 FDM, in place
    bool ok = h->fdm2i_valid && std::memcmp(&h->fdm2i_mix, &mx, sizeof mx) == 0;
    if (!ok) {
      auto c = std::make_unique<stg::FdmCoef2i>();
      int nr = 0, np = 0;
      if (build_fdm2i(h->sp, mx, n1, nt, *c, nr, np) && stg::fdm2i_supported(h->g, nt, nr, np)) {
        h->fdm2iM.ensure(sizeof(stg::FdmCoef2i) / sizeof(double));
        ck(cudaMemcpyAsync(h->fdm2iM.p, c.get(), sizeof(stg::FdmCoef2i), cudaMemcpyHostToDevice,
                           h->stream), "H2D");
        ck(cudaStreamSynchronize(h->stream), "sync");
        h->fdm2i_host = std::move(c);
        h->fdm2i_mix = mx;
        h->fdm2i_valid = ok = true;
      }
    }
    if (ok) {
      const stg::FdmCoef2i* c = reinterpret_cast<const stg::FdmCoef2i*>(h->fdm2iM.p);
      const stg::FdmCoef2i* hc = h->fdm2i_host.get();
      return [h, c, hc, nt](const double* in, double* out) {
        if (stg::launch_precond_fdm2i(c, *hc, h->g, nt, in, out, h->stream, h->skip) < 0)
          throw std::runtime_error("element-block preconditioner launch failed");
        h->launches++;
      };
    }
  }
  if (d == 2 && n1 <= stg::kFdm2MaxN && nt <= stg::kFdm2MaxN) {  // d = 2 FDM
    bool ok = h->fdm2_valid && std::memcmp(&h->fdm2_mix, &mx, sizeof mx) == 0;
    if (!ok) {
      auto c = std::make_unique<stg::FdmCoef2>();
      int nr = 0, np = 0;
      if (build_fdm2(h->sp, mx, n1, nt, *c, nr, np) && stg::fdm2_supported(h->g, nt, nr, np)) {
        h->fdm2M.ensure(sizeof(stg::FdmCoef2) / sizeof(double));
        ck(cudaMemcpyAsync(h->fdm2M.p, c.get(), sizeof(stg::FdmCoef2), cudaMemcpyHostToDevice,
                           h->stream), "H2D");
        ck(cudaStreamSynchronize(h->stream), "sync");
        h->fdm2_host = std::move(c);
        h->fdm2_mix = mx;
        h->fdm2_nr = nr;
        h->fdm2_np = np;
        h->fdm2_valid = ok = true;
      }
    }
    if (ok) {
      const stg::FdmCoef2* c = reinterpret_cast<const stg::FdmCoef2*>(h->fdm2M.p);
      const stg::FdmCoef2* hc = h->fdm2_host.get();
      const int nr = h->fdm2_nr, np = h->fdm2_np;
      return [h, c, hc, nt, nr, np](const double* in, double* out) {
        if (stg::launch_precond_fdm2(c, *hc, h->g, nt, nr, np, in, out, h->stream, h->skip) < 0)
          throw std::runtime_error("element-block preconditioner launch failed");
        h->launches++;
      };
    }
  }
  if (d == 2) {  // one shared dense element block (advection)
    const int nbd = nt * npc;
    // the block depends only on (T, S) and the mesh: reuse the uploaded
    // inverse across Newton iterations and solves with the same mix
    if (h->dense_valid && std::memcmp(&h->dense_mix, &mx, sizeof mx) == 0) {
      const double* tab = h->dtab.p;
      const int ncells = h->g.n_cells;
      return dense_op(h, tab, nt, npc, ncells, ns);
    }
    std::vector<double> B(size_t(nbd) * nbd, 0.0);
    for (int r = 0; r < nt; ++r)
      for (int node = 0; node < npc; ++node) {
        const int iy = node / n1, ix = node % n1;
        for (int j = 0; j < nt; ++j)
          for (int node2 = 0; node2 < npc; ++node2) {
            const int jy = node2 / n1, jx = node2 % n1;
            const double K = (iy == jy ? h->sp.V[0][ix][jx] : 0.0) +
                             (ix == jx ? h->sp.V[1][iy][jy] : 0.0);
            B[size_t(r * npc + node) * nbd + size_t(j * npc + node2)] =
                (node == node2 ? mx.T[r][j] : 0.0) + mx.S[r][j] * K;
          }
      }
    const std::vector<double> Bi = stg::inverse(B, nbd);
    h->dtab.ensure(Bi.size());
    ck(cudaMemcpyAsync(h->dtab.p, Bi.data(), sizeof(double) * Bi.size(), cudaMemcpyHostToDevice,
                       h->stream), "H2D");
    ck(cudaStreamSynchronize(h->stream), "sync");
    h->dense_mix = mx;
    h->dense_valid = true;
    const double* tab = h->dtab.p;
    const int ncells = h->g.n_cells;
    return dense_op(h, tab, nt, npc, ncells, ns);
  }
  if (d == 3 && stg::fdm3_supported(h->g, nt)) {  // fast diagonalisation, direct t solve
    bool ok = h->fdm3_valid && std::memcmp(&h->fdm3_mix, &mx, sizeof mx) == 0;
    if (!ok) {
      auto c = std::make_unique<stg::FdmCoef3>();
      if (build_fdm3(h->sp, mx, *c)) {
        h->fdm3M.ensure(sizeof(stg::FdmCoef3) / sizeof(double));
        ck(cudaMemcpyAsync(h->fdm3M.p, c.get(), sizeof(stg::FdmCoef3), cudaMemcpyHostToDevice,
                           h->stream), "H2D");
        ck(cudaStreamSynchronize(h->stream), "sync");
        h->fdm3_mix = mx;
        h->fdm3_host = std::move(c);
        h->fdm3_valid = ok = true;
      }
    }
    if (ok) {
      const stg::FdmCoef3* c = reinterpret_cast<const stg::FdmCoef3*>(h->fdm3M.p);
      const stg::FdmCoef3* hc = h->fdm3_host.get();
      return [h, c, hc](const double* in, double* out) {
        if (stg::launch_precond_fdm3(c, *hc, h->g, in, out, h->stream, h->skip) < 0)
          throw std::runtime_error("element-block preconditioner launch failed");
        h->launches++;
      };
    }
    Op tb = make_precond(h, STG_PRECOND_TBLOCK, mx, U);  // spectrum not of the FDM form
    h->block_exact = false;
    return tb;
  }
  if (d == 3) {  // element-block Jacobi by fast diagonalisation
    stg::FdmCoef c;
    bool ok = h->fdm_valid && std::memcmp(&h->fdm_mix, &mx, sizeof mx) == 0;
    if (ok) {
      c = h->fdm;
    } else if (build_fdm(h->sp, mx, c)) {
      h->fdm = c;
      h->fdm_mix = mx;
      h->fdm_valid = ok = true;
    }
    if (ok)
      return [h, c](const double* in, double* out) {
        if (stg::launch_precond_fdm(c, h->g, in, out, h->stream, h->skip) < 0)
          throw std::runtime_error("element-block preconditioner launch failed");
        h->launches++;
      };
    if (h->desc.model != STG_MODEL_ADVECTION)
      throw std::invalid_argument("element-block Jacobi: no factorisation");
    Op tb = make_precond(h, STG_PRECOND_TBLOCK, mx, U);  // spectrum not of the FDM form
    h->block_exact = false;
    return tb;
  }
  // element-block Jacobi, d = 1: block (r,i),(j,q) of the element-local Jacobian
  const int nb = nt * n1;
  const int ncells = h->g.n_cells;
  long long bstride = 0;
  const double* tab = nullptr;
  if (h->desc.model == STG_MODEL_ADVECTION) {
    tab = eblock_table_1d(h, mx);
  } else {
    stg::SlabArgs a{};
    a.sp = h->sp;
    a.mx = mx;
    a.g = h->g;
    a.n_in = nt;
    a.n_out = nt;
    if (!stg::eblock_f32_supported(nt, n1))
      throw std::invalid_argument("element-block Jacobi (Burgers): n_tau * (N+1) <= 16 and even");
    static const bool rebuild = std::getenv("STG_PRECOND_REBUILD") != nullptr;
    const bool sweep = kind == STG_PRECOND_SWEEP;
    float* fb = reinterpret_cast<float*>(h->ptab.p);
    if (!h->eblock_valid || rebuild || (sweep && !h->eblock_sweep) ||
        std::memcmp(&h->eblock_mix, &mx, sizeof mx) != 0) {
      h->eblock_mix = mx;
      h->eblock_age = 0;
      h->eblock_built_now = true;
      h->ptab_kind = -1;  // ptab now holds Burgers blocks
      h->ptab.ensure((size_t(ncells) * nb * nb + 1) / 2);  // fp32 blocks
      fb = reinterpret_cast<float*>(h->ptab.p);
      float* G = nullptr;
      if (sweep) {
        h->sweepG.ensure((size_t(ncells) * nb * nt + 1) / 2);
        G = reinterpret_cast<float*>(h->sweepG.p);
      }
      if (!stg::build_burgers_eblock(fb, G, U, a, h->stream))
        throw std::invalid_argument("element-block Jacobi: degree <= 3 for Burgers");
      h->launches++;
      check_launch(h);
      h->eblock_valid = true;
      h->eblock_sweep = sweep;
    }
    h->eblock_in_use = true;
    if (sweep) {
      h->sweepW.ensure(stg::sweep_work_doubles(nt, ncells, n1));
      const float* G = reinterpret_cast<const float*>(h->sweepG.p);
      double* wk = h->sweepW.p;
      // the sweep also reduces <out, out> into the slot the FD Jacobian
      // action reads its step from (fd_jvp skips its own dot for out)
      return [h, fb, G, wk, nt, n1, ncells, ns](const double* in, double* out) {
        stg::precond_sweep(out, in, fb, G, wk, nt, n1, ncells, ns, h->stream, h->skip,
                           h->partial.p, h->small.p + kVVSlot);
        h->vv_of = out;
        h->launches += 2;
      };
    }
    return [h, fb, nt, n1, ncells, ns](const double* in, double* out) {
      stg::precond_eblock_f32(out, in, fb, nt, n1, ncells, ns, h->stream, h->skip);
      h->launches++;
    };
  }
  return [h, tab, bstride, nt, n1, ncells, ns](const double* in, double* out) {
    stg::precond_eblock(out, in, tab, bstride, nt, n1, ncells, ns, h->stream, h->skip);
    h->launches++;
  };
}

// The right preconditioner of a solve with Jacobian action A: make_precond's
// block preconditioner P0, and for STG_PRECOND_POLY the truncated Neumann
// series of (P0^-1 A)^-1 P0^-1 around it:
//   z = P0^-1 r,  y_0 = z,  y_{i+1} = z + y_i - P0^-1 A y_i   (i < m).
// A fixed linear operator, so GMRES stays exact; every launch honours the
// handle's skip flag (speculative Arnoldi steps).
Op precond_for(stg_handle* h, int kind, const stg::MixCoef& mx, const double* U, const Op& A) {
  const int rk = resolve_precond(h, kind);
  Op P0 = make_precond(h, rk, mx, U);
  const int m = poly_terms();
  if (rk != STG_PRECOND_POLY || !P0 || m == 0) return P0;
  const long long n = h->n_dof;
  h->polyZ.ensure(size_t(n));
  h->polyW.ensure(size_t(n));
  double* z = h->polyZ.p;
  double* w = h->polyW.p;
  // P0 the exact element-block inverse of constant-velocity advection (no
  // neighbour coupling inside a block): y_{i+1} = P0^-1 (r - L y_i) with the
  // neighbour couplings L = J - P0 applied directly (one pass instead of a
  // Jacobian action, a block apply and an axpy per term)
  static const bool generic = std::getenv("STG_POLY_GENERIC") != nullptr;
  // d = 3 with the fdm3 blocks and a diagonal temporal mix: the neighbour
  // couplings are folded into the block apply (fdm3_kernel with FdmOffdiag),
  // y_{i+1} = P0^-1 (r - L y_i) in one pass, ping-ponging between z and y
  bool s_diag = true;
  for (int t = 0; t < h->nt; ++t)
    for (int j = 0; j < h->nt; ++j)
      if (t != j && mx.S[t][j] != 0.0) s_diag = false;
  static const bool no_fused = std::getenv("STG_POLY_UNFUSED") != nullptr;
  if (h->block_exact && h->desc.dim == 3 && stg::fdm3_supported(h->g, h->nt) && h->fdm3_valid &&
      std::memcmp(&h->fdm3_mix, &mx, sizeof mx) == 0 && s_diag && !generic && !no_fused) {
    stg::FdmOffdiag od{};
    for (int t = 0; t < 4; ++t) od.S[t] = mx.S[t][t];
    for (int a = 0; a < 3; ++a) {
      od.cL[a] = h->sp.cL[a];
      od.cR[a] = h->sp.cR[a];
    }
    const stg::FdmCoef3* c = reinterpret_cast<const stg::FdmCoef3*>(h->fdm3M.p);
    const stg::FdmCoef3* hc = h->fdm3_host.get();
    // intermediate terms exist only as their face traces (compact, ping-pong
    // in z): the first apply and every coupled step but the last write the
    // traces alone, the last writes the result
    const long long nt3 = stg::fdm_trace_doubles(h->g, h->nt);
    h->polyZ.ensure(size_t(2 * nt3));
    double* tr[2] = {h->polyZ.p, h->polyZ.p + nt3};
    return [h, m, od, c, hc, tr](const double* r, double* y) {
      stg::FdmOffdiag o = od;
      o.tr_in = nullptr;
      o.tr_out = tr[0];
      o.full_out = 0;
      if (stg::launch_precond_fdm3(c, *hc, h->g, r, y, h->stream, h->skip, &o) < 0)
        throw std::runtime_error("element-block preconditioner launch failed");
      h->launches++;
      for (int i = 0; i < m; ++i) {
        const bool last = i + 1 == m;
        o.tr_in = tr[i & 1];
        o.tr_out = last ? nullptr : tr[(i + 1) & 1];
        o.full_out = last ? 1 : 0;
        if (stg::launch_precond_fdm3(c, *hc, h->g, r, y, h->stream, h->skip, &o) < 0)
          throw std::runtime_error("element-block preconditioner launch failed");
        h->launches++;
      }
    };
  }
  // d = 2 with the in-place FDM blocks: the same with fdm2i_kernel
  if (h->block_exact && h->desc.dim == 2 && h->fdm2i_valid &&
      std::memcmp(&h->fdm2i_mix, &mx, sizeof mx) == 0 && s_diag && !generic && !no_fused &&
      h->nt <= stg::kFdm2MaxN) {
    stg::FdmOffdiag2 od{};
    for (int t = 0; t < h->nt; ++t) od.S[t] = mx.S[t][t];
    for (int a = 0; a < 2; ++a) {
      od.cL[a] = h->sp.cL[a];
      od.cR[a] = h->sp.cR[a];
    }
    const stg::FdmCoef2i* c = reinterpret_cast<const stg::FdmCoef2i*>(h->fdm2iM.p);
    const stg::FdmCoef2i* hc = h->fdm2i_host.get();
    const long long nt2 = stg::fdm2_trace_doubles(h->g, h->nt);
    h->polyZ.ensure(size_t(2 * nt2));
    double* tr[2] = {h->polyZ.p, h->polyZ.p + nt2};
    const int nt = h->nt;
    return [h, m, od, c, hc, tr, nt](const double* r, double* y) {
      stg::FdmOffdiag2 o = od;
      o.tr_in = nullptr;
      o.tr_out = tr[0];
      o.full_out = 0;
      if (stg::launch_precond_fdm2i(c, *hc, h->g, nt, r, y, h->stream, h->skip, &o) < 0)
        throw std::runtime_error("element-block preconditioner launch failed");
      h->launches++;
      for (int i = 0; i < m; ++i) {
        const bool last = i + 1 == m;
        o.tr_in = tr[i & 1];
        o.tr_out = last ? nullptr : tr[(i + 1) & 1];
        o.full_out = last ? 1 : 0;
        if (stg::launch_precond_fdm2i(c, *hc, h->g, nt, r, y, h->stream, h->skip, &o) < 0)
          throw std::runtime_error("element-block preconditioner launch failed");
        h->launches++;
      }
    };
  }
  if (h->block_exact && stg::offdiag_supported(h->g, h->nt) && !generic) {
    const stg::MixCoef mj = mx;
    return [h, P0, m, mj, z](const double* r, double* y) {
      P0(r, y);
      for (int i = 0; i < m; ++i) {
        stg::offdiag_residual(z, r, y, h->sp, mj, h->g, h->nt, h->stream, h->skip);
        h->launches++;
        P0(z, y);
      }
    };
  }
  h->polyQ.ensure(size_t(n));
  double* q = h->polyQ.p;
  return [h, A, P0, m, n, z, w, q](const double* r, double* y) {
    P0(r, z);
    const double* x = z;
    for (int i = 0; i < m; ++i) {
      A(x, w);
      P0(w, q);
      stg::vec_poly_step(y, z, x, q, n, h->stream, h->skip);
      h->launches++;
      x = y;
    }
  };
}

stg_newton_config effective_cfg(const stg_newton_config* cfg) {
  stg_newton_config c;
  stg_newton_config_default(&c);
  if (cfg) c = *cfg;
  if (c.linear != STG_LINEAR_AUTO && c.linear != STG_LINEAR_GMRES)
    throw std::invalid_argument("linear method: only GMRES runs on the device");
  if (c.max_iter < 0) throw std::invalid_argument("max_iter >= 0");
  return c;
}

// Whole Newton-GMRES solve in one single-CTA kernel (kernels_small.cu) for
// small d = 1 advection problems (c1); false when not applicable.  Same
// Newton / GMRES control flow, tolerances and error behaviour as the
// host-driven path.
bool small_solve(stg_handle* h, bool rk, const stg::MixCoef& mres, const stg::MixCoef& mjac,
                 const stg::MixCoef& mnext, const double* W, const stg_newton_config& cfg,
                 double* U, double* u_next, stg_solve_info* info, const std::string& ctx) {
  static const bool off = std::getenv("STG_NO_FUSED_SMALL") != nullptr;
  if (off || h->desc.model != STG_MODEL_ADVECTION || h->kernel_pref != STG_KERNEL_AUTO ||
      !stg::small_solve_supported(h->g, h->nt, h->desc.model, cfg.gmres_restart))
    return false;
  const int kind = resolve_precond(h, cfg.precond);
  if (kind != STG_PRECOND_NONE && kind != STG_PRECOND_EBLOCK) return false;
  ensure_workspace(h);
  stg::SmallSolveArgs a{};
  a.sp = h->sp;
  a.mx_res = mres;
  a.mx_jac = mjac;
  a.mx_next = mnext;
  a.n = int(h->n_dof);
  a.K = h->g.n_cells;
  a.nt = h->nt;
  a.n1 = h->n1;
  a.ns = h->n_sdof;
  a.ld = round_up(h->n_dof, 32);
  a.restart = cfg.gmres_restart;
  a.max_it = cfg.gmres_max_it;
  a.max_iter = cfg.max_iter;
  a.rk = rk ? 1 : 0;
  a.tol = cfg.gmres_tol;
  a.abs_tol = cfg.abs_tol;
  a.rel_tol = cfg.rel_tol;
  a.W = W;
  a.B = kind == STG_PRECOND_EBLOCK ? eblock_table_1d(h, mjac) : nullptr;
  h->basis.ensure(size_t(a.ld) * (a.restart + 1));
  a.V = h->basis.p;
  a.U_out = U;
  a.u_next = u_next;
  const size_t out_doubles = (sizeof(stg::SmallSolveOut) + 7) / 8;
  h->small_out.ensure(out_doubles);
  a.out = reinterpret_cast<stg::SmallSolveOut*>(h->small_out.p);
  if (stg::launch_small_solve(a, h->stream) < 0) return false;
  h->launches++;
  check_launch(h);
  stg::SmallSolveOut* o = reinterpret_cast<stg::SmallSolveOut*>(h->pinned + 512);
  ck(cudaMemcpyAsync(o, a.out, sizeof(stg::SmallSolveOut), cudaMemcpyDeviceToHost, h->stream),
     "memcpy");
  ck(cudaStreamSynchronize(h->stream), "sync");
  NewtonOut out;
  out.iterations = o->newton_iterations;
  out.linear_iterations = o->linear_iterations;
  out.final_residual = o->final_residual;
  out.history.assign(o->history, o->history + o->n_history);
  if (o->status == 1) {
    fill_info(info, out);
    throw NonconvergenceError(ctx + ": newton_solve: no convergence in " +
                                  std::to_string(cfg.max_iter) + " iterations, residual " +
                                  fmt_short(o->final_residual),
                              out.history, out.linear_iterations);
  }
  if (o->status == 2)
    throw std::runtime_error("linear_solve: GMRES did not converge, error " +
                             fmt_short(o->gmres_rel));
  fill_info(info, out);
  return true;
}

// A new slab / stage solve: the lagged Burgers element blocks (and sweep
// couplings) of the previous steps stay in use for STG_PRECOND_LAG_STEPS
// steps (default 4; 1: rebuilt every step).  The state moves by O(dt) per
// step, so the blocks barely change; GMRES absorbs the difference (c3: the
// same 11 steps per slab) and the 0.15 ms build runs once per 4 slabs.
void new_step(stg_handle* h) {
  static const int lag = [] {
    const char* e = std::getenv("STG_PRECOND_LAG_STEPS");
    return e ? std::max(1, std::atoi(e)) : 4;
  }();
  if (++h->eblock_age >= lag) h->eblock_valid = false;
}

// The initial guess 1 (x) u of a slab / stage solve.  For linear advection on
// the fast 3-D path it is not written: the first residual reads u through
// zero-stride tensor maps and the first Newton update writes
// U = 1 (x) u + correction (apply, gmres).  Otherwise, and whenever anything
// else needs U, it is broadcast into U.  The destructor writes it out if it
// is still pending (Newton converged at once, or an exception: U must hold
// the last iterate, newton.hpp:40-48).
struct LazyGuess {
  stg_handle* h;
  LazyGuess(stg_handle* hh, double* U, const double* u) : h(hh) {
    h->lazy_dst = U;
    h->lazy_src = u;
    const bool lazy = h->desc.model == STG_MODEL_ADVECTION && h->g.dim >= 2 &&
                      stg::slab_fast_bcast_ok();
    if (!lazy) materialise(h);
  }
  ~LazyGuess() {
    try {
      materialise(h);
    } catch (...) {
    }
    h->lazy_dst = nullptr;
  }
  LazyGuess(const LazyGuess&) = delete;
  LazyGuess& operator=(const LazyGuess&) = delete;
};

void do_stdg_step(stg_handle* h, double t_n, double dt, const double* u_n,
                  const stg_newton_config* cfgp, double* U, double* u_next,
                  stg_solve_info* info) {
  (void)t_n;  // the advection / Burgers fluxes are time independent
  if (!(dt > 0)) throw std::invalid_argument("stdg_step: dt > 0 required");
  const stg_newton_config cfg = effective_cfg(cfgp);
  const long long n = h->n_dof;
  if (small_solve(h, false, st_mix(h, dt, true), st_mix(h, dt, false), zero_mix(), u_n, cfg, U,
                  u_next, info,
                  "stdg_step element at t=" + fmt_short(t_n) + ", dt=" + fmt_short(dt)))
    return;
  new_step(h);
  // guess 1 (x) u_n (stdg.hpp:131)
  LazyGuess guess(h, U, u_n);
  const double eps = cfg.fd_eps;
  NewtonOut o;
  try {
    o = newton(
        h, [&](const double* X, double* R) { st_residual(h, dt, u_n, X, R); },
        [&](const double* X) -> LinSys {
          LinSys L;
          const double un2 = fd_norm(h, eps, X, n);
          L.A = [h, dt, X, eps, un2](const double* v, double* Jv) {
            st_jvp(h, dt, X, v, Jv, eps, un2);
          };
          L.P = precond_for(h, cfg.precond, st_mix(h, dt, false), X, L.A);
          return L;
        },
        U, n, cfg);
  } catch (const NonconvergenceError& e) {
    // stdg.hpp:132-137: rethrown with the slab context; U holds the last
    // iterate, info the history (newton.hpp:40-48)
    fill_info(info, partial_out(e));
    throw NonconvergenceError("stdg_step element at t=" + fmt_short(t_n) + ", dt=" + fmt_short(dt) +
                                  ": " + e.what(),
                              e.history, e.linear_iterations);
  }
  materialise(h);  // (Newton converged at the initial guess)
  if (u_next) {
    stg::vec_copy(u_next, U + (h->nt - 1) * h->n_sdof, h->n_sdof, h->stream);
    h->launches++;
  }
  fill_info(info, o);
}

void do_rk_step(stg_handle* h, int form, double t, double dt, const double* u,
                const stg_newton_config* cfgp, double* U, double* u_next, stg_solve_info* info) {
  if (!(dt > 0)) throw std::invalid_argument("rk_step: dt > 0 required");
  if (form != STG_FORM_A && form != STG_FORM_A_INV) throw std::invalid_argument("bad form");
  const stg_newton_config cfg = effective_cfg(cfgp);
  const long long n = h->n_dof;
  {
    stg::MixCoef mn = zero_mix();  // u_next = u + dt sum_j b_j F(U_j)  (lodg.hpp:142-145)
    for (int j = 0; j < h->nt; ++j) mn.S[0][j] = dt * h->tab.b[size_t(j)];
    mn.c[0] = 1.0;
    if (small_solve(h, true, stage_mix(h, form, dt, true), stage_mix(h, form, dt, false), mn, u,
                    cfg, U, u_next, info, "rk_step at t=" + fmt_short(t) + ", dt=" + fmt_short(dt)))
      return;
  }
  new_step(h);
  // guess 1 (x) u (lodg.hpp:131)
  LazyGuess guess(h, U, u);
  const double eps = cfg.fd_eps;
  NewtonOut o;
  try {
    o = newton(
        h, [&](const double* X, double* R) { stage_residual(h, form, dt, u, X, R); },
        [&](const double* X) -> LinSys {
          LinSys L;
          const double un2 = fd_norm(h, eps, X, n);
          L.A = [h, form, dt, X, eps, un2](const double* v, double* Jv) {
            stage_jvp(h, form, dt, X, v, Jv, eps, un2);
          };
          L.P = precond_for(h, cfg.precond, stage_mix(h, form, dt, false), X, L.A);
          return L;
        },
        U, n, cfg);
  } catch (const NonconvergenceError& e) {
    fill_info(info, partial_out(e));  // lodg.hpp:132-137; U holds the last iterate
    throw NonconvergenceError("rk_step at t=" + fmt_short(t) + ", dt=" + fmt_short(dt) + ": " +
                                  e.what(),
                              e.history, e.linear_iterations);
  }
  materialise(h);  // (Newton converged at the initial guess)
  if (u_next) {
    // u_next = u + dt sum_j b_j F(U_j)  (lodg.hpp:142-145)
    stg::MixCoef m = zero_mix();
    for (int j = 0; j < h->nt; ++j) m.S[0][j] = dt * h->tab.b[size_t(j)];
    m.c[0] = 1.0;
    apply(h, m, h->nt, 1, U, nullptr, u, u_next, false, true);
  }
  fill_info(info, o);
}

template <class F>
int guarded(stg_handle* h, F&& f) {
  std::string* err = h ? &h->err : &g_create_error;
  // a failed call leaves no deferred admissibility flag behind
  auto clear = [h] {
    if (h && h->adm_pending) {
      h->adm_pending = false;
      cudaMemsetAsync(h->genFlag.p, 0, sizeof(int), h->stream);
    }
  };
  if (h) h->vv_of = nullptr;  // no <v, v> carries over between calls
  try {
    f();
    if (h) h->vv_of = nullptr;
    return STG_OK;
  } catch (const NonconvergenceError& e) {
    clear();
    *err = e.what();
    return STG_ERR_NONCONVERGENCE;
  } catch (const CudaError& e) {
    clear();
    *err = e.what();
    return STG_ERR_CUDA;
  } catch (const AdmissibilityError& e) {
    clear();
    *err = e.what();
    return STG_ERR_ADMISSIBILITY;
  } catch (const std::invalid_argument& e) {
    clear();
    *err = e.what();
    return STG_ERR_INVALID;
  } catch (const std::exception& e) {
    clear();
    *err = e.what();
    return STG_ERR_RUNTIME;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string(what) + ": null pointer");
}

// march n_steps with `step(t_k, dt, u_k, U_k, u_{k+1}, info_k)` on the device
template <class Step>
void integrate_impl(stg_handle* h, double t0, const double* u0, double t_end, int n_steps,
                    double* u_final, double* states, double* U_all, stg_solve_info* info,
                    const char* who, Step&& step) {
  if (n_steps < 1) throw std::invalid_argument(std::string(who) + ": n_steps >= 1 required");
  const long long ns = h->n_sdof, nd = h->n_dof;
  const double dt = (t_end - t0) / n_steps;
  if (!(dt > 0)) throw std::invalid_argument(std::string(who) + ": t_end > t0 required");
  h->Ustage.ensure(size_t(nd));
  h->march.ensure(size_t(2 * ns));  // ping-pong states when `states` is not given
  if (states) {
    ck(cudaMemcpyAsync(states, u0, sizeof(double) * ns, cudaMemcpyDeviceToDevice, h->stream),
       "memcpy");
  }
  const double* cur = u0;
  stg_solve_info acc{};
  for (int k = 0; k < n_steps; ++k) {
    const double tk = t0 + (t_end - t0) * k / n_steps;  // stdg.hpp:160-161
    double* next = states ? states + (k + 1) * ns
                          : (k + 1 == n_steps ? u_final : h->march.p + (k % 2) * ns);
    double* Uk = U_all ? U_all + (long long)k * nd : h->Ustage.p;
    stg_solve_info ik{};
    try {
      step(tk, dt, cur, Uk, next, &ik);
    } catch (const NonconvergenceError&) {
      // totals so far plus the failing step's partial record (its last
      // iterate is in Uk)
      if (info) {
        *info = ik;
        info->newton_iterations += acc.newton_iterations;
        info->linear_iterations += acc.linear_iterations;
        info->failed_step = k;
      }
      throw;
    }
    acc.newton_iterations += ik.newton_iterations;
    acc.linear_iterations += ik.linear_iterations;
    acc.final_residual = ik.final_residual;
    acc.n_history = ik.n_history;
    std::memcpy(acc.residual_history, ik.residual_history, sizeof acc.residual_history);
    cur = next;
  }
  if (states && u_final)
    ck(cudaMemcpyAsync(u_final, states + (long long)n_steps * ns, sizeof(double) * ns,
                       cudaMemcpyDeviceToDevice, h->stream), "memcpy");
  acc.failed_step = -1;
  if (info) *info = acc;
}
}  // namespace

extern "C" {

void stg_newton_config_default(stg_newton_config* c) {
  if (!c) return;
  c->abs_tol = 1e-12;
  c->rel_tol = 1e-12;
  c->max_iter = 50;
  c->linear = STG_LINEAR_AUTO;
  c->gmres_restart = 30;
  c->gmres_tol = 1e-12;
  c->gmres_max_it = 1000;
  c->fd_eps = 0.0;
  c->precond = STG_PRECOND_AUTO;
}

const char* stg_last_error(const stg_handle* h) {
  return h ? h->err.c_str() : g_create_error.c_str();
}

int stg_create(const stg_desc* desc, stg_handle** out) {
  return guarded(nullptr, [&] {
    need(out, "stg_create");
    *out = nullptr;
    validate_desc(desc);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw CudaError("stg_create: no CUDA device (there is no CPU fallback)");
    }
    auto h = std::make_unique<stg_handle>();
    h->desc = *desc;
    build_constants(h.get());
    ensure_workspace(h.get());
    if (general_model(desc->model)) {
      h->genFlag.ensure(1);
      ck(cudaMemset(h->genFlag.p, 0, sizeof(double)), "cudaMemset");
    }
    *out = h.release();
  });
}

void stg_destroy(stg_handle* h) { delete h; }

int stg_set_stream(stg_handle* h, void* s) {
  return guarded(h, [&] {
    need(h, "stg_set_stream");
    h->stream = static_cast<cudaStream_t>(s);
  });
}

int stg_set_kernel(stg_handle* h, int k) {
  return guarded(h, [&] {
    need(h, "stg_set_kernel");
    if (k < STG_KERNEL_AUTO || k > STG_KERNEL_FAST) throw std::invalid_argument("bad kernel id");
    h->kernel_pref = k;
  });
}

int stg_sizes(const stg_handle* h, long long* n_sdof, long long* n_dof) {
  if (!h) return STG_ERR_INVALID;
  if (n_sdof) *n_sdof = h->n_sdof;
  if (n_dof) *n_dof = h->n_dof;
  return STG_OK;
}

int stg_constants(const stg_handle* h, double* nodes, double* weights, double* d_tau) {
  if (!h) return STG_ERR_INVALID;
  if (nodes) std::memcpy(nodes, h->rule.x.data(), sizeof(double) * h->n1);
  if (weights) std::memcpy(weights, h->rule.w.data(), sizeof(double) * h->n1);
  if (d_tau) std::memcpy(d_tau, h->Dt.data(), sizeof(double) * h->nt * h->nt);
  return STG_OK;
}

long long stg_kernel_launches(const stg_handle* h) { return h ? h->launches : 0; }

int stg_device_alloc(long long n, double** out) {
  return guarded(nullptr, [&] {
    need(out, "stg_device_alloc");
    if (n < 0) throw std::invalid_argument("stg_device_alloc: n >= 0");
    *out = nullptr;
    if (n > 0) ck(cudaMalloc(out, size_t(n) * sizeof(double)), "cudaMalloc");
  });
}

int stg_device_free(double* p) {
  return guarded(nullptr, [&] {
    if (p) ck(cudaFree(p), "cudaFree");
  });
}

int stg_host_alloc(long long n, double** out) {
  return guarded(nullptr, [&] {
    need(out, "stg_host_alloc");
    if (n < 0) throw std::invalid_argument("stg_host_alloc: n >= 0");
    *out = nullptr;
    if (n > 0)
      ck(cudaHostAlloc(reinterpret_cast<void**>(out), size_t(n) * sizeof(double),
                       cudaHostAllocPortable), "cudaHostAlloc");
  });
}

int stg_host_free(double* p) {
  return guarded(nullptr, [&] {
    if (p) ck(cudaFreeHost(p), "cudaFreeHost");
  });
}

namespace {
// stg_memcpy between pageable host memory and the device: a process-wide ring
// of four 8 MiB page-locked slots on the legacy default stream (the ordering
// cudaMemcpy has); the worker threads (hostcopy.hpp) fill or drain one slot
// while the copy engine moves the others.
void memcpy_staged(double* dst, const double* src, size_t n, bool h2d) {
  constexpr int kSlots = 4;
  constexpr size_t kSlot = kStageChunk;
  static std::mutex mu;
  static double* slot[kSlots] = {};
  std::lock_guard<std::mutex> lk(mu);
  for (double*& p : slot)
    if (!p)
      ck(cudaHostAlloc(reinterpret_cast<void**>(&p), kSlot * sizeof(double), cudaHostAllocPortable),
         "cudaHostAlloc");
  cudaEvent_t ev[kSlots] = {};
  struct Guard {
    cudaEvent_t* e;
    ~Guard() {
      for (int i = 0; i < kSlots; ++i)
        if (e[i]) cudaEventDestroy(e[i]);
    }
  } guard{ev};
  for (cudaEvent_t& e : ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  stg::HostCopyPool& pool = stg::HostCopyPool::get();
  const size_t nchunk = (n + kSlot - 1) / kSlot;
  auto cnt_of = [&](size_t i) { return std::min(kSlot, n - i * kSlot); };
  if (h2d) {
    for (size_t i = 0; i < nchunk; ++i) {
      const int sl = int(i % kSlots);
      if (i >= size_t(kSlots)) ck(cudaEventSynchronize(ev[sl]), "sync");  // slot drained
      const stg::CopyItem it{slot[sl], src + i * kSlot, cnt_of(i) * sizeof(double)};
      pool.par_copy(&it, 1);
      ck(cudaMemcpyAsync(dst + i * kSlot, slot[sl], cnt_of(i) * sizeof(double),
                         cudaMemcpyHostToDevice, cudaStreamLegacy), "H2D");
      ck(cudaEventRecord(ev[sl], cudaStreamLegacy), "event");
    }
    ck(cudaStreamSynchronize(cudaStreamLegacy), "sync");
    return;
  }
  auto issue = [&](size_t i) {
    const int sl = int(i % kSlots);
    ck(cudaMemcpyAsync(slot[sl], src + i * kSlot, cnt_of(i) * sizeof(double),
                       cudaMemcpyDeviceToHost, cudaStreamLegacy), "D2H");
    ck(cudaEventRecord(ev[sl], cudaStreamLegacy), "event");
  };
  for (size_t i = 0; i < std::min(nchunk, size_t(kSlots)); ++i) issue(i);
  for (size_t i = 0; i < nchunk; ++i) {
    const int sl = int(i % kSlots);
    ck(cudaEventSynchronize(ev[sl]), "sync");
    const stg::CopyItem it{dst + i * kSlot, slot[sl], cnt_of(i) * sizeof(double)};
    pool.par_copy(&it, 1);
    if (i + kSlots < nchunk) issue(i + kSlots);
  }
}
}  // namespace

int stg_memcpy(double* dst, const double* src, long long n, int dir) {
  return guarded(nullptr, [&] {
    if (n < 0 || dir < 0 || dir > 2) throw std::invalid_argument("stg_memcpy: bad arguments");
    if (n == 0) return;
    need(dst, "dst");
    need(src, "src");
    static const bool no_staging = std::getenv("STG_HOST_NO_STAGING") != nullptr;
    if (dir < 2 && !no_staging && size_t(n) * sizeof(double) >= (size_t(1) << 21) &&
        pageable(dir == 0 ? static_cast<const void*>(src) : static_cast<const void*>(dst))) {
      memcpy_staged(dst, src, size_t(n), dir == 0);
      return;
    }
    const cudaMemcpyKind k = dir == 0   ? cudaMemcpyHostToDevice
                             : dir == 1 ? cudaMemcpyDeviceToHost
                                        : cudaMemcpyDeviceToDevice;
    ck(cudaMemcpy(dst, src, size_t(n) * sizeof(double), k), "cudaMemcpy");
  });
}

int stg_device_synchronize(void) {
  return guarded(nullptr, [&] { ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize"); });
}

int stg_lgl_rule(int n, double* nodes, double* weights) {
  return guarded(nullptr, [&] {
    const stg::LglRule r = stg::lgl(n);
    if (nodes) std::memcpy(nodes, r.x.data(), sizeof(double) * n);
    if (weights) std::memcpy(weights, r.w.data(), sizeof(double) * n);
  });
}

int stg_diff_matrix(int n, double* D) {
  return guarded(nullptr, [&] {
    need(D, "D");
    const std::vector<double> M = stg::diff_matrix(stg::lgl(n));
    std::memcpy(D, M.data(), sizeof(double) * M.size());
  });
}

int stg_lobatto_tableau(int s, double* A, double* b, double* c) {
  return guarded(nullptr, [&] {
    const stg::Tableau t = stg::lobatto(s);
    if (A) std::memcpy(A, t.A.data(), sizeof(double) * s * s);
    if (b) std::memcpy(b, t.b.data(), sizeof(double) * s);
    if (c) std::memcpy(c, t.c.data(), sizeof(double) * s);
  });
}

int stg_spatial_rhs(stg_handle* h, double t, const double* u, double* F) {
  return guarded(h, [&] {
    need(h, "stg_spatial_rhs");
    need(u, "u");
    need(F, "F");
    (void)t;
    stg::MixCoef m = zero_mix();
    m.S[0][0] = 1.0;
    apply(h, m, 1, 1, u, nullptr, nullptr, F, false, false);
  });
}

int stg_spatial_jvp(stg_handle* h, double t, const double* u, const double* v, double* Jv) {
  return guarded(h, [&] {
    need(h, "stg_spatial_jvp");
    need(v, "v");
    need(Jv, "Jv");
    (void)t;
    stg::MixCoef m = zero_mix();
    m.S[0][0] = 1.0;
    const bool nl = !linear_model(h->desc.model);
    if (nl) need(u, "u");
    if (h->desc.model == STG_MODEL_EULER) {  // forward difference (no exact linearisation)
      const long long n = h->n_sdof;
      const double vn = std::sqrt(dev_dot(h, v, v, n));
      if (vn == 0.0) {
        stg::vec_fill(Jv, 0.0, n, h->stream);
        h->launches++;
        return;
      }
      const double eps = kEulerFdEps * std::sqrt(1.0 + std::sqrt(dev_dot(h, u, u, n))) / vn;
      h->tmp1.ensure(size_t(n));
      h->tmp2.ensure(size_t(n));
      stg::vec_copy(h->tmp1.p, u, n, h->stream);
      stg::vec_axpy(h->tmp1.p, eps, v, n, h->stream);
      h->launches += 2;
      apply(h, m, 1, 1, h->tmp1.p, nullptr, nullptr, Jv, false, false);
      stg::vec_axpy(h->tmp1.p, -2.0 * eps, v, n, h->stream);
      h->launches++;
      apply(h, m, 1, 1, h->tmp1.p, nullptr, nullptr, h->tmp2.p, false, false);
      stg::vec_axpby(Jv, -0.5 / eps, h->tmp2.p, 0.5 / eps, n, h->stream);
      h->launches++;
      return;
    }
    apply(h, m, 1, 1, v, nl ? u : nullptr, nullptr, Jv, nl, false);
  });
}

int stg_st_residual(stg_handle* h, double t_n, double dt, const double* u_n, const double* U,
                    double* R) {
  return guarded(h, [&] {
    need(h, "stg_st_residual");
    need(u_n, "u_n");
    need(U, "U");
    need(R, "R");
    (void)t_n;
    st_residual(h, dt, u_n, U, R);
  });
}

int stg_st_jvp(stg_handle* h, double t_n, double dt, const double* U, const double* v,
               double* Jv, double fd_eps) {
  return guarded(h, [&] {
    need(h, "stg_st_jvp");
    need(v, "v");
    need(Jv, "Jv");
    if (!linear_model(h->desc.model)) need(U, "U");
    (void)t_n;
    st_jvp(h, dt, U, v, Jv, fd_eps);
  });
}

int stg_stage_residual(stg_handle* h, int form, double t, double dt, const double* u,
                       const double* U, double* R) {
  return guarded(h, [&] {
    need(h, "stg_stage_residual");
    need(u, "u");
    need(U, "U");
    need(R, "R");
    (void)t;
    if (form != STG_FORM_A && form != STG_FORM_A_INV) throw std::invalid_argument("bad form");
    stage_residual(h, form, dt, u, U, R);
  });
}

int stg_stage_jvp(stg_handle* h, int form, double t, double dt, const double* U,
                  const double* v, double* Jv, double fd_eps) {
  return guarded(h, [&] {
    need(h, "stg_stage_jvp");
    need(v, "v");
    need(Jv, "Jv");
    (void)t;
    if (form != STG_FORM_A && form != STG_FORM_A_INV) throw std::invalid_argument("bad form");
    if (!linear_model(h->desc.model)) need(U, "U");
    stage_jvp(h, form, dt, U, v, Jv, fd_eps);
  });
}

int stg_gmres_st(stg_handle* h, double t_n, double dt, const double* U, const double* b,
                 double* x, int restart, double tol, int max_it, int precond, int* iterations,
                 double* rel_residual) {
  return guarded(h, [&] {
    need(h, "stg_gmres_st");
    need(b, "b");
    need(x, "x");
    (void)t_n;
    if (!linear_model(h->desc.model)) need(U, "U");
    h->eblock_valid = false;
    const Op A = [h, dt, U](const double* v, double* Jv) { st_jvp(h, dt, U, v, Jv, 0.0); };
    const Op P = precond_for(h, precond, st_mix(h, dt, false), U, A);
    h->pred_slot = 0;
    const GmresStats st = gmres(h, A, b, x, h->n_dof, restart, tol, max_it, P ? &P : nullptr,
                                /*x_zero=*/false, /*pipelined=*/true);
    if (iterations) *iterations = st.iterations;
    if (rel_residual) *rel_residual = st.rel_residual;
    if (!st.converged)
      throw std::runtime_error("linear_solve: GMRES did not converge, error " +
                               fmt_short(st.rel_residual));
  });
}

int stg_st_precond_apply(stg_handle* h, double dt, const double* U, int precond,
                         const double* in, double* out) {
  return guarded(h, [&] {
    need(h, "stg_st_precond_apply");
    need(in, "in");
    need(out, "out");
    if (!linear_model(h->desc.model)) need(U, "U");
    h->eblock_valid = false;
    const Op A = [h, dt, U](const double* v, double* Jv) { st_jvp(h, dt, U, v, Jv, 0.0); };
    const Op P = precond_for(h, precond, st_mix(h, dt, false), U, A);
    if (P) {
      P(in, out);
      check_launch(h);
    } else {
      stg::vec_copy(out, in, h->n_dof, h->stream);
      h->launches++;
      check_launch(h);
    }
  });
}

int stg_stdg_step(stg_handle* h, double t_n, double dt, const double* u_n,
                  const stg_newton_config* cfg, double* U, double* u_next,
                  stg_solve_info* info) {
  return guarded(h, [&] {
    need(h, "stg_stdg_step");
    need(u_n, "u_n");
    need(U, "U");
    do_stdg_step(h, t_n, dt, u_n, cfg, U, u_next, info);
  });
}


int stg_stdg_integrate(stg_handle* h, double t0, const double* u0, double t_end, int n_steps,
                       const stg_newton_config* cfg, double* u_final, double* states,
                       double* U_slabs, stg_solve_info* info) {
  return guarded(h, [&] {
    need(h, "stg_stdg_integrate");
    need(u0, "u0");
    need(u_final, "u_final");
    integrate_impl(h, t0, u0, t_end, n_steps, u_final, states, U_slabs, info, "stdg_integrate",
                   [&](double tk, double dt, const double* uk, double* Uk, double* un,
                       stg_solve_info* ik) { do_stdg_step(h, tk, dt, uk, cfg, Uk, un, ik); });
  });
}

int stg_rk_integrate(stg_handle* h, int form, double t0, const double* u0, double t_end,
                     int n_steps, const stg_newton_config* cfg, double* u_final, double* states,
                     double* U_stages, stg_solve_info* info) {
  return guarded(h, [&] {
    need(h, "stg_rk_integrate");
    need(u0, "u0");
    need(u_final, "u_final");
    integrate_impl(h, t0, u0, t_end, n_steps, u_final, states, U_stages, info, "integrate",
                   [&](double tk, double dt, const double* uk, double* Uk, double* un,
                       stg_solve_info* ik) { do_rk_step(h, form, tk, dt, uk, cfg, Uk, un, ik); });
  });
}

int stg_rk_step(stg_handle* h, int form, double t, double dt, const double* u,
                const stg_newton_config* cfg, double* U, double* u_next, stg_solve_info* info) {
  return guarded(h, [&] {
    need(h, "stg_rk_step");
    need(u, "u");
    need(U, "U");
    do_rk_step(h, form, t, dt, u, cfg, U, u_next, info);
  });
}

// ---- host-buffer variants -------------------------------------------------------
int stg_st_residual_host(stg_handle* h, double t_n, double dt, const double* u_n,
                         const double* U, double* R) {
  return guarded(h, [&] {
    need(h, "stg_st_residual_host");
    need(u_n, "u_n");
    need(U, "U");
    need(R, "R");
    (void)t_n;
    // pageable caller memory goes through the library's own page-locked
    // mirrors (hostcopy.hpp); STG_HOST_NO_STAGING=1 leaves it to the driver
    const bool staged = stage_large(h) && (pageable(U) || pageable(R) || pageable(u_n));
    if (!std::getenv("STG_HOST_NO_PIPELINE") &&
        (staged ? st_residual_host_staged(h, dt, u_n, U, R)
                : st_residual_host_pipelined(h, dt, u_n, U, R)))
      return;
    h->host_U.ensure(size_t(h->n_dof));
    h->host_R.ensure(size_t(h->n_dof));
    h->host_u.ensure(size_t(h->n_sdof));
    cudaStream_t s = h->stream;
    if (staged) {
      staged_h2d(h, h->host_U.p, U, size_t(h->n_dof), h->pin_U, s);
      staged_h2d(h, h->host_u.p, u_n, size_t(h->n_sdof), h->pin_u, s);
      st_residual(h, dt, h->host_u.p, h->host_U.p, h->host_R.p);
      staged_d2h(h, R, h->host_R.p, size_t(h->n_dof), h->pin_R, s);
      return;
    }
    ck(cudaMemcpyAsync(h->host_U.p, U, sizeof(double) * h->n_dof, cudaMemcpyHostToDevice, s), "H2D");
    ck(cudaMemcpyAsync(h->host_u.p, u_n, sizeof(double) * h->n_sdof, cudaMemcpyHostToDevice, s),
       "H2D");
    st_residual(h, dt, h->host_u.p, h->host_U.p, h->host_R.p);
    ck(cudaMemcpyAsync(R, h->host_R.p, sizeof(double) * h->n_dof, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
  });
}

int stg_stdg_step_host(stg_handle* h, double t_n, double dt, const double* u_n,
                       const stg_newton_config* cfg, double* U, double* u_next,
                       stg_solve_info* info) {
  return guarded(h, [&] {
    need(h, "stg_stdg_step_host");
    need(u_n, "u_n");
    need(U, "U");
    h->host_U.ensure(size_t(h->n_dof));
    h->host_u.ensure(size_t(h->n_sdof));
    h->host_u2.ensure(size_t(h->n_sdof));
    step_host_in(h, u_n);
    try {
      do_stdg_step(h, t_n, dt, h->host_u.p, cfg, h->host_U.p, h->host_u2.p, info);
    } catch (const NonconvergenceError&) {  // the last iterate goes back to U
      step_host_out(h, U, nullptr);
      throw;
    }
    step_host_out(h, U, u_next);
  });
}

int stg_rk_step_host(stg_handle* h, int form, double t, double dt, const double* u,
                     const stg_newton_config* cfg, double* U, double* u_next,
                     stg_solve_info* info) {
  return guarded(h, [&] {
    need(h, "stg_rk_step_host");
    need(u, "u");
    need(U, "U");
    h->host_U.ensure(size_t(h->n_dof));
    h->host_u.ensure(size_t(h->n_sdof));
    h->host_u2.ensure(size_t(h->n_sdof));
    step_host_in(h, u);
    try {
      do_rk_step(h, form, t, dt, h->host_u.p, cfg, h->host_U.p, h->host_u2.p, info);
    } catch (const NonconvergenceError&) {  // the last iterate goes back to U
      step_host_out(h, U, nullptr);
      throw;
    }
    step_host_out(h, U, u_next);
  });
}

}  // extern "C"
