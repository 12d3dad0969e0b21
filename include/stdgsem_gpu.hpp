// stdgsem_gpu.hpp -- C++ host mirror of the reference stdgsem slab interface,
// backed by the CUDA library through the C ABI (stg_cuda.h).
//
// Header-only; link against libstg_cuda.so.  Same free-function names,
// argument meaning and exception types as the reference headers:
//   st_residual   stdg.hpp:56-76        st_jacobian  stdg.hpp:79-110 (matrix-free)
//   stdg_step     stdg.hpp:120-143      stdg_integrate stdg.hpp:152-173
//   rk_step       lodg.hpp:89-149       integrate    lodg.hpp:158-181
//   NewtonConfig  newton.hpp:30-38      NonconvergenceError newton.hpp:40-48
// Vec is a std::vector<double> on the host (the reference's Eigen::VectorXd
// role) whose allocator hands out page-locked memory for large vectors, so
// every call's copies are plain DMA from / to the caller's vectors; each call
// moves them to the device once, runs there, and copies the result back.  For
// device-resident loops use the DeviceVec overloads.
// Status codes map back to std::invalid_argument / std::runtime_error /
// NonconvergenceError / AdmissibilityError; CUDA failures throw CudaError
// (there is no CPU path).
#pragma once

#include <cmath>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "stg_cuda.h"

namespace stdgsem {
namespace gpu {

// Allocator behind Vec.  Blocks of kPinBytes or more are page-locked
// (stg_host_alloc) and recycled through a process-wide free list keyed by
// size, so a time-marching loop that keeps creating result vectors, as the
// reference's value-returning API makes it, pays cudaHostAlloc and the first-
// touch page faults once per size, not per call (c4 stdg_step on fresh
// std::vector<double> results: 37 ms per call, of which 2.5 ms is the solve
// and its copies).  Smaller blocks, and every block when no device is present
// (host-only helpers), come from malloc.  Like Eigen::VectorXd(n), Vec(n)
// leaves its entries uninitialised; Vec(n, 0.0) zero-fills.
namespace detail {
constexpr std::size_t kPinBytes = std::size_t(256) << 10;
constexpr std::size_t kPoolCapBytes = std::size_t(2) << 30;  // cached free blocks

struct PinnedPool {
  std::mutex mu;
  std::multimap<std::size_t, double*> free_blocks;
  std::size_t cached = 0;
  int mode = 0;  // 0 undecided, 1 page-locked, 2 malloc (no device)

  double* take(std::size_t bytes) {
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = free_blocks.find(bytes);
      if (it != free_blocks.end()) {
        double* p = it->second;
        free_blocks.erase(it);
        cached -= bytes;
        return p;
      }
      if (mode == 2) return nullptr;
    }
    double* p = nullptr;
    const int code = stg_host_alloc((long long)(bytes / sizeof(double)), &p);
    std::lock_guard<std::mutex> lk(mu);
    if (code == STG_OK && p) {
      mode = 1;
      return p;
    }
    if (mode == 1) throw std::bad_alloc();  // page-locked memory exhausted
    mode = 2;
    return nullptr;
  }
  // returns false when the block is not the pool's (malloc mode)
  bool give(double* p, std::size_t bytes) {
    std::lock_guard<std::mutex> lk(mu);
    if (mode != 1) return false;
    if (cached + bytes <= kPoolCapBytes) {
      free_blocks.emplace(bytes, p);
      cached += bytes;
    } else {
      stg_host_free(p);
    }
    return true;
  }
};

inline PinnedPool& pinned_pool() {
  static PinnedPool* pool = new PinnedPool;  // never destroyed: outlives the CUDA context's users
  return *pool;
}
}  // namespace detail

template <class T>
struct HostAllocator {
  using value_type = T;
  HostAllocator() = default;
  template <class U>
  HostAllocator(const HostAllocator<U>&) noexcept {}
  T* allocate(std::size_t n) {
    const std::size_t bytes = n * sizeof(T);
    if (bytes >= detail::kPinBytes && bytes % sizeof(double) == 0)
      if (double* p = detail::pinned_pool().take(bytes)) return reinterpret_cast<T*>(p);
    void* p = std::malloc(bytes ? bytes : 1);
    if (!p) throw std::bad_alloc();
    return static_cast<T*>(p);
  }
  void deallocate(T* p, std::size_t n) noexcept {
    const std::size_t bytes = n * sizeof(T);
    if (bytes >= detail::kPinBytes && bytes % sizeof(double) == 0 &&
        detail::pinned_pool().give(reinterpret_cast<double*>(p), bytes))
      return;
    std::free(p);
  }
  // default-initialise (no zero fill of a vector about to be overwritten)
  template <class U>
  void construct(U* p) noexcept(std::is_nothrow_default_constructible<U>::value) {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
  template <class U>
  bool operator==(const HostAllocator<U>&) const noexcept { return true; }
  template <class U>
  bool operator!=(const HostAllocator<U>&) const noexcept { return false; }
};

using Vec = std::vector<double, HostAllocator<double>>;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// AdmissibilityError (models.hpp:15-20); the message names the temporal node.
struct AdmissibilityError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// NonconvergenceError (newton.hpp:40-48): the last Newton iterate and the
// residual history, rethrown with the step context (stdg.hpp:132-137).
struct NonconvergenceError : std::runtime_error {
  Vec last_iterate;
  std::vector<double> residual_history;
  NonconvergenceError(const std::string& what, Vec u, std::vector<double> history)
      : std::runtime_error(what),
        last_iterate(std::move(u)),
        residual_history(std::move(history)) {}
};

inline std::vector<double> history_of(const stg_solve_info& info) {
  return std::vector<double>(info.residual_history, info.residual_history + info.n_history);
}

inline void check(int code, const stg_handle* h) {
  if (code == STG_OK) return;
  const std::string msg = stg_last_error(h);
  switch (code) {
    case STG_ERR_INVALID: throw std::invalid_argument(msg);
    case STG_ERR_NONCONVERGENCE: throw NonconvergenceError(msg, {}, {});
    case STG_ERR_CUDA: throw CudaError(msg);
    case STG_ERR_ADMISSIBILITY: throw AdmissibilityError(msg);
    default: throw std::runtime_error(msg);
  }
}

// RAII device vector.
class DeviceVec {
 public:
  DeviceVec() = default;
  explicit DeviceVec(size_t n) : n_(n) { check(stg_device_alloc((long long)n, &p_), nullptr); }
  explicit DeviceVec(const Vec& v) : DeviceVec(v.size()) { upload(v); }
  DeviceVec(DeviceVec&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  DeviceVec& operator=(DeviceVec&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    return *this;
  }
  DeviceVec(const DeviceVec&) = delete;
  DeviceVec& operator=(const DeviceVec&) = delete;
  ~DeviceVec() {
    if (p_) stg_device_free(p_);
  }
  void upload(const Vec& v) {
    if (v.size() != n_) throw std::invalid_argument("DeviceVec::upload: size mismatch");
    check(stg_memcpy(p_, v.data(), (long long)n_, 0), nullptr);
  }
  Vec download() const {
    Vec v(n_);
    check(stg_memcpy(v.data(), p_, (long long)n_, 1), nullptr);
    return v;
  }
  double* data() { return p_; }
  const double* data() const { return p_; }
  size_t size() const { return n_; }

 private:
  double* p_ = nullptr;
  size_t n_ = 0;
};

// ---- discretisation data (mesh.hpp, models.hpp) ------------------------------
struct Mesh {  // mesh.hpp:14-35; d = 3 is an extension of the reference
  int d = 1;
  std::vector<double> lower, upper;
  std::vector<int> cells;
};

inline Mesh uniform_mesh(int d, const std::vector<double>& lower,
                         const std::vector<double>& upper, const std::vector<int>& cells) {
  if (d < 1 || d > 3) throw std::invalid_argument("uniform_mesh: d in {1,2,3}");
  if (int(lower.size()) != d || int(upper.size()) != d || int(cells.size()) != d)
    throw std::invalid_argument("uniform_mesh: inconsistent sizes");
  return Mesh{d, lower, upper, cells};
}

struct DgSpace {  // mesh.hpp:59-91
  Mesh mesh;
  int p = 1;
  int r = 1;  // components per node
  int dof() const {
    int npc = 1, nc = 1;
    for (int a = 0; a < mesh.d; ++a) {
      npc *= p + 1;
      nc *= mesh.cells[size_t(a)];
    }
    return r * npc * nc;
  }
};
inline DgSpace dg_space(const Mesh& m, int p, int r = 1) {  // mesh.hpp:93-110
  if (p < 1) throw std::invalid_argument("dg_space: need p >= 1 (p = 0 has no LGL rule)");
  if (r < 1) throw std::invalid_argument("dg_space: need r >= 1");
  return DgSpace{m, p, r};
}

// ---- host-side field helpers (mesh.hpp:82-90, 113-181) -----------------------
// Same index map as the library: cell = (cz*ny + cy)*nx + cx, node x-fastest,
// coefficient (cell * npc + node) * r + comp (mesh.hpp:70-81; d = 3 extended).
inline Vec lgl_nodes(int n) {  // lgl_rule(n).nodes (quadrature.hpp:66-105)
  Vec x(static_cast<size_t>(n)), w(static_cast<size_t>(n));
  check(stg_lgl_rule(n, x.data(), w.data()), nullptr);
  return x;
}
inline Vec lgl_weights(int n) {
  Vec x(static_cast<size_t>(n)), w(static_cast<size_t>(n));
  check(stg_lgl_rule(n, x.data(), w.data()), nullptr);
  return w;
}
inline int nodes_per_cell(const DgSpace& s) {
  int npc = 1;
  for (int a = 0; a < s.mesh.d; ++a) npc *= s.p + 1;
  return npc;
}
inline int n_cells(const Mesh& m) {
  int nc = 1;
  for (int a = 0; a < m.d; ++a) nc *= m.cells[size_t(a)];
  return nc;
}

// node_coord (mesh.hpp:82-90): x_a = lower_a + (c_a + (1 + xi_{i_a}) / 2) h_a,
// evaluated in the reference's operation order (bitwise equal)
inline Vec node_coord(const DgSpace& s, const Vec& xi, int cell, int node) {
  const int n = s.p + 1;
  int ci[3] = {0, 0, 0}, ni[3] = {0, 0, 0};
  int c = cell, q = node;
  for (int a = 0; a < s.mesh.d; ++a) {
    ci[a] = c % s.mesh.cells[size_t(a)];
    c /= s.mesh.cells[size_t(a)];
    ni[a] = q % n;
    q /= n;
  }
  Vec x(size_t(s.mesh.d));
  for (int a = 0; a < s.mesh.d; ++a) {
    const double h = (s.mesh.upper[size_t(a)] - s.mesh.lower[size_t(a)]) / s.mesh.cells[size_t(a)];
    x[size_t(a)] = s.mesh.lower[size_t(a)] + (ci[a] + 0.5 * (1.0 + xi[size_t(ni[a])])) * h;
  }
  return x;
}
inline Vec node_coord(const DgSpace& s, int cell, int node) {
  return node_coord(s, lgl_nodes(s.p + 1), cell, node);
}

struct DiscreteField {  // mesh.hpp:113-117
  DgSpace space;
  Vec coeffs;
  double time_tag = 0.0;
};

// interpolate (mesh.hpp:145-157): f maps a point to r component values
template <class F>
DiscreteField interpolate(const DgSpace& s, F&& f, double t = 0.0) {
  DiscreteField field{s, Vec(size_t(s.dof())), t};
  const Vec xi = lgl_nodes(s.p + 1);
  const int npc = nodes_per_cell(s), nc = n_cells(s.mesh);
  for (int cell = 0; cell < nc; ++cell)
    for (int node = 0; node < npc; ++node) {
      const Vec val = f(node_coord(s, xi, cell, node));
      for (int comp = 0; comp < s.r; ++comp)
        field.coeffs[(size_t(cell) * npc + node) * s.r + comp] = val[size_t(comp)];
    }
  return field;
}

// interpolate_scalar (mesh.hpp:159-165)
template <class F>
DiscreteField interpolate_scalar(const DgSpace& s, F&& f, double t = 0.0) {
  return interpolate(s, [&](const Vec& x) { return Vec{f(x)}; }, t);
}

struct GlobalMassDiagonal {  // mesh.hpp:121-124
  DgSpace space;
  Vec diag;
};

// global_mass (mesh.hpp:125-141): cell volume / 2^d times tensor LGL weights,
// replicated across the r components
inline GlobalMassDiagonal global_mass(const DgSpace& s) {
  GlobalMassDiagonal m{s, Vec(size_t(s.dof()))};
  double vol = 1.0;
  for (int a = 0; a < s.mesh.d; ++a)
    vol *= (s.mesh.upper[size_t(a)] - s.mesh.lower[size_t(a)]) / s.mesh.cells[size_t(a)];
  double pw = 1.0;
  for (int a = 0; a < s.mesh.d; ++a) pw *= 2.0;
  const double vol_scale = vol / pw;
  const Vec w = lgl_weights(s.p + 1);
  const int n = s.p + 1, npc = nodes_per_cell(s), nc = n_cells(s.mesh);
  for (int cell = 0; cell < nc; ++cell)
    for (int node = 0; node < npc; ++node) {
      double wn = w[size_t(node % n)];
      if (s.mesh.d >= 2) wn *= w[size_t((node / n) % n)];
      if (s.mesh.d == 3) wn *= w[size_t(node / (n * n))];
      for (int comp = 0; comp < s.r; ++comp)
        m.diag[(size_t(cell) * npc + node) * s.r + comp] = vol_scale * wn;
    }
  return m;
}

// l2_norm (mesh.hpp:167-172): one square root of the mass-weighted sum
inline double l2_norm(const DiscreteField& f) {
  const Vec d = global_mass(f.space).diag;
  double acc = 0.0;
  for (size_t i = 0; i < d.size(); ++i) acc += f.coeffs[i] * f.coeffs[i] * d[i];
  return std::sqrt(acc);
}

// l2_error (mesh.hpp:174-181): exact(x, t) returns the r component values
template <class F>
double l2_error(const DiscreteField& field, F&& exact, double t) {
  DiscreteField diff = interpolate(field.space, [&](const Vec& x) { return exact(x, t); }, t);
  for (size_t i = 0; i < diff.coeffs.size(); ++i)
    diff.coeffs[i] = field.coeffs[i] - diff.coeffs[i];
  return l2_norm(diff);
}

// FluxModel (models.hpp:23-36): which of the library's models, with its data.
struct FluxModel {
  int kind = STG_MODEL_ADVECTION;
  std::vector<double> b;               // constant velocity
  int field = STG_FIELD_CONSTANT;      // advdiff velocity field
  double eps = 0.0;                    // advdiff diffusion
  double gamma = 1.4;                  // euler
  int r = 1;
};
// VelocityField (models.hpp:38): constant b, or rotating_field() (models.hpp:79-85)
struct VelocityField {
  int kind = STG_FIELD_CONSTANT;
  std::vector<double> b;
};
inline VelocityField rotating_field() { return VelocityField{STG_FIELD_ROTATING, {0.0, 0.0}}; }
inline VelocityField constant_field(const std::vector<double>& b) {
  return VelocityField{STG_FIELD_CONSTANT, b};
}
inline FluxModel advection_model(const std::vector<double>& b) {  // models.hpp:40-66
  FluxModel m;
  m.b = b;
  return m;
}
inline FluxModel burgers_model() {  // EXTENSION (not in the reference)
  FluxModel m;
  m.kind = STG_MODEL_BURGERS;
  m.b = {0.0};
  return m;
}
inline FluxModel advdiff_model(int d, const VelocityField& b, double eps) {  // models.hpp:68-76
  if (eps < 0) throw std::invalid_argument("advdiff_model: need eps >= 0");
  FluxModel m;
  m.kind = STG_MODEL_ADVDIFF;
  m.b = b.b;
  m.b.resize(size_t(d), 0.0);
  m.field = b.kind;
  m.eps = eps;
  return m;
}
inline FluxModel euler_model(double gamma = 1.4) {  // models.hpp:118-159, r = 4, d = 2
  if (!(gamma > 1.0)) throw std::invalid_argument("euler_model: gamma > 1");
  FluxModel m;
  m.kind = STG_MODEL_EULER;
  m.b = {0.0, 0.0};
  m.gamma = gamma;
  m.r = 4;
  return m;
}

enum class LinearMethod { auto_select = STG_LINEAR_AUTO, gmres = STG_LINEAR_GMRES };
enum class JacobianForm { a_form = STG_FORM_A, a_inv_form = STG_FORM_A_INV };

struct NewtonConfig {  // newton.hpp:30-38
  double abs_tol = 1e-12;
  double rel_tol = 1e-12;
  int max_iter = 50;
  LinearMethod linear = LinearMethod::auto_select;
  int gmres_restart = 30;
  double gmres_tol = 1e-12;
  int gmres_max_it = 1000;
  double fd_eps = 0.0;
  int precond = STG_PRECOND_AUTO;  // right preconditioner, STG_PRECOND_* (stg_cuda.h)
  stg_newton_config c() const {
    return stg_newton_config{abs_tol,      rel_tol, max_iter, int(linear), gmres_restart,
                             gmres_tol,    gmres_max_it, fd_eps, precond};
  }
};

// The slab operator for one (space, model, n_tau): owns a C-ABI handle.
class SlabOperator {
 public:
  SlabOperator(const DgSpace& space, const FluxModel& model, int n_tau, double eta = 0.0) {
    stg_desc d{};
    d.dim = space.mesh.d;
    d.degree = space.p;
    d.n_tau = n_tau;
    d.model = model.kind;
    d.velocity_field = model.field;
    d.eps = model.eps;
    d.eta = eta;
    d.gamma = model.gamma;
    for (int a = 0; a < 3; ++a) {
      d.cells[a] = a < d.dim ? space.mesh.cells[size_t(a)] : 1;
      d.lower[a] = a < d.dim ? space.mesh.lower[size_t(a)] : 0.0;
      d.upper[a] = a < d.dim ? space.mesh.upper[size_t(a)] : 1.0;
      d.velocity[a] = a < int(model.b.size()) ? model.b[size_t(a)] : 0.0;
    }
    stg_handle* h = nullptr;
    check(stg_create(&d, &h), nullptr);
    h_.reset(h);
    long long ns = 0, nd = 0;
    stg_sizes(h, &ns, &nd);
    n_sdof_ = size_t(ns);
    n_dof_ = size_t(nd);
  }
  stg_handle* handle() const { return h_.get(); }
  size_t n_sdof() const { return n_sdof_; }
  size_t n_dof() const { return n_dof_; }

 private:
  struct Del {
    void operator()(stg_handle* h) const { stg_destroy(h); }
  };
  std::unique_ptr<stg_handle, Del> h_;
  size_t n_sdof_ = 0, n_dof_ = 0;
};

// SemiDiscreteSystem (system.hpp:16-23): the seam.  Lazily creates one slab
// operator per number of temporal nodes.
class SemiDiscreteSystem {
 public:
  SemiDiscreteSystem(DgSpace space, FluxModel model, double eta = 0.0)
      : space_(std::move(space)), model_(std::move(model)), eta_(eta) {}
  int dof() const { return space_.dof(); }
  // the interior-penalty parameter in use (spatial.hpp:366 default 10 p^2)
  double eta() const { return eta_ > 0 ? eta_ : 10.0 * space_.p * space_.p; }
  SlabOperator& op(int n_tau) const {
    for (auto& e : ops_)
      if (e.first == n_tau) return *e.second;
    ops_.emplace_back(n_tau, std::make_shared<SlabOperator>(space_, model_, n_tau, eta_));
    return *ops_.back().second;
  }
  // rhs(t, u) = F(u) (spatial.hpp:107-266)
  Vec rhs(double t, const Vec& u) const {
    SlabOperator& o = op(2);
    DeviceVec du(u), F(o.n_sdof());
    check(stg_spatial_rhs(o.handle(), t, du.data(), F.data()), o.handle());
    return F.download();
  }

 private:
  DgSpace space_;
  FluxModel model_;
  double eta_ = 0.0;
  mutable std::vector<std::pair<int, std::shared_ptr<SlabOperator>>> ops_;
};

// assemble_semidiscrete (spatial.hpp:352-385); eta <= 0: the default 10 p^2.
inline SemiDiscreteSystem assemble_semidiscrete(const DgSpace& space, const FluxModel& model,
                                                double eta = 0.0) {
  if (model.kind == STG_MODEL_ADVECTION && int(model.b.size()) != space.mesh.d)
    throw std::invalid_argument("assemble_semidiscrete: dimension mismatch");
  if (model.kind == STG_MODEL_EULER && space.mesh.d != 2)
    throw std::invalid_argument("assemble_semidiscrete: dimension mismatch");
  if (model.r != space.r)
    throw std::invalid_argument("assemble_semidiscrete: component mismatch");
  return SemiDiscreteSystem(space, model, eta);
}

struct SbpOperators {  // operators.hpp:16-22 (the library builds D, M itself)
  int n = 0;
};
inline SbpOperators sbp_operators(int n) {
  if (n < 2) throw std::invalid_argument("sbp_operators: need n >= 2");
  return SbpOperators{n};
}
struct ButcherTableau {  // operators.hpp:24-30
  int s = 0;
};
inline ButcherTableau lobatto_tableau(int s) {
  if (s < 2 || s > 4)
    throw std::invalid_argument("lobatto_tableau: closed forms stored for s in {2,3,4}");
  return ButcherTableau{s};
}

struct TimeElementSystem {  // stdg.hpp:21-29
  SemiDiscreteSystem system;
  SbpOperators ops;
  double t_n = 0.0;
  double dt = 0.0;
  Vec u_n;
  int n_tau() const { return ops.n; }
};

// st_residual (stdg.hpp:56-76)
inline Vec st_residual(const TimeElementSystem& sys, const Vec& U) {
  SlabOperator& o = sys.system.op(sys.ops.n);
  if (U.size() != o.n_dof())
    throw std::invalid_argument("st_residual: expected " + std::to_string(o.n_dof()) +
                                " unknowns");
  Vec R(o.n_dof());
  check(stg_st_residual_host(o.handle(), sys.t_n, sys.dt, sys.u_n.data(), U.data(), R.data()),
        o.handle());
  return R;
}

// st_jacobian (stdg.hpp:79-110) as a matrix-free action J(U) v.
inline Vec st_jacobian_apply(const TimeElementSystem& sys, const Vec& U, const Vec& v,
                             double fd_eps = 0.0) {
  SlabOperator& o = sys.system.op(sys.ops.n);
  if (U.size() != o.n_dof() || v.size() != o.n_dof())
    throw std::invalid_argument("st_jacobian: expected " + std::to_string(o.n_dof()) +
                                " unknowns");
  DeviceVec dU(U), dv(v), Jv(o.n_dof());
  check(stg_st_jvp(o.handle(), sys.t_n, sys.dt, dU.data(), dv.data(), Jv.data(), fd_eps),
        o.handle());
  return Jv.download();
}

struct StdgStepResult {  // stdg.hpp:112-116
  Vec U;
  Vec u_next;
  int newton_iterations = 0;
  int linear_iterations = 0;
};

// stdg_step (stdg.hpp:120-143)
inline StdgStepResult stdg_step(const SemiDiscreteSystem& system, const SbpOperators& ops,
                                double t_n, const Vec& u_n, double dt,
                                const NewtonConfig& cfg = {}) {
  SlabOperator& o = system.op(ops.n);
  if (u_n.size() != o.n_sdof()) throw std::invalid_argument("stdg_step: u_n size mismatch");
  StdgStepResult r;
  r.U.resize(o.n_dof());
  r.u_next.resize(o.n_sdof());
  stg_solve_info info{};
  const stg_newton_config c = cfg.c();
  const int code = stg_stdg_step_host(o.handle(), t_n, dt, u_n.data(), &c, r.U.data(),
                                      r.u_next.data(), &info);
  if (code == STG_ERR_NONCONVERGENCE)  // the library left the last iterate in U
    throw NonconvergenceError(stg_last_error(o.handle()), std::move(r.U), history_of(info));
  check(code, o.handle());
  r.newton_iterations = info.newton_iterations;
  r.linear_iterations = info.linear_iterations;
  return r;
}

struct StdgTrajectory {  // stdg.hpp:145-150
  Vec times;
  std::vector<Vec> states;
  std::vector<Vec> element_solutions;
  int total_newton_iterations = 0;
};

// stdg_integrate (stdg.hpp:152-173)
inline StdgTrajectory stdg_integrate(const SemiDiscreteSystem& system, const SbpOperators& ops,
                                     double t0, const Vec& u0, double t_end, int n_steps,
                                     const NewtonConfig& cfg = {}) {
  if (n_steps < 1) throw std::invalid_argument("stdg_integrate: n_steps >= 1 required");
  SlabOperator& o = system.op(ops.n);
  if (u0.size() != o.n_sdof()) throw std::invalid_argument("stdg_integrate: u0 size mismatch");
  StdgTrajectory traj;
  traj.times.resize(size_t(n_steps) + 1);
  for (int k = 0; k <= n_steps; ++k) traj.times[size_t(k)] = t0 + (t_end - t0) * k / n_steps;
  // marched on the device (stg_stdg_integrate), one download at the end
  DeviceVec du(u0), uf(o.n_sdof()), st((size_t(n_steps) + 1) * o.n_sdof()),
      sol(size_t(n_steps) * o.n_dof());
  const stg_newton_config c = cfg.c();
  stg_solve_info info{};
  const int code = stg_stdg_integrate(o.handle(), t0, du.data(), t_end, n_steps, &c, uf.data(),
                                      st.data(), sol.data(), &info);
  if (code == STG_ERR_NONCONVERGENCE) {  // the failing slab's last iterate is in its slot
    Vec last;
    if (info.failed_step >= 0) {
      const Vec sols = sol.download();
      last.assign(sols.begin() + long(size_t(info.failed_step) * o.n_dof()),
                  sols.begin() + long(size_t(info.failed_step + 1) * o.n_dof()));
    }
    throw NonconvergenceError(stg_last_error(o.handle()), std::move(last), history_of(info));
  }
  check(code, o.handle());
  const Vec all = st.download(), sols = sol.download();
  for (int k = 0; k <= n_steps; ++k)
    traj.states.emplace_back(all.begin() + long(size_t(k) * o.n_sdof()),
                             all.begin() + long(size_t(k + 1) * o.n_sdof()));
  for (int k = 0; k < n_steps; ++k)
    traj.element_solutions.emplace_back(sols.begin() + long(size_t(k) * o.n_dof()),
                                        sols.begin() + long(size_t(k + 1) * o.n_dof()));
  traj.total_newton_iterations = info.newton_iterations;
  return traj;
}

struct RkStepResult {  // lodg.hpp:33-38
  Vec u_next;
  std::vector<Vec> stages;
  int newton_iterations = 0;
  double t_next = 0.0;
};

// rk_step (lodg.hpp:89-149)
inline RkStepResult rk_step(const SemiDiscreteSystem& system, const ButcherTableau& tab, double t,
                            const Vec& u, double dt, const NewtonConfig& cfg = {},
                            JacobianForm jac_form = JacobianForm::a_form) {
  SlabOperator& o = system.op(tab.s);
  if (u.size() != o.n_sdof()) throw std::invalid_argument("rk_step: u size mismatch");
  Vec U(o.n_dof());
  RkStepResult r;
  r.u_next.resize(o.n_sdof());
  stg_solve_info info{};
  const stg_newton_config c = cfg.c();
  const int code = stg_rk_step_host(o.handle(), int(jac_form), t, dt, u.data(), &c, U.data(),
                                    r.u_next.data(), &info);
  if (code == STG_ERR_NONCONVERGENCE)  // the library left the last iterate in U
    throw NonconvergenceError(stg_last_error(o.handle()), std::move(U), history_of(info));
  check(code, o.handle());
  const size_t ns = o.n_sdof();
  for (int j = 0; j < tab.s; ++j)
    r.stages.emplace_back(U.begin() + long(j * ns), U.begin() + long((j + 1) * ns));
  r.newton_iterations = info.newton_iterations;
  r.t_next = t + dt;
  return r;
}

struct RkTrajectory {  // lodg.hpp:151-156
  Vec times;
  std::vector<Vec> states;
  std::vector<std::vector<Vec>> stage_solutions;
  int total_newton_iterations = 0;
};

// integrate (lodg.hpp:158-181)
inline RkTrajectory integrate(const SemiDiscreteSystem& system, const ButcherTableau& tab,
                              double t0, const Vec& u0, double t_end, int n_steps,
                              const NewtonConfig& cfg = {},
                              JacobianForm jac_form = JacobianForm::a_form) {
  if (n_steps < 1) throw std::invalid_argument("integrate: n_steps >= 1 required");
  RkTrajectory traj;
  traj.times.resize(size_t(n_steps) + 1);
  for (int k = 0; k <= n_steps; ++k) traj.times[size_t(k)] = t0 + (t_end - t0) * k / n_steps;
  traj.states.push_back(u0);
  const double dt = (t_end - t0) / n_steps;
  for (int k = 0; k < n_steps; ++k) {
    RkStepResult st =
        rk_step(system, tab, traj.times[size_t(k)], traj.states.back(), dt, cfg, jac_form);
    traj.states.push_back(std::move(st.u_next));
    traj.stage_solutions.push_back(std::move(st.stages));
    traj.total_newton_iterations += st.newton_iterations;
  }
  return traj;
}

}  // namespace gpu
}  // namespace stdgsem
