// ===========================================================================
// oracle_capi.cpp -- CPU ORACLE C API (TEST INFRASTRUCTURE ONLY).
//
// extern "C" entry points over stdg_oracle.hpp so the Python tests, smoke()
// and bench.py's CPU-baseline legs can drive the restatement through ctypes.
// Never linked into the product library.  Errors: return non-zero and set a
// thread-local message readable with or_last_error().
// ===========================================================================
#include <cstring>
#include <memory>
#include <string>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "stdg_oracle.hpp"

using namespace stdg_oracle;

namespace {
thread_local std::string g_err;

struct Problem {
  int model = 0;  // 0 = advection, 1 = burgers, 4 = general (advdiff / euler)
  Space space;
  std::shared_ptr<GenOperator> gen;  // general models only
  System sys;
  Sbp ops;        // temporal SBP operators (n_tau)
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const NonconvergenceError& e) {
    g_err = e.what();
    return 3;
  } catch (const AdmissibilityError& e) {
    g_err = e.what();
    return 5;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

NewtonConfig make_cfg(const double* dcfg, const int* icfg) {
  NewtonConfig c;
  c.abs_tol = dcfg[0];
  c.rel_tol = dcfg[1];
  c.gmres_tol = dcfg[2];
  c.max_iter = icfg[0];
  c.linear = LinearMethod(icfg[1]);
  c.gmres_restart = icfg[2];
  c.gmres_max_it = icfg[3];
  return c;
}
}  // namespace

extern "C" {

const char* or_last_error() { return g_err.c_str(); }

int or_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n);
  return n;
#else
  (void)n;
  return 1;
#endif
}

int or_max_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

int or_lgl(int n, double* nodes, double* weights) {
  return guarded([&] {
    const Rule r = lgl_rule(n);
    std::memcpy(nodes, r.nodes.data(), sizeof(double) * n);
    std::memcpy(weights, r.weights.data(), sizeof(double) * n);
  });
}

int or_barycentric(int n, double* bw) {
  return guarded([&] {
    const Vec v = barycentric_weights(lgl_rule(n));
    std::memcpy(bw, v.data(), sizeof(double) * n);
  });
}

// D row-major: D[j*n+i] = D(j,i) = psi_i'(x_j)
int or_diff_matrix(int n, double* D) {
  return guarded([&] {
    const Mat M = diff_matrix(lgl_rule(n));
    std::memcpy(D, M.a.data(), sizeof(double) * n * n);
  });
}

int or_eval_interpolant(int n, const double* coeffs, double tau, double* out) {
  return guarded([&] {
    Vec c(coeffs, coeffs + n);
    *out = eval_interpolant(lgl_rule(n), c, tau);
  });
}

int or_sbp_defect(int n, double* out) {
  return guarded([&] { *out = sbp_defect(sbp_operators(n)); });
}

int or_lobatto(int s, double* A, double* b, double* c) {
  return guarded([&] {
    const Tableau t = lobatto_tableau(s);
    std::memcpy(A, t.A.a.data(), sizeof(double) * s * s);
    std::memcpy(b, t.b.data(), sizeof(double) * s);
    std::memcpy(c, t.c.data(), sizeof(double) * s);
  });
}

int or_to_butcher(int n, double* A, double* b, double* c) {
  return guarded([&] {
    const Tableau t = to_butcher(sbp_operators(n));
    std::memcpy(A, t.A.a.data(), sizeof(double) * n * n);
    std::memcpy(b, t.b.data(), sizeof(double) * n);
    std::memcpy(c, t.c.data(), sizeof(double) * n);
  });
}

// model: 0 advection (velocity b), 1 burgers (d = 1), 2 test equation u' = -u
// (system.hpp:26-44), 3 zero system (test_stdg.cpp:30-38).  n_tau temporal nodes.
int or_create(int d, int p, int n_tau, const int* cells, const double* lower,
              const double* upper, const double* b, int model, void** out) {
  return guarded([&] {
    auto pr = std::make_unique<Problem>();
    pr->model = model;
    pr->space = make_space(d, p, cells, lower, upper);
    if (model == 0) {
      pr->sys = advection_system(make_advection(pr->space, b));
    } else if (model == 1) {
      if (d != 1) throw std::invalid_argument("burgers: d = 1 only");
      Burgers bu;
      bu.s = pr->space;
      pr->sys = burgers_system(bu);
    } else if (model == 2) {
      pr->sys = test_equation_system();
    } else if (model == 3) {
      pr->sys = zero_system();
    } else {
      throw std::invalid_argument("unknown model");
    }
    pr->ops = sbp_operators(n_tau);
    *out = pr.release();
  });
}

// General flux models (models.hpp:23-192): kind 0 advdiff_model (field 0:
// constant b, 1: rotating_field; eps >= 0), kind 1 euler_model(gamma), r = 4.
// eta <= 0: the default 10 p^2 (spatial.hpp:366).
int or_create_general(int d, int p, int n_tau, const int* cells, const double* lower,
                      const double* upper, int kind, int r, int field, const double* b,
                      double eps, double eta, double gamma, void** out) {
  return guarded([&] {
    auto pr = std::make_unique<Problem>();
    pr->model = 4;
    pr->space = make_space(d, p, cells, lower, upper);
    GenModel m;
    m.kind = kind;
    m.r = r;
    m.d = d;
    m.field = field;
    for (int a = 0; a < 3; ++a) m.b[a] = b[a];
    m.eps = eps;
    m.gamma = gamma;
    pr->gen = std::make_shared<GenOperator>(make_gen_operator(pr->space, m, eta));
    pr->sys = gen_system(*pr->gen);
    pr->ops = sbp_operators(n_tau);
    *out = pr.release();
  });
}

double or_eta(void* h) {
  auto* p = static_cast<Problem*>(h);
  return p->gen ? p->gen->eta : 0.0;
}

void or_destroy(void* h) { delete static_cast<Problem*>(h); }

long long or_dof(void* h) { return static_cast<Problem*>(h)->sys.dof; }

int or_mass(void* h, double* m) {
  return guarded([&] {
    auto* pr = static_cast<Problem*>(h);
    const Vec v = pr->gen ? pr->gen->mass : global_mass(pr->space);
    std::memcpy(m, v.data(), sizeof(double) * v.size());
  });
}

int or_node_coords(void* h, double* xyz) {
  return guarded([&] {
    const Space& s = static_cast<Problem*>(h)->space;
    for (int cell = 0; cell < s.n_cells(); ++cell)
      for (int node = 0; node < s.npc(); ++node) {
        double x[3];
        s.node_coord(cell, node, x);
        const int64_t k = s.coeff(cell, node);
        xyz[3 * k + 0] = x[0];
        xyz[3 * k + 1] = x[1];
        xyz[3 * k + 2] = x[2];
      }
  });
}

int or_spatial_rhs(void* h, double t, const double* u, double* F) {
  return guarded([&] { static_cast<Problem*>(h)->sys.rhs(t, u, F); });
}

int or_spatial_jvp(void* h, double t, const double* u, const double* v, double* Jv) {
  return guarded([&] { static_cast<Problem*>(h)->sys.jac(t, u, v, Jv); });
}

int or_st_residual(void* h, double t_n, double dt, const double* u_n,
                   const double* U, double* R) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    st_residual(p->sys, p->ops, t_n, dt, u_n, U, R);
  });
}

int or_st_jvp(void* h, double t_n, double dt, const double* U, const double* v,
              double* Jv) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    st_jacobian_apply(p->sys, p->ops, t_n, dt, U, v, Jv);
  });
}

int or_stage_residual(void* h, int s, int form, double t, double dt,
                      const double* u, const double* U, double* R) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    stage_residual(p->sys, lobatto_tableau(s), t, dt, u, U, JacForm(form), R);
  });
}

int or_stage_jvp(void* h, int s, int form, double t, double dt, const double* U,
                 const double* v, double* Jv) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    stage_jacobian_apply(p->sys, lobatto_tableau(s), t, dt, U, JacForm(form), v, Jv);
  });
}

// dcfg = {abs_tol, rel_tol, gmres_tol}; icfg = {max_iter, linear, restart, gmres_max_it}
// iout = {newton_iterations, linear_iterations}
int or_stdg_step(void* h, double t_n, double dt, const double* u_n,
                 const double* dcfg, const int* icfg, double* U, double* u_next,
                 int* iout) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    const int64_t dof = p->sys.dof;
    Vec un(u_n, u_n + dof);
    const StepResult r = stdg_step(p->sys, p->ops, t_n, un, dt, make_cfg(dcfg, icfg));
    std::memcpy(U, r.U.data(), sizeof(double) * r.U.size());
    std::memcpy(u_next, r.u_next.data(), sizeof(double) * dof);
    iout[0] = r.newton_iterations;
    iout[1] = r.linear_iterations;
  });
}

int or_rk_step(void* h, int s, int form, double t, double dt, const double* u,
               const double* dcfg, const int* icfg, double* U, double* u_next,
               int* iout) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    const int64_t dof = p->sys.dof;
    Vec uu(u, u + dof);
    const RkResult r = rk_step(p->sys, lobatto_tableau(s), t, uu, dt,
                               make_cfg(dcfg, icfg), JacForm(form));
    std::memcpy(U, r.U.data(), sizeof(double) * r.U.size());
    std::memcpy(u_next, r.u_next.data(), sizeof(double) * dof);
    iout[0] = r.newton_iterations;
    iout[1] = r.linear_iterations;
  });
}

// Stand-alone restarted GMRES on a small dense row-major matrix (pins the
// GMRES restatement against dense LU like test_newton.cpp:50-58).
int or_gmres_dense(int n, const double* A, const double* b, double* x, int restart,
                   double tol, int max_it, int* iters, double* relres) {
  return guarded([&] {
    LinOp op = [&](const double* v, double* Av) {
      for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int j = 0; j < n; ++j) s += A[size_t(i) * n + j] * v[j];
        Av[i] = s;
      }
    };
    for (int i = 0; i < n; ++i) x[i] = 0.0;
    const GmresStats st = gmres(op, b, x, n, restart, tol, max_it);
    *iters = st.iterations;
    *relres = st.rel_residual;
    if (!st.converged) throw std::runtime_error("gmres did not converge");
  });
}

int or_lu_solve_dense(int n, const double* A, const double* b, double* x) {
  return guarded([&] {
    Mat M(n, n);
    std::memcpy(M.a.data(), A, sizeof(double) * n * n);
    const LU f = lu_factor(M);
    if (f.singular) throw std::runtime_error("lu: singular");
    const Vec r = lu_solve(f, Vec(b, b + n));
    std::memcpy(x, r.data(), sizeof(double) * n);
  });
}

}  // extern "C"
