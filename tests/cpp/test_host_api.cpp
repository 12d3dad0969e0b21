// C++ tests of the reference-mirroring host API (include/stdgsem_gpu.hpp),
// written like the reference's own doctest cases (test_stdg.cpp,
// test_lodg.cpp) but with a tiny local CHECK harness (doctest is absent).
// Built and run by tests/test_cpp_host_api.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>

#include "stdgsem_gpu.hpp"

using namespace stdgsem::gpu;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    if (cond) {                                                          \
      ++g_pass;                                                          \
    } else {                                                             \
      ++g_fail;                                                          \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
    }                                                                    \
  } while (0)

static double maxabs(const Vec& a) {
  double m = 0;
  for (double x : a) m = std::max(m, std::abs(x));
  return m;
}
static double maxdiff(const Vec& a, const Vec& b) {
  double m = 0;
  for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
  return m;
}
static double norm2(const Vec& a) {
  double s = 0;
  for (double x : a) s += x * x;
  return std::sqrt(s);
}

static SemiDiscreteSystem advection_1d(int cells, int p) {  // test_stdg.cpp:23-28
  return assemble_semidiscrete(dg_space(uniform_mesh(1, {0.0}, {1.0}, {cells}), p),
                               advection_model({1.0}));
}

// interpolate_scalar of a 1-D profile on [0, 1] (mesh.hpp:145-165)
static Vec interp_1d(int cells, int p, double (*f)(double)) {
  const DgSpace s = dg_space(uniform_mesh(1, {0.0}, {1.0}, {cells}), p);
  return interpolate_scalar(s, [&](const Vec& x) { return f(x[0]); }).coeffs;
}

static bool near(double a, double b, double eps) {  // doctest::Approx(b).epsilon(eps)
  return std::abs(a - b) <= eps * (1.0 + std::max(std::abs(a), std::abs(b)));
}
static DgSpace unit_interval(int n, int p, int r = 1) {
  return dg_space(uniform_mesh(1, {0.0}, {1.0}, {n}), p, r);
}
static DgSpace unit_square(int n, int p, int r = 1) {
  return dg_space(uniform_mesh(2, {0.0, 0.0}, {1.0, 1.0}, {n, n}), p, r);
}

// ---- host-side field helpers: test_mesh.cpp:70-190 (no device needed) --------
static void test_node_coords() {  // test_mesh.cpp:70-86
  CHECK(near(node_coord(unit_interval(10, 1), 3, 0)[0], 0.3, 1e-14));
  CHECK(near(node_coord(unit_interval(10, 1), 3, 1)[0], 0.4, 1e-14));
  CHECK(near(node_coord(unit_interval(10, 2), 0, 1)[0], 0.05, 1e-14));
  const DgSpace s3 = unit_square(4, 2, 3);
  CHECK(s3.dof() == 3 * 16 * 9);
  const Vec x = node_coord(s3, /*cell (1,0)*/ 1, /*node (2,0)*/ 2);
  CHECK(near(x[0], 0.5, 1e-14) && near(x[1], 0.0, 1e-14));
  // d = 3 extension: cell (cz*ny + cy)*nx + cx, node (iz*n + iy)*n + ix
  const DgSpace c = dg_space(uniform_mesh(3, {0, 0, 0}, {1, 2, 4}, {2, 2, 2}), 1);
  const Vec y = node_coord(c, (1 * 2 + 0) * 2 + 1, (1 * 2 + 0) * 2 + 1);
  CHECK(near(y[0], 1.0, 1e-15) && near(y[1], 0.0, 1e-15) && near(y[2], 4.0, 1e-15));
}

static void test_global_mass() {  // test_mesh.cpp:98-113
  for (int p : {1, 2, 3}) {
    const auto m1 = global_mass(unit_interval(8, p));
    double s1 = 0.0, mn = 1.0;
    for (double v : m1.diag) s1 += v, mn = std::min(mn, v);
    CHECK(mn > 0.0 && near(s1, 1.0, 1e-12));
    const auto m2 = global_mass(unit_square(5, p, 4));
    double s2 = 0.0;
    for (double v : m2.diag) s2 += v;
    CHECK(near(s2, 4.0, 1e-12));
    const auto m3 = global_mass(dg_space(uniform_mesh(3, {0, 0, 0}, {1, 1, 2}, {3, 2, 2}), p));
    double s3 = 0.0;
    for (double v : m3.diag) s3 += v;
    CHECK(near(s3, 2.0, 1e-12));
  }
  const DgSpace s = unit_square(2, 2);
  CHECK(near(global_mass(s).diag[size_t(1 * 3 + 1)], 0.0625 * 16.0 / 9.0, 1e-14));
}

static void test_interpolate_and_l2() {  // test_mesh.cpp:115-190
  const auto constant = interpolate_scalar(unit_interval(1, 1), [](const Vec&) { return 3.0; });
  CHECK(constant.coeffs[0] == 3.0 && constant.coeffs[1] == 3.0);
  const auto lin = interpolate_scalar(unit_interval(1, 1), [](const Vec& x) { return x[0]; });
  CHECK(near(lin.coeffs[0], 0.0, 1e-14) && near(lin.coeffs[1], 1.0, 1e-14));
  CHECK(l2_norm(interpolate_scalar(unit_interval(4, 2), [](const Vec&) { return 0.0; })) == 0.0);
  CHECK(near(l2_norm(interpolate_scalar(unit_interval(4, 2), [](const Vec&) { return 1.0; })),
             1.0, 1e-13));
  for (int p : {1, 2, 3})
    CHECK(near(l2_norm(interpolate_scalar(unit_square(3, p), [](const Vec&) { return 2.0; })),
               2.0, 1e-13));
  auto exact = [](const Vec& x, double t) { return Vec{std::cos(x[0] + t)}; };
  const DgSpace s = unit_interval(6, 2);
  const auto field = interpolate(s, [&](const Vec& x) { return exact(x, 0.75); }, 0.75);
  CHECK(l2_error(field, exact, 0.75) <= 1e-14);
  const auto flat = interpolate_scalar(s, [](const Vec&) { return 1.0; });
  CHECK(near(l2_error(flat, [](const Vec&, double) { return Vec{1.125}; }, 0.0), 0.125, 1e-13));
  // r = 4 (component-innermost coefficients, test_mesh.cpp:88-96)
  const auto f4 = interpolate(unit_square(2, 1, 4),
                              [](const Vec& x) { return Vec{1.0, x[0], x[1], 2.0}; });
  CHECK(f4.coeffs.size() == size_t(4 * 4 * 4));
  CHECK(f4.coeffs[4 * 1 + 1] == node_coord(unit_square(2, 1, 4), 0, 1)[0]);
  CHECK(f4.coeffs[3] == 2.0);
}

static void test_stdg_equals_rk() {  // test_stdg.cpp:111-135
  auto adv = advection_1d(8, 2);
  const Vec u0 = interp_1d(8, 2, [](double x) { return std::sin(2 * M_PI * x) + 0.3; });
  NewtonConfig tight;
  tight.abs_tol = 1e-14;
  tight.rel_tol = 1e-13;
  tight.gmres_tol = 1e-14;
  for (int n_tau : {2, 3}) {
    auto a = stdg_step(adv, sbp_operators(n_tau), 0.0, u0, 0.05, tight);
    auto b = rk_step(adv, lobatto_tableau(n_tau), 0.0, u0, 0.05, tight, JacobianForm::a_inv_form);
    Vec d(a.u_next.size());
    for (size_t i = 0; i < d.size(); ++i) d[i] = a.u_next[i] - b.u_next[i];
    CHECK(norm2(d) / norm2(b.u_next) <= 1e-10);
    const size_t ns = u0.size();
    for (int j = 0; j < n_tau; ++j) {
      Vec aj(a.U.begin() + long(j * ns), a.U.begin() + long((j + 1) * ns));
      CHECK(maxdiff(aj, b.stages[size_t(j)]) <= 1e-9);
    }
  }
}

static void test_st_residual_constant_and_dt() {  // test_stdg.cpp:53-73
  auto adv = advection_1d(4, 1);
  const int dof = adv.dof();
  TimeElementSystem e0{adv, sbp_operators(3), 0.0, 0.25, Vec(size_t(dof), 2.5)};
  CHECK(maxabs(st_residual(e0, Vec(size_t(3 * dof), 2.5))) <= 1e-12);
  Vec U(size_t(3 * dof));
  for (int i = 0; i < 3 * dof; ++i) U[size_t(i)] = -0.7 + 2.0 * i / (3 * dof - 1);
  TimeElementSystem e1{adv, sbp_operators(3), 0.0, 0.1, Vec(size_t(dof), 0.0)};
  TimeElementSystem e2{adv, sbp_operators(3), 0.0, 0.2, Vec(size_t(dof), 0.0)};
  const double w3[3] = {1.0 / 3, 4.0 / 3, 1.0 / 3};
  Vec R1 = st_residual(e1, U), R2 = st_residual(e2, U);
  double worst = 0.0;
  for (int i = 0; i < 3; ++i) {
    Vec Ui(U.begin() + i * dof, U.begin() + (i + 1) * dof);
    const Vec F = adv.rhs(0.0, Ui);
    for (int k = 0; k < dof; ++k)
      worst = std::max(worst, std::abs(R2[size_t(i * dof + k)] - R1[size_t(i * dof + k)] +
                                       0.05 * w3[i] * F[size_t(k)]));
  }
  CHECK(worst <= 1e-14);
}

static void test_st_jacobian_fd() {  // test_stdg.cpp:88-109
  auto adv = advection_1d(4, 1);
  const int dof = adv.dof();
  Vec un(static_cast<size_t>(dof));
  for (int i = 0; i < dof; ++i) un[size_t(i)] = 0.1 + 0.8 * i / (dof - 1);
  TimeElementSystem elem{adv, sbp_operators(3), 0.2, 0.13, un};
  Vec U(size_t(3 * dof));
  for (int i = 0; i < 3 * dof; ++i) U[size_t(i)] = std::sin(0.7 * i + 0.3);
  std::mt19937 gen(17);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  const double h = 1e-6;
  for (int trial = 0; trial < 3; ++trial) {
    Vec v(U.size()), Up(U), Um(U);
    for (size_t i = 0; i < v.size(); ++i) {
      v[i] = dist(gen);
      Up[i] += h * v[i];
      Um[i] -= h * v[i];
    }
    const Vec rp = st_residual(elem, Up), rm = st_residual(elem, Um);
    const Vec jv = st_jacobian_apply(elem, U, v);
    double worst = 0.0;
    for (size_t i = 0; i < v.size(); ++i)
      worst = std::max(worst, std::abs((rp[i] - rm[i]) / (2 * h) - jv[i]));
    CHECK(worst <= 1e-6 * (1.0 + maxabs(jv)));
  }
}

static void test_integrate_basics() {  // test_stdg.cpp:169-192, test_lodg.cpp:159-175
  auto adv = advection_1d(8, 1);
  const Vec u0 = interp_1d(8, 1, [](double x) { return std::cos(2 * M_PI * x); });
  bool threw = false;
  try {
    stdg_integrate(adv, sbp_operators(2), 0.0, u0, 1.0, 0);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  auto tr = stdg_integrate(adv, sbp_operators(2), 0.0, u0, 1.0, 4);
  CHECK(tr.times.size() == 5);
  for (int k = 0; k <= 4; ++k) CHECK(tr.times[size_t(k)] == 0.25 * k);
  CHECK(tr.states.size() == 5);
  CHECK(tr.element_solutions.size() == 4);
  auto rk = integrate(adv, lobatto_tableau(2), 0.0, u0, 1.0, 4);
  CHECK(rk.stage_solutions.size() == 4 && rk.stage_solutions[0].size() == 2);
}

static void test_rk_stiffly_accurate_and_forms() {  // test_lodg.cpp:64-95
  auto adv = advection_1d(16, 2);
  const Vec u0 = interp_1d(16, 2, [](double x) { return std::sin(2 * M_PI * x); });
  for (auto form : {JacobianForm::a_form, JacobianForm::a_inv_form}) {
    auto st = rk_step(adv, lobatto_tableau(3), 0.0, u0, 0.01, {}, form);
    CHECK(maxdiff(st.u_next, st.stages.back()) <= 1e-12);
  }
  auto adv8 = advection_1d(8, 2);
  const Vec v0 = interp_1d(8, 2, [](double x) { return std::exp(std::sin(2 * M_PI * x)); });
  for (int s : {2, 3}) {
    auto a = rk_step(adv8, lobatto_tableau(s), 0.0, v0, 0.05, {}, JacobianForm::a_form);
    auto b = rk_step(adv8, lobatto_tableau(s), 0.0, v0, 0.05, {}, JacobianForm::a_inv_form);
    Vec d(a.u_next.size());
    for (size_t i = 0; i < d.size(); ++i) d[i] = a.u_next[i] - b.u_next[i];
    CHECK(norm2(d) / norm2(b.u_next) <= 1e-11);
  }
}

static void test_linear_one_newton_iteration() {  // test_lodg.cpp:123-132
  auto adv = advection_1d(8, 1);
  const Vec u0 = interp_1d(8, 1, [](double x) { return std::cos(2 * M_PI * x); });
  NewtonConfig cfg;
  cfg.gmres_tol = 1e-14;
  for (auto form : {JacobianForm::a_form, JacobianForm::a_inv_form})
    CHECK(rk_step(adv, lobatto_tableau(2), 0.0, u0, 0.1, cfg, form).newton_iterations == 1);
}

static void test_nonconvergence_context() {  // test_lodg.cpp:179-194
  auto adv = advection_1d(8, 1);
  const Vec u0 = interp_1d(8, 1, [](double x) { return std::cos(2 * M_PI * x); });
  NewtonConfig cfg;
  cfg.max_iter = 0;
  bool threw = false;
  try {
    rk_step(adv, lobatto_tableau(2), 0.5, u0, 0.1, cfg);
  } catch (const NonconvergenceError& e) {
    threw = true;
    CHECK(std::string(e.what()).find("rk_step at t=0.5") != std::string::npos);
    CHECK(e.residual_history.size() == 1);
    // newton.hpp:40-48: the last iterate is the initial guess 1 (x) u here
    CHECK(e.last_iterate.size() == 2 * u0.size());
    CHECK(maxdiff(Vec(e.last_iterate.begin(), e.last_iterate.begin() + long(u0.size())), u0) == 0.0);
  }
  CHECK(threw);
  // one Newton step allowed on a 3-D slab (host-driven path): the last
  // iterate is that step's result, and its residual is the history's tail
  {
    auto sys = assemble_semidiscrete(
        dg_space(uniform_mesh(3, {0, 0, 0}, {1, 1, 1}, {8, 4, 4}), 3), advection_model({1, 1, 1}));
    const DgSpace& sp = dg_space(uniform_mesh(3, {0, 0, 0}, {1, 1, 1}, {8, 4, 4}), 3);
    const Vec un = interpolate_scalar(sp, [](const Vec& x) {
                     return std::sin(2 * M_PI * (x[0] + x[1] + x[2]));
                   }).coeffs;
    NewtonConfig one;
    one.max_iter = 1;
    one.abs_tol = 0.0;
    one.rel_tol = 1e-30;  // unreachable after one step
    one.gmres_tol = 1e-3;
    bool t3 = false;
    try {
      stdg_step(sys, sbp_operators(4), 0.0, un, 0.002, one);
    } catch (const NonconvergenceError& e) {
      t3 = true;
      CHECK(e.residual_history.size() == 2);
      TimeElementSystem el{sys, sbp_operators(4), 0.0, 0.002, un};
      CHECK(e.last_iterate.size() == 4 * un.size());
      if (e.last_iterate.size() == 4 * un.size())
        CHECK(near(maxabs(st_residual(el, e.last_iterate)), e.residual_history[1], 1e-12));
    }
    CHECK(t3);
  }
  bool inv = false;
  try {
    uniform_mesh(4, {0, 0, 0, 0}, {1, 1, 1, 1}, {2, 2, 2, 2});
  } catch (const std::invalid_argument&) {
    inv = true;
  }
  CHECK(inv);
  bool bad_dt = false;
  try {
    stdg_step(adv, sbp_operators(2), 0.0, u0, -0.1);
  } catch (const std::invalid_argument&) {
    bad_dt = true;
  }
  CHECK(bad_dt);
}

static void test_3d_free_stream() {  // EXTENSION: d = 3 (acceptance.cpp:334-343 analogue)
  auto sys = assemble_semidiscrete(
      dg_space(uniform_mesh(3, {0, 0, 0}, {1, 1, 1}, {8, 4, 4}), 3), advection_model({1, 1, 1}));
  const int dof = sys.dof();
  TimeElementSystem e{sys, sbp_operators(4), 0.0, 0.002, Vec(size_t(dof), 0.37)};
  CHECK(maxabs(st_residual(e, Vec(size_t(4 * dof), 0.37))) <= 1e-12);
}

static void test_general_models() {  // test_spatial.cpp:67-89, models.hpp:108-113
  auto pulse = assemble_semidiscrete(dg_space(uniform_mesh(2, {0, 0}, {1, 1}, {5, 5}), 3),
                                     advdiff_model(2, rotating_field(), 0.001));
  CHECK(pulse.eta() == 90.0);
  CHECK(maxabs(pulse.rhs(0.0, Vec(size_t(pulse.dof()), -0.6))) <= 1e-12);
  auto euler = assemble_semidiscrete(
      dg_space(uniform_mesh(2, {-10, -10}, {10, 10}, {4, 4}), 1, 4), euler_model(1.4));
  Vec c3(size_t(euler.dof()));
  for (size_t i = 0; i < c3.size(); i += 4) {
    c3[i] = 1.0;
    c3[i + 1] = 0.3;
    c3[i + 2] = -0.2;
    c3[i + 3] = 2.5;
  }
  CHECK(maxabs(euler.rhs(0.0, c3)) <= 1e-12);
  Vec bad = c3;
  for (size_t i = 0; i < bad.size(); i += 4) bad[i + 1] = 4.0, bad[i + 3] = 1.0;
  bool threw = false;
  try {
    euler.rhs(0.0, bad);
  } catch (const AdmissibilityError&) {
    threw = true;
  }
  CHECK(threw);
  bool mismatch = false;
  try {
    assemble_semidiscrete(dg_space(uniform_mesh(1, {0}, {1}, {4}), 1, 4), euler_model());
  } catch (const std::invalid_argument&) {
    mismatch = true;
  }
  CHECK(mismatch);
}

// Vec's allocator: large blocks are page-locked and recycled by size when a
// device is present, plain malloc otherwise; either way a vector works.
static void test_vec_allocator(bool device) {
  const size_t n = size_t(1) << 17;  // 1 MiB: above the page-locking threshold
  const double *first = nullptr, *second = nullptr;
  {
    Vec a(n, 1.5);
    first = a.data();
    double s = 0.0;
    for (double v : a) s += v;
    CHECK(s == 1.5 * double(n));
    Vec b(a);  // a second live block of the same size
    CHECK(b.data() != a.data() && b[n - 1] == 1.5);
    second = b.data();
  }
  Vec c(n);  // uninitialised, like Eigen::VectorXd(n)
  c[0] = 2.0;
  CHECK(c[0] == 2.0);
  if (device) CHECK(c.data() == first || c.data() == second);  // recycled by size
  Vec small(3, 0.25), grown;
  for (int i = 0; i < 100000; ++i) grown.push_back(double(i));  // crosses the threshold
  CHECK(small[2] == 0.25 && grown[99999] == 99999.0);
}

static void test_vec_pool_recycles() {  // needs a device
  const size_t n = size_t(1) << 18;
  const double* p0;
  { Vec a(n); p0 = a.data(); }
  Vec b(n);
  CHECK(b.data() == p0);  // the freed page-locked block is handed out again
}

int main(int argc, char** argv) {
  test_node_coords();
  test_global_mass();
  test_interpolate_and_l2();
  if (argc > 1 && std::string(argv[1]) == "--host-only") {  // no device needed
    test_vec_allocator(false);
    std::printf("passed %d failed %d\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
  }
  test_vec_allocator(true);
  test_vec_pool_recycles();
  test_stdg_equals_rk();
  test_st_residual_constant_and_dt();
  test_st_jacobian_fd();
  test_integrate_basics();
  test_rk_stiffly_accurate_and_forms();
  test_linear_one_newton_iteration();
  test_nonconvergence_context();
  test_3d_free_stream();
  test_general_models();
  std::printf("passed %d failed %d\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
