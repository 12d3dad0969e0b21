// End-to-end c4 slab solve through the C++ mirror of the reference API
// (include/stdgsem_gpu.hpp), as a caller of the reference's stdg_step
// (stdg.hpp:120-143) would do it: Vec u_n in, fresh Vec U / u_next out every
// call (Vec's allocator recycles page-locked blocks).  Beside it, the same
// solve through the C ABI on fresh std::vector<double> results (pageable,
// zero-filled: what the call cost before Vec had its allocator).  bench.py
// compiles and runs this and records the JSON line it prints.
#include <chrono>
#include <cmath>
#include <cstdio>

#include "stdgsem_gpu.hpp"

using namespace stdgsem::gpu;

int main() {
  const DgSpace space = dg_space(uniform_mesh(3, {0, 0, 0}, {1, 1, 1}, {32, 32, 32}), 3);
  const SemiDiscreteSystem sys = assemble_semidiscrete(space, advection_model({1, 1, 1}));
  const Vec un = interpolate_scalar(space, [](const Vec& x) {
                   return std::sin(2.0 * M_PI * (x[0] + x[1] + x[2]));
                 }).coeffs;
  NewtonConfig cfg;
  cfg.abs_tol = 0.0;
  cfg.rel_tol = 1e-9;
  cfg.gmres_tol = 1e-10;
  StdgStepResult r = stdg_step(sys, sbp_operators(4), 0.0, un, 0.002, cfg);  // warm
  double best = 1e30;
  for (int k = 0; k < 6; ++k) {
    const auto t0 = std::chrono::steady_clock::now();
    r = stdg_step(sys, sbp_operators(4), 0.0, un, 0.002, cfg);
    const auto t1 = std::chrono::steady_clock::now();
    best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
  }
  // the same call on pageable vectors through the C ABI
  SlabOperator& o = sys.op(4);
  const std::vector<double> un_p(un.begin(), un.end());
  const stg_newton_config c = cfg.c();
  double best_p = 1e30;
  bool same = true;
  for (int k = 0; k < 3; ++k) {
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<double> U(o.n_dof()), u1(o.n_sdof());
    stg_solve_info info{};
    check(stg_stdg_step_host(o.handle(), 0.0, 0.002, un_p.data(), &c, U.data(), u1.data(), &info),
          o.handle());
    const auto t1 = std::chrono::steady_clock::now();
    best_p = std::min(best_p, std::chrono::duration<double>(t1 - t0).count());
    for (size_t i = 0; i < u1.size(); ++i) same = same && u1[i] == r.u_next[i];
  }
  std::printf("{\"seconds\": %.9g, \"newton\": %d, \"gmres_iterations\": %d, "
              "\"path\": \"stdgsem::gpu::stdg_step (Vec in, fresh Vec results per call; "
              "page-locked blocks recycled by Vec's allocator)\", "
              "\"fresh_std_vector_seconds\": %.9g, \"results_bitwise_equal\": %s}\n",
              best, r.newton_iterations, r.linear_iterations, best_p, same ? "true" : "false");
  return 0;
}
