// End-to-end c4 slab solve through the C++ mirror of the reference API
// (include/stdgsem_gpu.hpp): std::vector u_n in, std::vector U / u_next out
// (pageable host memory, copies inside stg_stdg_step_host), as a caller of
// the reference's stdg_step (stdg.hpp:120-143) would do it.  bench.py
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
  for (int k = 0; k < 3; ++k) {
    const auto t0 = std::chrono::steady_clock::now();
    r = stdg_step(sys, sbp_operators(4), 0.0, un, 0.002, cfg);
    const auto t1 = std::chrono::steady_clock::now();
    best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
  }
  std::printf("{\"seconds\": %.9g, \"newton\": %d, \"gmres_iterations\": %d, "
              "\"path\": \"stdgsem::gpu::stdg_step (std::vector in/out, pageable)\"}\n",
              best, r.newton_iterations, r.linear_iterations);
  return 0;
}
