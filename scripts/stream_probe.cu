// Streaming ceiling at the c4 R(U) traffic shape: read U (n_dof doubles) and
// u_n (n_sdof, broadcast over the n_tau blocks), write R (n_dof): the
// 150,994,944 algorithmic bytes of one R(U) apply, with three rotating
// buffer sets (> L2).  Vector widths 16 / 32 bytes, several grid sizes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr long long NS = 2097152, NT = 4, ND = NS * NT;

template <int V>
__global__ void __launch_bounds__(256) k_rlike(double* __restrict__ R, const double* __restrict__ U,
                                               const double* __restrict__ un) {
  const long long nv = ND / V;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nv;
       i += (long long)gridDim.x * blockDim.x) {
    const long long e = i * V;
    const long long s = e % NS;
    double x[V], w[V];
    if constexpr (V == 2) {
      const double2 a = __ldcs(reinterpret_cast<const double2*>(U) + i);
      const double2 b = __ldg(reinterpret_cast<const double2*>(un + s));
      x[0] = a.x; x[1] = a.y; w[0] = b.x; w[1] = b.y;
    } else {
      asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3]) : "l"(U + e));
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(w[0]), "=d"(w[1]), "=d"(w[2]), "=d"(w[3]) : "l"(un + s));
    }
#pragma unroll
    for (int q = 0; q < V; ++q) x[q] = fma(0.5, x[q], -w[q]);
    if constexpr (V == 2) {
      __stcs(reinterpret_cast<double2*>(R) + i, make_double2(x[0], x[1]));
    } else {
      asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(R + e), "d"(x[0]), "d"(x[1]), "d"(x[2]), "d"(x[3]) : "memory");
    }
  }
}

int main() {
  double *U[3], *un[3], *R[3];
  for (int k = 0; k < 3; ++k) {
    cudaMalloc(&U[k], ND * 8); cudaMalloc(&R[k], ND * 8); cudaMalloc(&un[k], NS * 8);
    cudaMemset(U[k], 0, ND * 8); cudaMemset(un[k], 0, NS * 8);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double bytes = 8.0 * (2 * ND + NS);
  printf("{");
  bool first = true;
  for (int v : {2, 4})
    for (int per : {2, 4, 8, 16, 32}) {
      const int grid = 148 * per;
      auto run = [&](int k) {
        if (v == 2) k_rlike<2><<<grid, 256>>>(R[k % 3], U[k % 3], un[k % 3]);
        else k_rlike<4><<<grid, 256>>>(R[k % 3], U[k % 3], un[k % 3]);
      };
      for (int k = 0; k < 10; ++k) run(k);
      cudaDeviceSynchronize();
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        for (int k = 0; k < 20; ++k) run(k);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const double us = best * 1e3 / 20;
      printf("%s\"v%d_g%d\": [%.2f, %.1f]", first ? "" : ", ", v * 8, grid, us, bytes / (us * 1e-6) / 1e9);
      first = false;
    }
  printf("}\n");
  return 0;
}
