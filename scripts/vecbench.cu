// Microbenchmark of the GMRES vector kernels at the c4 vector length
// (n = 8,388,608 doubles): event-timed multidot and update+normalise for
// k = 1..12 basis vectors, against a device-to-device copy.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2201_05800_b200/csrc \
//        scripts/vecbench.cu -L paper_2201_05800_b200 -lstg_cuda -Xlinker -rpath=<lib dir>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "kernels.hpp"

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      std::printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

// ---- prototype: thread-per-chunk, exact-k template ------------------------
namespace proto {
constexpr int TB = 256;
__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
template <int K>
__global__ void __launch_bounds__(TB) multidot(const double* __restrict__ V, long long ldv,
                                               const double* __restrict__ w, long long n2,
                                               double* part, double* out, unsigned* counter) {
  double acc[K + 1];
#pragma unroll
  for (int j = 0; j <= K; ++j) acc[j] = 0.0;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  for (long long i = blockIdx.x * (long long)TB + threadIdx.x; i < n2;
       i += (long long)gridDim.x * TB) {
    const double2 x = __ldcs(w2 + i);
    double2 v[K];
#pragma unroll
    for (int j = 0; j < K; ++j) v[j] = __ldcs(reinterpret_cast<const double2*>(V + j * ldv) + i);
#pragma unroll
    for (int j = 0; j < K; ++j) acc[j] = fma(v[j].x, x.x, fma(v[j].y, x.y, acc[j]));
    acc[K] = fma(x.x, x.x, fma(x.y, x.y, acc[K]));
  }
  __shared__ double red[TB / 32][K + 1];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j <= K; ++j) {
    const double s = wsum(acc[j]);
    if (lane == 0) red[wp][j] = s;
  }
  __syncthreads();
  if (threadIdx.x <= K) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < TB / 32; ++q) s += red[q][threadIdx.x];
    part[(size_t)blockIdx.x * (K + 1) + threadIdx.x] = s;
  }
  __shared__ unsigned last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  for (int j = wp; j <= K; j += TB / 32) {
    double s = 0.0;
    for (int bb = lane; bb < (int)gridDim.x; bb += 32) s += __ldcg(part + (size_t)bb * (K + 1) + j);
    s = wsum(s);
    if (lane == 0) out[j] = s;
  }
  if (threadIdx.x == 0) *counter = 0u;
}
template <int K>
__global__ void __launch_bounds__(TB) update(double* __restrict__ w, const double* __restrict__ V,
                                             long long ldv, const double* __restrict__ h,
                                             long long n2, double* part, double* out,
                                             unsigned* counter) {
  __shared__ double hs[K + 1];
  if (threadIdx.x <= K) hs[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  double hh = 0.0;
#pragma unroll
  for (int j = 0; j < K; ++j) hh = fma(hs[j], hs[j], hh);
  const double est = hs[K] - hh;
  const double sc = est > 1e-28 * hs[K] ? 1.0 / sqrt(est) : 1.0;
  double nrm = 0.0;
  double2* w2 = reinterpret_cast<double2*>(w);
  for (long long i = blockIdx.x * (long long)TB + threadIdx.x; i < n2;
       i += (long long)gridDim.x * TB) {
    double2 x = __ldcs(w2 + i);
    double2 v[K];
#pragma unroll
    for (int j = 0; j < K; ++j) v[j] = __ldcs(reinterpret_cast<const double2*>(V + j * ldv) + i);
#pragma unroll
    for (int j = 0; j < K; ++j) {
      x.x = fma(-hs[j], v[j].x, x.x);
      x.y = fma(-hs[j], v[j].y, x.y);
    }
    x.x *= sc;
    x.y *= sc;
    __stcs(w2 + i, x);
    nrm = fma(x.x, x.x, fma(x.y, x.y, nrm));
  }
  __shared__ double red[TB / 32];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  nrm = wsum(nrm);
  if (lane == 0) red[wp] = nrm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < TB / 32; ++q) s += red[q];
    part[blockIdx.x] = s;
  }
  __shared__ unsigned last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last || wp) return;
  double s = 0.0;
  for (int bb = lane; bb < (int)gridDim.x; bb += 32) s += __ldcg(part + bb);
  s = wsum(s);
  if (lane == 0) {
    out[0] = s;
    *counter = 0u;
  }
}
template <int K>
void run(int grid, double* V, double* w, double* h, long long n, double* part, double* out,
         unsigned* c, bool upd) {
  if (upd)
    update<K><<<grid, TB>>>(w, V, n, h, n / 2, part, out, c);
  else
    multidot<K><<<grid, TB>>>(V, n, w, n / 2, part, out, c);
}
void dispatch(int k, int grid, double* V, double* w, double* h, long long n, double* part,
              double* out, unsigned* c, bool upd) {
  switch (k) {
#define C_(K) case K: run<K>(grid, V, w, h, n, part, out, c, upd); break;
    C_(1) C_(2) C_(3) C_(4) C_(5) C_(6) C_(7) C_(8) C_(9) C_(10) C_(11) C_(12)
#undef C_
  }
}
}  // namespace proto

int main() {
  const long long n = 8388608;
  const int kmax = 12;
  double *V, *w, *w2, *part, *out, *h;
  CK(cudaMalloc(&V, sizeof(double) * n * (kmax + 1)));
  CK(cudaMalloc(&w, sizeof(double) * n));
  CK(cudaMalloc(&w2, sizeof(double) * n));
  CK(cudaMalloc(&part, sizeof(double) * (stg::kPartialDoubles + 8)));
  CK(cudaMalloc(&out, sizeof(double) * 64));
  CK(cudaMalloc(&h, sizeof(double) * 64));
  CK(cudaMemset(part, 0, sizeof(double) * (stg::kPartialDoubles + 8)));
  stg::vec_fill(V, 1e-3, n * (kmax + 1), 0);
  stg::vec_fill(w, 1.0, n, 0);
  stg::vec_fill(h, 1e-6, 64, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 20;
  float ms;
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r)
    cudaMemcpyAsync(r & 1 ? w2 : w, r & 1 ? w : w2, sizeof(double) * n, cudaMemcpyDeviceToDevice);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  cudaEventElapsedTime(&ms, a, b);
  std::printf("{\"copy_gbs\": %.1f", 16.0 * n * reps / (ms * 1e-3) / 1e9);
  for (int k = 1; k <= kmax; ++k) {
    // warm-up (module load) outside the timed region
    stg::vec_multidot(V, n, k, w, n, part, out, 0);
    stg::vec_update_dot(w, V, n, k, h, n, 0, part, out, 0, h, out + 32);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) stg::vec_multidot(V, n, k, w, n, part, out, 0);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    const double us_d = 1e3 * ms / reps;
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r)
      stg::vec_update_dot(w, V, n, k, h, n, 0, part, out, 0, h, out + 32);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    const double us_u = 1e3 * ms / reps;
    double pd[3], pu[3];
    unsigned* cnt = reinterpret_cast<unsigned*>(part + stg::kPartialDoubles);
    const int grids[3] = {148 * 4, 148 * 8, 148 * 16};
    for (int gi = 0; gi < 3; ++gi) {
      for (int upd = 0; upd < 2; ++upd) {
        proto::dispatch(k, grids[gi], V, w, h, n, part, out, cnt, upd);
        cudaEventRecord(a);
        for (int r = 0; r < reps; ++r) proto::dispatch(k, grids[gi], V, w, h, n, part, out, cnt, upd);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        (upd ? pu : pd)[gi] = 1e3 * ms / reps;
      }
    }
    std::printf(", \"k%d\": {\"multidot_gbs\": %.0f, \"update_gbs\": %.0f, \"proto_multidot_gbs\": "
                "[%.0f, %.0f, %.0f], \"proto_update_gbs\": [%.0f, %.0f, %.0f]}",
                k, 8.0 * n * (k + 1) / us_d / 1e3, 8.0 * n * (k + 2) / us_u / 1e3,
                8.0 * n * (k + 1) / pd[0] / 1e3, 8.0 * n * (k + 1) / pd[1] / 1e3,
                8.0 * n * (k + 1) / pd[2] / 1e3, 8.0 * n * (k + 2) / pu[0] / 1e3,
                8.0 * n * (k + 2) / pu[1] / 1e3, 8.0 * n * (k + 2) / pu[2] / 1e3);
  }
  std::printf("}\n");
  CK(cudaGetLastError());
  return 0;
}
