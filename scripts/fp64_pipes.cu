// Microbenchmark: FP64 throughput of DFMA (FP64 pipe) and DMMA
// (mma.sync.m8n8k4.f64, tensor pipe) on sm_100a, alone and interleaved --
// do they share hardware?  Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_pipes fp64_pipes.cu
#include <cstdio>

#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <bool FMA, bool MMA>
__global__ void __launch_bounds__(256) k(double* out, double seed) {
  double f[16];
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = seed + i + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = seed * i;
  const double a = seed * 1.0001, b = seed * 0.9999;
  for (int it = 0; it < ITERS; ++it) {
    if (MMA) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i], a, b);
    }
    if (FMA) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] = fma(f[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += f[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <bool FMA, bool MMA>
float run(double* out, int blocks) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<FMA, MMA><<<blocks, 256>>>(out, 1.0);
  cudaEventRecord(e0);
  k<FMA, MMA><<<blocks, 256>>>(out, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  double* out;
  cudaMalloc(&out, 4096);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8;  // 64 warps per SM
  const double threads = double(blocks) * 256;
  const double fma_flops = threads * ITERS * 64 * 2;         // 64 DFMA per iteration
  const double mma_flops = double(blocks) * 8 * ITERS * 8 * 512 * 2 / 1.0;  // per warp: 8 mma of 8x8x4 = 256 FMA
  const float t_f = run<true, false>(out, blocks);
  const float t_m = run<false, true>(out, blocks);
  const float t_b = run<true, true>(out, blocks);
  // mma_flops: warps = blocks * 8; each mma m8n8k4 = 8*8*4 = 256 FMA = 512 flop
  const double mflops = double(blocks) * 8 * ITERS * 8 * 512;
  std::printf("{\"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"both_ms\": %.3f, \"dfma_ms\": %.3f, "
              "\"dmma_ms\": %.3f, \"both_tflops\": %.2f, \"err\": \"%s\"}\n",
              fma_flops / (t_f * 1e9), mflops / (t_m * 1e9), t_b, t_f, t_m,
              (fma_flops + mflops) / (t_b * 1e9), cudaGetErrorString(cudaGetLastError()));
  (void)mma_flops;
  return 0;
}
