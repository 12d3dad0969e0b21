// PCIe schedule probe for the host-buffer R(U) call at c4 sizes (U: 4 temporal
// blocks of 32 z-layers x 512 KiB, u_n: 32 layers x 512 KiB in; R like U out).
// Copy-only schedules (no compute), each the best of 5 rounds of 10 calls:
//   duplex          one H2D of U + u_n and one D2H of R, on two streams
//   chain K/nin/nout K z-chunks (ramp 1,2,4,8,..,8,4,2,1 or uniform), chunk k's
//                   D2H waits on chunk k's H2D; H2D chunks alternate over nin
//                   streams and D2H chunks over nout streams
//   zc_*            zero-copy: a kernel reads mapped pinned host memory or
//                   writes it (the SMs issue the PCIe traffic, no copy engine)
// nvcc -O2 -gencode arch=compute_100a,code=sm_100a scripts/pcie_sched.cu -o /tmp/pcie_sched
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <functional>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); std::exit(1); } } while (0)

constexpr int NT = 4, NZ = 32;
constexpr size_t LAYER = 65536;                // doubles per z-layer per block
constexpr size_t NS = LAYER * NZ, ND = NS * NT;

double *hU, *hu, *hR, *dU, *du, *dR;
cudaStream_t st[8], mainS;
cudaEvent_t ev[64], evm;

float timed(const std::function<void()>& f) {
  f();
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a, mainS);
    for (int i = 0; i < 10; ++i) f();
    cudaEventRecord(b, mainS);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = std::min(best, ms / 10);
  }
  return best;
}

void fork(int n) {
  cudaEventRecord(evm, mainS);
  for (int i = 0; i < n; ++i) cudaStreamWaitEvent(st[i], evm, 0);
}
void join(int n) {
  for (int i = 0; i < n; ++i) {
    cudaEventRecord(ev[63], st[i]);
    cudaStreamWaitEvent(mainS, ev[63], 0);
  }
}

std::vector<int> bounds(int K, bool ramp) {
  std::vector<double> w(K);
  double ws = 0;
  for (int k = 0; k < K; ++k) {
    int d = std::min(k, K - 1 - k);
    w[k] = ramp ? double(1 << std::min(d, 3)) : 1.0;
    ws += w[k];
  }
  std::vector<int> zb(K + 1, 0);
  double c = 0;
  for (int k = 0; k < K; ++k) {
    c += w[k];
    int b = k + 1 == K ? NZ : int(std::lround(NZ * c / ws));
    b = std::max(b, zb[k] + 1);
    b = std::min(b, NZ - (K - 1 - k));
    zb[k + 1] = b;
  }
  return zb;
}

void chain(int K, bool ramp, int nin, int nout, bool un_sep) {
  auto zb = bounds(K, ramp);
  const size_t pitch = NS * sizeof(double);
  // streams: [0, nin) H2D, [nin, nin + nout) D2H, nin + nout: u_n (un_sep)
  const int total = nin + nout + (un_sep ? 1 : 0);
  fork(total);
  for (int k = 0; k < K; ++k) {
    cudaStream_t s = st[k % nin];
    const size_t off = zb[k] * LAYER, cnt = (zb[k + 1] - zb[k]) * LAYER;
    CK(cudaMemcpy2DAsync(dU + off, pitch, hU + off, pitch, cnt * 8, NT, cudaMemcpyHostToDevice, s));
    cudaStream_t su = un_sep ? st[nin + nout] : s;
    CK(cudaMemcpyAsync(du + off, hu + off, cnt * 8, cudaMemcpyHostToDevice, su));
    cudaEventRecord(ev[k], s);
    if (un_sep) {
      cudaEventRecord(ev[32 + k], su);
    }
  }
  for (int k = 0; k < K; ++k) {
    cudaStream_t s = st[nin + k % nout];
    cudaStreamWaitEvent(s, ev[k], 0);
    if (un_sep) cudaStreamWaitEvent(s, ev[32 + k], 0);
    const size_t off = zb[k] * LAYER, cnt = (zb[k + 1] - zb[k]) * LAYER;
    CK(cudaMemcpy2DAsync(hR + off, pitch, dR + off, pitch, cnt * 8, NT, cudaMemcpyDeviceToHost, s));
  }
  join(total);
}

__global__ void zc_copy(const double2* __restrict__ src, double2* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

// rows x cnt2 double2 elements, row pitch pitch2 (double2): one chunk of all temporal blocks
__global__ void zc_copy2d(const double2* __restrict__ src, double2* __restrict__ dst, size_t cnt2,
                          size_t pitch2, int rows) {
  const size_t n = cnt2 * rows;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const size_t r = i / cnt2, c = i - r * cnt2;
    dst[r * pitch2 + c] = src[r * pitch2 + c];
  }
}

// copy engine in (chunked), SM-written zero-copy out per chunk (blocks CTAs of 512 threads)
void chain_zc(int K, bool ramp, int blocks) {
  auto zb = bounds(K, ramp);
  const size_t pitch = NS * sizeof(double);
  fork(2);
  for (int k = 0; k < K; ++k) {
    const size_t off = zb[k] * LAYER, cnt = (zb[k + 1] - zb[k]) * LAYER;
    CK(cudaMemcpy2DAsync(dU + off, pitch, hU + off, pitch, cnt * 8, NT, cudaMemcpyHostToDevice, st[0]));
    CK(cudaMemcpyAsync(du + off, hu + off, cnt * 8, cudaMemcpyHostToDevice, st[0]));
    cudaEventRecord(ev[k], st[0]);
  }
  for (int k = 0; k < K; ++k) {
    cudaStreamWaitEvent(st[1], ev[k], 0);
    const size_t off = zb[k] * LAYER, cnt = (zb[k + 1] - zb[k]) * LAYER;
    zc_copy2d<<<blocks, 512, 0, st[1]>>>((const double2*)(dR + off), (double2*)(hR + off), cnt / 2, NS / 2, NT);
  }
  join(2);
}

// SM-issued zero-copy reads in (one kernel per chunk, in stream order), copy engine out
void chain_zcin(int K, bool ramp, int blocks) {
  auto zb = bounds(K, ramp);
  const size_t pitch = NS * sizeof(double);
  fork(2);
  for (int k = 0; k < K; ++k) {
    const size_t off = zb[k] * LAYER, cnt = (zb[k + 1] - zb[k]) * LAYER;
    zc_copy2d<<<blocks, 512, 0, st[0]>>>((const double2*)(hU + off), (double2*)(dU + off), cnt / 2, NS / 2, NT);
    zc_copy2d<<<blocks, 512, 0, st[0]>>>((const double2*)(hu + off), (double2*)(du + off), cnt / 2, NS / 2, 1);
    cudaEventRecord(ev[k], st[0]);
  }
  for (int k = 0; k < K; ++k) {
    cudaStreamWaitEvent(st[1], ev[k], 0);
    const size_t off = zb[k] * LAYER, cnt = (zb[k + 1] - zb[k]) * LAYER;
    CK(cudaMemcpy2DAsync(hR + off, pitch, dR + off, pitch, cnt * 8, NT, cudaMemcpyDeviceToHost, st[1]));
  }
  join(2);
}

int main() {
  CK(cudaHostAlloc(&hU, ND * 8, cudaHostAllocMapped));
  CK(cudaHostAlloc(&hu, NS * 8, cudaHostAllocMapped));
  CK(cudaHostAlloc(&hR, ND * 8, cudaHostAllocMapped));
  CK(cudaMalloc(&dU, ND * 8));
  CK(cudaMalloc(&du, NS * 8));
  CK(cudaMalloc(&dR, ND * 8));
  for (size_t i = 0; i < ND; ++i) hU[i] = double(i % 977);
  for (auto& s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&mainS, cudaStreamNonBlocking));
  for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&evm, cudaEventDisableTiming));
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  std::printf("{");
  std::printf("\"h2d\": %.4f", timed([] {
    cudaMemcpyAsync(dU, hU, ND * 8, cudaMemcpyHostToDevice, mainS);
    cudaMemcpyAsync(du, hu, NS * 8, cudaMemcpyHostToDevice, mainS);
  }));
  std::printf(", \"d2h\": %.4f", timed([] { cudaMemcpyAsync(hR, dR, ND * 8, cudaMemcpyDeviceToHost, mainS); }));
  std::printf(", \"duplex\": %.4f", timed([] {
    fork(2);
    cudaMemcpyAsync(dU, hU, ND * 8, cudaMemcpyHostToDevice, st[0]);
    cudaMemcpyAsync(du, hu, NS * 8, cudaMemcpyHostToDevice, st[0]);
    cudaMemcpyAsync(hR, dR, ND * 8, cudaMemcpyDeviceToHost, st[1]);
    join(2);
  }));
  for (int K : {8})
    for (int ramp : {0, 1})
      for (int nin : {1, 2})
        for (int nout : {1, 2})
          for (int sep : {0, 1}) {
            float t = timed([&] { chain(K, ramp, nin, nout, sep); });
            std::printf(", \"chain_K%d_r%d_i%d_o%d_u%d\": %.4f", K, ramp, nin, nout, sep, t);
          }
  // zero-copy: SM-issued PCIe reads / writes (mapped pinned memory, UVA pointers)
  for (int blocks : {nsm, 2 * nsm, 4 * nsm}) {
    std::printf(", \"zc_read_b%d\": %.4f", blocks, timed([&] {
      zc_copy<<<blocks, 512, 0, mainS>>>((const double2*)hU, (double2*)dU, ND / 2);
      zc_copy<<<blocks, 512, 0, mainS>>>((const double2*)hu, (double2*)du, NS / 2);
    }));
    std::printf(", \"zc_write_b%d\": %.4f", blocks, timed([&] {
      zc_copy<<<blocks, 512, 0, mainS>>>((const double2*)dR, (double2*)hR, ND / 2);
    }));
    std::printf(", \"zc_both_b%d\": %.4f", blocks, timed([&] {
      fork(2);
      zc_copy<<<blocks / 2, 512, 0, st[0]>>>((const double2*)hU, (double2*)dU, ND / 2);
      zc_copy<<<blocks / 2, 512, 0, st[0]>>>((const double2*)hu, (double2*)du, NS / 2);
      zc_copy<<<blocks / 2, 512, 0, st[1]>>>((const double2*)dR, (double2*)hR, ND / 2);
      join(2);
    }));
    // copy engine in, SMs write out
    std::printf(", \"ce_in_zc_out_b%d\": %.4f", blocks, timed([&] {
      fork(2);
      cudaMemcpyAsync(dU, hU, ND * 8, cudaMemcpyHostToDevice, st[0]);
      cudaMemcpyAsync(du, hu, NS * 8, cudaMemcpyHostToDevice, st[0]);
      zc_copy<<<blocks, 512, 0, st[1]>>>((const double2*)dR, (double2*)hR, ND / 2);
      join(2);
    }));
  }
  for (int K : {8})
    for (int ramp : {0, 1})
      for (int blocks : {148}) {
        float t = timed([&] { chain_zc(K, ramp, blocks); });
        std::printf(", \"chainzc_K%d_r%d_b%d\": %.4f", K, ramp, blocks, t);
      }
  for (int blocks : {148, 592})
    std::printf(", \"zc_in_ce_out_b%d\": %.4f", blocks, timed([&] {
      fork(2);
      zc_copy<<<blocks, 512, 0, st[0]>>>((const double2*)hU, (double2*)dU, ND / 2);
      zc_copy<<<blocks, 512, 0, st[0]>>>((const double2*)hu, (double2*)du, NS / 2);
      cudaMemcpyAsync(hR, dR, ND * 8, cudaMemcpyDeviceToHost, st[1]);
      join(2);
    }));
  for (int K : {8, 16, 32})
    for (int ramp : {0, 1})
      for (int blocks : {148, 592}) {
        float t = timed([&] { chain_zcin(K, ramp, blocks); });
        std::printf(", \"chainzcin_K%d_r%d_b%d\": %.4f", K, ramp, blocks, t);
      }
  std::printf("}\n");
  CK(cudaDeviceSynchronize());
  return 0;
}
