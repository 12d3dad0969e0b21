// Host-side staging for the *_host entry points when the caller's buffers are
// pageable (malloc / std::vector / Eigen memory, what a caller of the
// reference passes): the CUDA driver would stage such copies itself, on one
// thread (about 13 GB/s on the bench boxes, 11 ms for the 151 MB of a c4 R(U)
// call).  Here a small pool of worker threads copies between the caller's
// memory and page-locked mirrors owned by the handle, chunk by chunk, while
// the copy engines move the previous chunk (stg.cpp: st_residual_host_staged,
// staged_h2d, staged_d2h).
#pragma once

#if defined(__x86_64__) || defined(_M_X64)
#include <emmintrin.h>
#define STG_HOSTCOPY_SSE2 1
#endif

#include <algorithm>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace stg {

struct CopyItem {
  void* dst;
  const void* src;
  std::size_t bytes;
};

// memcpy with non-temporal stores: the destinations here (a page-locked
// mirror about to be read by the copy engine, or the caller's result buffer)
// are written once and not read back by this core, and a thread's share of a
// chunk (1-2 MB) is below the size at which glibc's memcpy switches to
// streaming stores itself, so a plain memcpy would first read every
// destination line into the cache (a third of the memory traffic).
// STG_HOST_PLAIN_MEMCPY=1 uses memcpy.
inline void stream_copy(void* dst, const void* src, std::size_t bytes) {
#ifdef STG_HOSTCOPY_SSE2
  static const bool plain = std::getenv("STG_HOST_PLAIN_MEMCPY") != nullptr;
  if (!plain && bytes >= 4096) {
    char* d = static_cast<char*>(dst);
    const char* s = static_cast<const char*>(src);
    const std::size_t head = (16 - (reinterpret_cast<std::uintptr_t>(d) & 15)) & 15;
    if (head) {
      std::memcpy(d, s, head);
      d += head;
      s += head;
      bytes -= head;
    }
    std::size_t n64 = bytes / 64;
    for (; n64; --n64, d += 64, s += 64) {
      const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s));
      const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 16));
      const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 32));
      const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + 48));
      _mm_stream_si128(reinterpret_cast<__m128i*>(d), a);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + 16), b);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + 32), c);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + 48), e);
    }
    _mm_sfence();
    bytes &= 63;
    if (bytes) std::memcpy(d, s, bytes);
    return;
  }
#endif
  std::memcpy(dst, src, bytes);
}

// Process-wide fork-join pool: par_copy() splits the concatenated byte range
// of its items into one contiguous share per thread (the caller's thread takes
// share 0).  STG_HOST_THREADS overrides the thread count (default: three
// quarters of the hardware threads, at most 16).  Calls are serialised.
class HostCopyPool {
 public:
  static HostCopyPool& get() {
    static HostCopyPool* pool = new HostCopyPool;  // never destroyed (workers park forever)
    return *pool;
  }
  int threads() const { return nthreads_; }

  void par_copy(const CopyItem* items, int n) {
    std::size_t total = 0;
    for (int i = 0; i < n; ++i) total += items[i].bytes;
    if (total == 0) return;
    if (nthreads_ == 1 || total < (std::size_t(1) << 20)) {
      for (int i = 0; i < n; ++i) stream_copy(items[i].dst, items[i].src, items[i].bytes);
      return;
    }
    std::lock_guard<std::mutex> call(call_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      items_ = items;
      n_items_ = n;
      total_ = total;
      pending_ = nthreads_ - 1;
      ++generation_;
    }
    cv_.notify_all();
    share(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  HostCopyPool() {
    int t = 0;
    if (const char* e = std::getenv("STG_HOST_THREADS")) t = std::atoi(e);
    if (t <= 0) {
      const unsigned hw = std::thread::hardware_concurrency();
      t = int(std::min(16u, std::max(1u, hw * 3 / 4)));
    }
    nthreads_ = std::min(t, 64);
    for (int i = 1; i < nthreads_; ++i) std::thread([this, i] { worker(i); }).detach();
  }

  // bytes [total * id / T, total * (id + 1) / T) of the concatenated items,
  // cut at 4 KiB so shares start page-aligned within an item
  void share(int id) {
    const std::size_t T = std::size_t(nthreads_);
    auto cut = [&](std::size_t j) {
      if (j >= T) return total_;
      return (total_ / T * j) & ~std::size_t(4095);
    };
    std::size_t lo = cut(std::size_t(id)), hi = cut(std::size_t(id) + 1), base = 0;
    for (int i = 0; i < n_items_ && lo < hi; ++i) {
      const std::size_t end = base + items_[i].bytes;
      if (lo < end) {
        const std::size_t a = lo - base, b = std::min(hi, end) - base;
        stream_copy(static_cast<char*>(items_[i].dst) + a,
                    static_cast<const char*>(items_[i].src) + a, b - a);
        lo = base + b;
      }
      base = end;
    }
  }

  void worker(int id) {
    unsigned long long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return generation_ != seen; });
        seen = generation_;
      }
      share(id);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }

  int nthreads_ = 1;
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  const CopyItem* items_ = nullptr;
  int n_items_ = 0;
  std::size_t total_ = 0;
  int pending_ = 0;
  unsigned long long generation_ = 0;
};

}  // namespace stg
