// HostCopyPool (paper_2201_05800_b200/csrc/hostcopy.hpp): par_copy over
// several items of ragged sizes equals memcpy of each item, whatever the
// thread count; small totals take the single-thread path.
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "../../paper_2201_05800_b200/csrc/hostcopy.hpp"

int main() {
  stg::HostCopyPool& pool = stg::HostCopyPool::get();
  std::mt19937_64 gen(5);
  int fail = 0;
  for (int round = 0; round < 40; ++round) {
    const int n = 1 + int(gen() % 6);
    std::vector<std::vector<unsigned char>> src(n), dst(n), ref(n);
    std::vector<stg::CopyItem> items;
    for (int i = 0; i < n; ++i) {
      // ragged sizes, some empty, totals on both sides of the 1 MiB threshold
      const size_t bytes = round % 4 == 0 ? gen() % 5000 : gen() % (3u << 20);
      src[i].resize(bytes + 16);
      dst[i].assign(bytes + 16, 0xAB);
      for (auto& b : src[i]) b = (unsigned char)gen();
      ref[i] = dst[i];
      const size_t shift = gen() % 8;  // unaligned starts
      const size_t len = bytes > shift ? bytes - shift : 0;
      std::memcpy(ref[i].data() + shift, src[i].data() + shift, len);
      items.push_back({dst[i].data() + shift, src[i].data() + shift, len});
    }
    pool.par_copy(items.data(), n);
    for (int i = 0; i < n; ++i)
      if (dst[i] != ref[i]) ++fail;
  }
  pool.par_copy(nullptr, 0);
  std::printf("threads %d failed %d\n", pool.threads(), fail);
  return fail == 0 ? 0 : 1;
}
