// Host expansion of the compact ParentArray transfer (gk_expand.cpp) against
// a direct restatement: random parent arrays with ragged last blocks, an
// unaligned destination, 1 and 4 threads, expansion from block 0 and from a
// later block.  Run by tests/test_expand_host.py (CPU).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
namespace gk { void expand_parents(const uint32_t* buf, int64_t n, int32_t* dst, int threads, int64_t first_block); bool expand_uses_avx512(); }
int main() {
  for (int64_t n : {1, 1023, 1024, 1025, 100000, 4194381}) for (int thr : {1, 4}) {
    std::mt19937_64 r(n);
    std::vector<int32_t> p(n);
    for (auto& x : p) x = (r() % 3 == 0) ? -1 : (int32_t)(r() % n);
    int64_t nblk = (n + 1023) / 1024;
    std::vector<uint32_t> buf(nblk + 1 + 32 * nblk + n, 0);
    uint32_t c = 0;
    std::vector<int32_t> packed;
    for (int64_t b = 0; b < nblk; b++) {
      buf[b] = c;
      for (int k = 0; k < 1024; k++) { int64_t v = b * 1024 + k; if (v < n && p[v] >= 0) { buf[nblk + 1 + b * 32 + k / 32] |= 1u << (k % 32); packed.push_back(p[v]); c++; } }
    }
    buf[nblk] = c;
    for (size_t i = 0; i < packed.size(); i++) buf[nblk + 1 + 32 * nblk + i] = (uint32_t)packed[i];
    for (int64_t first : {int64_t(0), nblk / 2}) {
      std::vector<int32_t> out(n + 1, 5);
      gk::expand_parents(buf.data(), n, out.data() + (n & 1), thr, first);  // odd n: unaligned destination
      int64_t bad = 0;
      for (int64_t v = 0; v < n; v++) bad += out[v + (n & 1)] != (v < first * 1024 ? 5 : p[v]);
      printf("n %ld thr %d first %ld avx512 %d bad %ld\n", (long)n, thr, (long)first, (int)gk::expand_uses_avx512(),
             (long)bad);
      if (bad) return 1;
    }
  }
}
