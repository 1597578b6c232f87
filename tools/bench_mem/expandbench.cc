// Host expansion rate of the compact ParentArray transfer (gk_expand.cpp):
// kron27-sized array (2^27 vertices, 47 % reached), T threads, 5 passes.
// Build: g++ -O3 -std=c++17 -pthread expandbench.cc ../../build/gk_expand.o
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>
namespace gk { void expand_parents(const uint32_t*, int64_t, int32_t*, int, int64_t); }
int main(int argc, char** argv) {
  const int64_t n = int64_t(1) << 27, nblk = n / 1024;
  std::vector<uint32_t> buf(nblk + 1 + 32 * nblk + n);
  std::mt19937 r(1);
  uint32_t c = 0;
  for (int64_t b = 0; b < nblk; b++) {
    buf[b] = c;
    for (int k = 0; k < 32; k++) {
      uint32_t w = 0;
      for (int j = 0; j < 32; j++) if (r() % 100 < 47) { w |= 1u << j; buf[nblk + 1 + 32 * nblk + c++] = r() % n; }
      buf[nblk + 1 + b * 32 + k] = w;
    }
  }
  buf[nblk] = c;
  int32_t* dst = static_cast<int32_t*>(aligned_alloc(64, n * 4));
  memset(dst, 0, n * 4);
  for (int t : {4, 8, 15, 16}) {
    for (int rep = 0; rep < 3; rep++) {
      auto t0 = std::chrono::steady_clock::now();
      gk::expand_parents(buf.data(), n, dst, t, 0);
      double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      printf("threads %2d: %.2f ms (%.1f GB/s written)\n", t, ms, n * 4 / ms / 1e6);
    }
  }
  return 0;
}
