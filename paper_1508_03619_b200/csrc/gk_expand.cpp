// gk_expand.cpp -- host side of the compact ParentArray transfer (gk_pack.cu).
//
// Expands [off (nblk + 1)] [bits (32 nblk)] [packed] into the caller's full
// ParentArray: vertex v gets the next packed parent when its reached bit is
// set, else -1 (bfs.hpp:126-132 / :171-175: unreached vertices keep a
// negative parent; the reference's final sweep makes them -1).  Blocks are
// independent (off[b] is their start in packed), so threads split the block
// range.  With AVX-512 a 16-vertex half-word is one masked expand-load
// (vpexpandd) and one 64-byte store -- non-temporal when the destination is
// 64-byte aligned, so the 537 MB output does not pay read-for-ownership
// traffic; otherwise a branchless scalar loop.
#include <immintrin.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace gk {
namespace {

void expand_scalar(const uint32_t* off, const uint32_t* bits, const int32_t* packed, int32_t* dst, int64_t n,
                   int64_t b0, int64_t b1) {
  for (int64_t b = b0; b < b1; b++) {
    const int32_t* src = packed + off[b];
    const int64_t v0 = b * 1024, vend = std::min<int64_t>(1024, n - v0);
    for (int64_t i = 0; i < vend; i++) {
      const uint32_t bit = (bits[b * 32 + (i >> 5)] >> (i & 31)) & 1u;
      dst[v0 + i] = bit ? *src : -1;
      src += bit;
    }
  }
}

__attribute__((target("avx512f"))) void expand_avx512(const uint32_t* off, const uint32_t* bits,
                                                      const int32_t* packed, int32_t* dst, int64_t n, int64_t b0,
                                                      int64_t b1) {
  const __m512i neg = _mm512_set1_epi32(-1);
  const bool aligned = (reinterpret_cast<uintptr_t>(dst) & 63) == 0;
  for (int64_t b = b0; b < b1; b++) {
    if ((b + 1) * 1024 > n) {  // the ragged last block
      expand_scalar(off, bits, packed, dst, n, b, b + 1);
      continue;
    }
    const int32_t* src = packed + off[b];
    int32_t* out = dst + b * 1024;
    for (int k = 0; k < 64; k++) {
      const uint32_t w = bits[b * 32 + (k >> 1)];
      const __mmask16 m = (__mmask16)((k & 1) ? (w >> 16) : (w & 0xffffu));
      const __m512i v = _mm512_mask_expandloadu_epi32(neg, m, src);
      src += __builtin_popcount((unsigned)m);
      if (aligned) _mm512_stream_si512(reinterpret_cast<__m512i*>(out + 16 * k), v);
      else _mm512_storeu_si512(out + 16 * k, v);
    }
  }
  _mm_sfence();
}

}  // namespace

// buf: the transfer as gk_pack.cu lays it out; dst: n int32; blocks from
// first_block on (the ones before travelled raw).  threads <= 0: hardware
// concurrency.
void expand_parents(const uint32_t* buf, int64_t n, int32_t* dst, int threads, int64_t first_block) {
  if (n <= 0) return;
  const int64_t nblk = (n + 1023) / 1024;
  if (first_block >= nblk) return;
  const uint32_t* off = buf;
  const uint32_t* bits = buf + nblk + 1;
  const int32_t* packed = reinterpret_cast<const int32_t*>(bits + 32 * nblk);
  static const bool avx512 = __builtin_cpu_supports("avx512f");
  auto run = [&](int64_t b0, int64_t b1) {
    if (avx512) expand_avx512(off, bits, packed, dst, n, b0, b1);
    else expand_scalar(off, bits, packed, dst, n, b0, b1);
  };
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  const int64_t nb = nblk - first_block;
  threads = (int)std::min<int64_t>(threads, std::max<int64_t>(1, nb / 16));
  if (threads <= 1) {
    run(first_block, nblk);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(threads - 1);
  const int64_t per = (nb + threads - 1) / threads;
  for (int t = 1; t < threads; t++) {
    const int64_t b0 = first_block + std::min(nb, t * per), b1 = std::min(nblk, b0 + per);
    pool.emplace_back(run, b0, b1);
  }
  run(first_block, first_block + std::min(nb, per));
  for (auto& th : pool) th.join();
}

bool expand_uses_avx512() { return __builtin_cpu_supports("avx512f"); }

}  // namespace gk
