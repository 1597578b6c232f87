// Is random-access throughput over a large array limited by DRAM or by
// address translation?  Compare fully random 32 B accesses over 16 GB with
// accesses where each warp instruction stays inside one random 2 MB page
// (translation-friendly, DRAM-random), and with a 64 KB page-local window.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t xs(uint64_t& x) {
  x ^= x << 13; x ^= x >> 7; x ^= x << 17;
  return x;
}

// mode 0: fully random sectors; mode 1: one random page per warp-instruction,
// random sectors within it (page = 1 << page_bits bytes).
__global__ void probe(const uint32_t* __restrict__ a, uint64_t nsec_mask, int page_bits, int mode,
                      uint64_t iters, unsigned long long* sink) {
  const int lane = threadIdx.x & 31;
  uint64_t x = 0x9e3779b97f4a7c15ULL * (blockIdx.x * 1024 + threadIdx.x + 1);
  uint64_t wx = 0xbf58476d1ce4e5b9ULL * (blockIdx.x * 64 + (threadIdx.x >> 5) + 7);
  const uint64_t sec_per_page_mask = (1ull << (page_bits - 5)) - 1;
  uint32_t acc = 0;
  for (uint64_t it = 0; it < iters; it++) {
    uint32_t v[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      uint64_t sec;
      if (mode == 0) {
        sec = xs(x) & nsec_mask;
      } else {
        const uint64_t page = __shfl_sync(0xffffffffu, xs(wx), 0) & (nsec_mask >> (page_bits - 5));
        sec = (page << (page_bits - 5)) | (xs(x) & sec_per_page_mask);
      }
      v[k] = __ldg(a + sec * 8 + (lane & 7));
    }
#pragma unroll
    for (int k = 0; k < 8; k++) acc += v[k];
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
  const size_t bytes = 16ull << 30;
  uint32_t* a;
  unsigned long long* sink;
  cudaMalloc(&a, bytes);
  cudaMalloc(&sink, 8);
  cudaMemset(a, 1, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int tpb = 512, blocks = sms * 4;
  const uint64_t iters = 64;
  struct { int mode, page_bits; const char* name; } cfgs[] = {
      {0, 21, "fully random 32B"}, {1, 21, "warp-local 2MB page"}, {1, 16, "warp-local 64KB"},
      {1, 12, "warp-local 4KB"}};
  for (auto c : cfgs) {
    float ms;
    cudaEventRecord(e0);
    probe<<<blocks, tpb>>>(a, bytes / 32 - 1, c.page_bits, c.mode, iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double acc = (double)blocks * tpb * iters * 8;
    printf("%-22s: %6.1f G accesses/s (%6.0f GB/s at 32 B)\n", c.name, acc / ms / 1e6, acc * 32 / ms / 1e6);
  }
  return 0;
}
