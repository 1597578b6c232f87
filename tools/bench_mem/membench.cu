// Random-gather bandwidth calibration for the BFS byte model.
// gather<W>: each thread issues 8 independent loads of W bytes (W = 4, 16)
// at random W-aligned... positions within a 32-byte sector grid, or whole
// 64/128-byte chunks read by 4/8 consecutive lanes; over working sets from
// 256 MB to 16 GB.  Reports useful bytes/s and sectors/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t xs(uint64_t& x) {
  x ^= x << 13; x ^= x >> 7; x ^= x << 17;
  return x;
}

// kLanes consecutive lanes read one kLanes*16-byte chunk together.
template <int kLanes>
__global__ void gather(const uint4* __restrict__ a, uint64_t mask_chunks, uint64_t iters, uint64_t seed,
                       unsigned long long* sink) {
  const int lane = threadIdx.x & 31, grp = lane / kLanes, sub = lane % kLanes;
  uint64_t x = seed ^ ((blockIdx.x * 131 + (threadIdx.x >> 5)) * 0x9e3779b97f4a7c15ULL + grp * 0xbf58476d1ce4e5b9ULL);
  uint32_t acc = 0;
  for (uint64_t it = 0; it < iters; it++) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = __ldg(a + (xs(x) & mask_chunks) * kLanes + sub);
#pragma unroll
    for (int k = 0; k < 8; k++) acc += v[k].x;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

__global__ void gather4(const uint32_t* __restrict__ a, uint64_t mask_sec, uint64_t iters, uint64_t seed,
                        unsigned long long* sink) {
  uint64_t x = seed ^ (blockIdx.x * 0x9e3779b97f4a7c15ULL + threadIdx.x * 0xbf58476d1ce4e5b9ULL);
  uint32_t acc = 0;
  for (uint64_t it = 0; it < iters; it++) {
    uint32_t v[8];
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = __ldg(a + (xs(x) & mask_sec) * 8);
#pragma unroll
    for (int k = 0; k < 8; k++) acc += v[k];
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
  const size_t maxb = 16ull << 30;
  uint4* a;
  unsigned long long* sink;
  cudaMalloc(&a, maxb);
  cudaMalloc(&sink, 8);
  cudaMemset(a, 1, maxb);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int tpb = 512, blocks = sms * 4;
  const uint64_t iters = 64;
  const double nthreads = (double)blocks * tpb;
  for (size_t ws : {256ull << 20, 2ull << 30, 16ull << 30}) {
    float ms;
    cudaEventRecord(e0);
    gather4<<<blocks, tpb>>>((const uint32_t*)a, ws / 32 - 1, iters, 77, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double acc = nthreads * iters * 8;
    printf("ws %5zu MB  4B/sector   : %6.1f Gsect/s  useful %6.0f GB/s  (sector-equiv %6.0f GB/s)\n", ws >> 20,
           acc / ms / 1e6, acc * 4 / ms / 1e6, acc * 32 / ms / 1e6);
#define RUN(L)                                                                                     \
    cudaEventRecord(e0);                                                                           \
    gather<L><<<blocks, tpb>>>(a, ws / (16 * L) - 1, iters, 99, sink);                             \
    cudaEventRecord(e1);                                                                           \
    cudaEventSynchronize(e1);                                                                      \
    cudaEventElapsedTime(&ms, e0, e1);                                                             \
    acc = nthreads * iters * 8 / L;                                                                \
    printf("ws %5zu MB  %3d B chunks: %6.1f Gchunk/s useful %6.0f GB/s\n", ws >> 20, 16 * L,      \
           acc / ms / 1e6, acc * 16 * L / ms / 1e6);
    RUN(2) RUN(4) RUN(8)
  }
  return 0;
}
