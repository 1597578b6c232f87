// Random 4-byte access rate when the working set is L2-resident (16-64 MB):
// plain loads, .cg loads, atomicOr with return, and fire-and-forget RED.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t xs(uint64_t& x) {
  x ^= x << 13; x ^= x >> 7; x ^= x << 17;
  return x;
}
template <int kMode>
__global__ void k(uint32_t* a, uint64_t mask, uint64_t iters, unsigned long long* sink) {
  uint64_t x = 0x9e3779b97f4a7c15ULL * (blockIdx.x * 1024 + threadIdx.x + 1);
  uint32_t acc = 0;
  for (uint64_t it = 0; it < iters; it++) {
    uint32_t v[8];
#pragma unroll
    for (int j = 0; j < 8; j++) {
      uint32_t* p = a + (xs(x) & mask);
      if (kMode == 0) v[j] = __ldg(p);
      else if (kMode == 1) v[j] = __ldcg(p);
      else if (kMode == 2) v[j] = atomicOr(p, 1u << (x & 31));
      else { atomicOr(p, 1u << (x & 31)); v[j] = 0; }
    }
#pragma unroll
    for (int j = 0; j < 8; j++) acc += v[j];
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}
int main() {
  uint32_t* a;
  unsigned long long* sink;
  cudaMalloc(&a, 1ull << 30);
  cudaMalloc(&sink, 8);
  cudaMemset(a, 0, 1ull << 30);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int tpb = 512, blocks = sms * 4;
  const uint64_t iters = 64;
  const char* names[] = {"ldg", "ld.cg", "atomicOr+ret", "red.or"};
  for (size_t ws : {16ull << 20, 64ull << 20, 1024ull << 20}) {
    for (int m = 0; m < 4; m++) {
      float ms;
      for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0);
        if (m == 0) k<0><<<blocks, tpb>>>(a, ws / 4 - 1, iters, sink);
        if (m == 1) k<1><<<blocks, tpb>>>(a, ws / 4 - 1, iters, sink);
        if (m == 2) k<2><<<blocks, tpb>>>(a, ws / 4 - 1, iters, sink);
        if (m == 3) k<3><<<blocks, tpb>>>(a, ws / 4 - 1, iters, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      const double n = (double)blocks * tpb * iters * 8;
      printf("ws %5zu MB %-13s %7.1f G ops/s\n", ws >> 20, names[m], n / ms / 1e6);
    }
  }
  return 0;
}
