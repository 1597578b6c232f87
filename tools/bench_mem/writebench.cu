// Cost of scattered 4-byte stores into a 512 MB array (the parent array of
// a 2^27-vertex BFS): random order vs sorted order vs 4096-bucketed order,
// 17M stores (a hub-expansion top-down step's claims).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void scatter(int* a, const uint32_t* idx, int64_t k) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
    a[idx[i]] = (int)i;
}
__global__ void fill(int* a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = -1;
}

int main() {
  const int64_t n = int64_t(1) << 27, k = 17000000;
  std::mt19937_64 rng(1);
  std::vector<uint32_t> idx(k);
  for (auto& x : idx) x = rng() % n;
  std::vector<uint32_t> sorted = idx;
  std::sort(sorted.begin(), sorted.end());
  std::vector<uint32_t> bucketed = idx;
  std::stable_sort(bucketed.begin(), bucketed.end(), [](uint32_t a, uint32_t b) { return (a >> 15) < (b >> 15); });
  int* a;
  uint32_t* d;
  cudaMalloc(&a, n * 4);
  cudaMalloc(&d, k * 4);
  int* flush;
  cudaMalloc(&flush, size_t(512) << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"random", "sorted", "bucketed(4096)"};
  std::vector<uint32_t>* sets[] = {&idx, &sorted, &bucketed};
  for (int rep = 0; rep < 2; rep++)
    for (int s = 0; s < 3; s++) {
      cudaMemcpy(d, sets[s]->data(), k * 4, cudaMemcpyHostToDevice);
      fill<<<148 * 8, 512>>>(a, n);
      fill<<<148 * 8, 512>>>(flush, int64_t(128) << 20);  // evict L2
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      scatter<<<148 * 8, 512>>>(a, d, k);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%-16s %7.3f ms  (%.1f G stores/s)\n", names[s], ms, k / ms / 1e6);
    }
  return 0;
}
