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
// block r stores its own contiguous slice of idx in order (idx sorted by
// range r = v / span and by v inside the range)
__global__ void scatter_ranges(int* a, const uint32_t* idx, const int64_t* start) {
  const int64_t b = start[blockIdx.x], e = start[blockIdx.x + 1];
  for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) a[idx[i]] = (int)i;
}
// as scatter_ranges, but each thread walks its own contiguous sub-slice
// (lanes of a warp far apart: one line per lane per store instruction)
__global__ void scatter_ranges_strided(int* a, const uint32_t* idx, const int64_t* start) {
  const int64_t b = start[blockIdx.x], e = start[blockIdx.x + 1];
  const int64_t per = (e - b + blockDim.x - 1) / blockDim.x;
  const int64_t lo = b + threadIdx.x * per, hi = lo + per < e ? lo + per : e;
  for (int64_t i = lo; i < hi; i++) a[idx[i]] = (int)i;
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
  // range-sorted: 296 ranges (one per CTA of a 2-CTA/SM persistent grid)
  const int R = 296;
  const int64_t span = (n + R - 1) / R;
  std::vector<int64_t> start(R + 1, 0);
  for (auto x : sorted) start[x / span + 1]++;
  for (int r = 0; r < R; r++) start[r + 1] += start[r];
  int64_t* dstart;
  cudaMalloc(&dstart, (R + 1) * 8);
  cudaMemcpy(dstart, start.data(), (R + 1) * 8, cudaMemcpyHostToDevice);
  // range-random: same partition, random order inside each range
  std::vector<uint32_t> rrand = idx;
  std::stable_sort(rrand.begin(), rrand.end(), [&](uint32_t a, uint32_t b) { return a / span < b / span; });
  // 296 ranges, sub-windows of W ids in order, random order inside a window
  std::vector<uint32_t> rw[3];
  const int64_t wsz[3] = {2048, 8192, 32768};
  for (int j = 0; j < 3; j++) {
    rw[j] = idx;
    const int64_t W = wsz[j];
    std::stable_sort(rw[j].begin(), rw[j].end(), [&](uint32_t a, uint32_t b) {
      return a / span != b / span ? a / span < b / span : (a % span) / W < (b % span) / W; });
  }
  int* a;
  uint32_t* d;
  cudaMalloc(&a, n * 4);
  cudaMalloc(&d, k * 4);
  int* flush;
  cudaMalloc(&flush, size_t(512) << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"random", "sorted", "bucketed(4096)", "296 ranges, sorted", "296 ranges, random",
                         "296 ranges, 2K-id windows", "296 ranges, 8K-id windows", "296 ranges, 32K-id windows",
                         "296 ranges, sorted, lanes strided"};
  std::vector<uint32_t>* sets[] = {&idx, &sorted, &bucketed, &sorted, &rrand, &rw[0], &rw[1], &rw[2], &sorted};
  for (int rep = 0; rep < 2; rep++)
    for (int s = 0; s < 9; s++) {
      cudaMemcpy(d, sets[s]->data(), k * 4, cudaMemcpyHostToDevice);
      fill<<<148 * 8, 512>>>(a, n);
      fill<<<148 * 8, 512>>>(flush, int64_t(128) << 20);  // evict L2
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      if (s < 3) scatter<<<148 * 8, 512>>>(a, d, k);
      else if (s < 8) scatter_ranges<<<R, 512>>>(a, d, dstart);
      else scatter_ranges_strided<<<R, 512>>>(a, d, dstart);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%-16s %7.3f ms  (%.1f G stores/s)\n", names[s], ms, k / ms / 1e6);
    }
  return 0;
}
