// hostcopy.cu -- where a ParentArray's e2e time goes on the box's host:
// std::vector value-init of n int32, pageable vs pinned D2H, threaded
// memcpy from a pinned staging buffer.  nvcc -O2 -o hostcopy hostcopy.cu
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  const size_t n = argc > 1 ? strtoull(argv[1], nullptr, 10) : (size_t(1) << 27);
  const int nt = argc > 2 ? atoi(argv[2]) : 16;
  const size_t bytes = n * 4;
  int32_t* d;
  cudaMalloc(&d, bytes);
  cudaMemset(d, 0x11, bytes);
  int32_t* pin;
  cudaHostAlloc(&pin, bytes, cudaHostAllocDefault);
  memset(pin, 0, bytes);
  cudaDeviceSynchronize();
  for (int rep = 0; rep < 3; rep++) {
    double t0 = now();
    std::vector<int32_t> v(n);
    double t1 = now();
    cudaMemcpy(v.data(), d, bytes, cudaMemcpyDeviceToHost);
    double t2 = now();
    cudaMemcpy(v.data(), d, bytes, cudaMemcpyDeviceToHost);
    double t3 = now();
    cudaMemcpy(pin, d, bytes, cudaMemcpyDeviceToHost);
    double t4 = now();
    std::vector<std::thread> th;
    for (int i = 0; i < nt; i++)
      th.emplace_back([&, i] {
        size_t a = bytes * i / nt, b = bytes * (i + 1) / nt;
        memcpy((char*)v.data() + a, (char*)pin + a, b - a);
      });
    for (auto& x : th) x.join();
    double t5 = now();
    std::vector<int32_t> w;
    w.reserve(n);
    std::vector<std::thread> th2;
    for (int i = 0; i < nt; i++)
      th2.emplace_back([&, i] {
        size_t a = bytes * i / nt, b = bytes * (i + 1) / nt;
        for (size_t o = a; o < b; o += 4096) ((volatile char*)w.data())[o] = 0;
      });
    for (auto& x : th2) x.join();
    double t6 = now();
    w.resize(n);
    double t7 = now();
    printf("n=%zu: vector(n) %.1f ms | pageable D2H fresh-faulted %.1f ms (%.1f GB/s), again %.1f ms (%.1f GB/s) | "
           "pinned D2H %.1f ms (%.1f GB/s) | %d-thread memcpy pinned->vector %.1f ms | %d-thread prefault %.1f ms + "
           "resize %.1f ms\n",
           n, (t1 - t0) * 1e3, (t2 - t1) * 1e3, bytes / (t2 - t1) / 1e9, (t3 - t2) * 1e3, bytes / (t3 - t2) / 1e9,
           (t4 - t3) * 1e3, bytes / (t4 - t3) / 1e9, nt, (t5 - t4) * 1e3, nt, (t6 - t5) * 1e3, (t7 - t6) * 1e3);
  }
  return 0;
}
