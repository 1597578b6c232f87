// Grid-barrier latency on B200: per-barrier cost of several software grid
// barriers inside one cooperative launch (10000 back-to-back barriers).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

struct Bar { unsigned count; unsigned gen; unsigned pad[30]; };

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned r;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// mode 0: threadfence + atomicAdd + acquire spin (current gk kernel, no sleep)
// mode 1: atom.acq_rel arrive, last arriver red.release, ld.acquire spin
// mode 2: counter-only (monotonic count, target = gen*grid), red.release arrive, acquire spin
// mode 3: cooperative_groups grid.sync()
template <int kMode>
__global__ void bar_kernel(Bar* b, int iters, unsigned long long* out) {
  unsigned gen = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
    if (kMode == 3) {
      cg::this_grid().sync();
      continue;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (kMode == 0) {
        __threadfence();
        unsigned a = atomicAdd(&b->count, 1u);
        if (a == gridDim.x - 1) {
          atomicExch(&b->count, 0u);
          __threadfence();
          atomicAdd(&b->gen, 1u);
        } else {
          while (ld_acquire(&b->gen) == gen) {}
        }
        __threadfence();
      } else if (kMode == 1) {
        unsigned a = atom_add_acqrel(&b->count, 1u);
        if (a == gridDim.x - 1) {
          b->count = 0;
          red_release(&b->gen, 1u);
        } else {
          while (ld_acquire(&b->gen) == gen) {}
        }
      } else {
        red_release(&b->count, 1u);
        const unsigned target = (gen + 1) * gridDim.x;
        while (ld_acquire(&b->count) < target) {}
      }
    }
    gen++;
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

template <int kMode>
void run(int grid, int block, const char* name) {
  Bar* b;
  unsigned long long* out;
  cudaMalloc(&b, sizeof(Bar));
  cudaMalloc(&out, 8);
  cudaMemset(b, 0, sizeof(Bar));
  int iters = 10000;
  void* args[] = {&b, &iters, &out};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchCooperativeKernel((void*)bar_kernel<kMode>, grid, block, args, 0, 0);  // warm
  cudaMemset(b, 0, sizeof(Bar));
  cudaEventRecord(e0);
  cudaError_t e = cudaLaunchCooperativeKernel((void*)bar_kernel<kMode>, grid, block, args, 0, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("%-34s grid %4d x %4d: %.3f us/barrier  (%s)\n", name, grid, block, ms * 1000 / iters,
         cudaGetErrorString(e));
  cudaFree(b);
  cudaFree(out);
}

int main() {
  for (auto gb : {std::pair<int, int>{296, 512}, {148, 1024}, {148, 512}, {592, 256}}) {
    run<0>(gb.first, gb.second, "fence+atomicAdd+gen");
    run<1>(gb.first, gb.second, "atom.acq_rel + red.release gen");
    run<2>(gb.first, gb.second, "red.release count, acquire spin");
    run<3>(gb.first, gb.second, "cg::grid.sync");
  }
  return 0;
}
