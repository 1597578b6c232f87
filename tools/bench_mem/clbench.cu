// Calibration of the small-graph kernel's building blocks on one 16-CTA
// cluster of 1024 threads: __syncthreads, warp scan + barrier, cluster
// barrier, dependent L2 loads, dependent DSMEM loads, DSMEM atomics.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;
__global__ void __launch_bounds__(1024, 1) k(const uint32_t* chain, unsigned long long* out, int iters) {
  extern __shared__ uint32_t sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int t = threadIdx.x;
  for (int i = t; i < 8192; i += 1024) sm[i] = (i * 7 + 1) & 8191;
  cl.sync();
  unsigned long long c0, c1;
  uint32_t acc = 0;
  // 1 syncthreads
  c0 = clock64();
  for (int i = 0; i < iters; i++) { __syncthreads(); }
  c1 = clock64();
  if (t == 0 && cl.block_rank() == 0) out[0] = (c1 - c0) / iters;
  // 2 warp scan + barrier + 32 LDS
  __shared__ unsigned red[2][32];
  c0 = clock64();
  for (int i = 0; i < iters; i++) {
    unsigned incl = t + i;
    for (int o = 1; o < 32; o <<= 1) { unsigned y = __shfl_up_sync(~0u, incl, o); if ((t & 31) >= o) incl += y; }
    if ((t & 31) == 31) red[i & 1][t >> 5] = incl;
    __syncthreads();
    unsigned s = 0;
    for (int j = 0; j < 32; j++) s += red[i & 1][j];
    acc += s;
  }
  c1 = clock64();
  if (t == 0 && cl.block_rank() == 0) out[1] = (c1 - c0) / iters;
  // 3 cluster barrier
  c0 = clock64();
  for (int i = 0; i < iters; i++) cl.sync();
  c1 = clock64();
  if (t == 0 && cl.block_rank() == 0) out[2] = (c1 - c0) / iters;
  // 4 dependent global loads (L2-resident 32 KB chain)
  uint32_t p = t & 8191;
  c0 = clock64();
  for (int i = 0; i < iters; i++) p = __ldcg(chain + p);
  c1 = clock64();
  acc += p;
  if (t == 0 && cl.block_rank() == 0) out[3] = (c1 - c0) / iters;
  // 5 dependent DSMEM loads
  p = t & 8191;
  c0 = clock64();
  for (int i = 0; i < iters; i++) { const uint32_t* r = cl.map_shared_rank(sm, (int)((cl.block_rank() + 1) % cl.num_blocks())); p = r[p]; }
  c1 = clock64();
  acc += p;
  if (t == 0 && cl.block_rank() == 0) out[4] = (c1 - c0) / iters;
  cl.sync();
  // 6 DSMEM atomics: every thread 8 atomics to random remote words per iteration
  c0 = clock64();
  for (int i = 0; i < iters; i++) {
    uint32_t* r = cl.map_shared_rank(sm, (int)((cl.block_rank() + i) % cl.num_blocks()));
    acc += atomicOr(r + ((t * 131 + i * 17) & 8191), 1u);
  }
  __syncthreads();
  c1 = clock64();
  if (t == 0 && cl.block_rank() == 0) out[5] = (c1 - c0) / iters;
  // 7 local smem atomics
  c0 = clock64();
  for (int i = 0; i < iters; i++) acc += atomicOr(sm + ((t * 131 + i * 17) & 8191), 1u);
  __syncthreads();
  c1 = clock64();
  if (t == 0 && cl.block_rank() == 0) out[6] = (c1 - c0) / iters;
  // 8 dependent global loads, HBM (64 MB chain, random)
  cl.sync();
  if (acc == 0x12345678) out[7] = acc;
}
int main() {
  uint32_t* chain; unsigned long long* out;
  cudaMalloc(&chain, 8192 * 4); cudaMalloc(&out, 64);
  uint32_t h[8192]; for (int i = 0; i < 8192; i++) h[i] = (i * 4099 + 77) & 8191;
  cudaMemcpy(chain, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {16, 8, 1}) {
    cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = 200 * 1024; cfg.attrs = a; cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; rep++) cudaLaunchKernelEx(&cfg, k, (const uint32_t*)chain, out, 200);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long r[8]; cudaMemcpy(r, out, 64, cudaMemcpyDeviceToHost);
    printf("cluster %d (%s): syncthreads %llu  scan+bar %llu  cl.sync %llu  L2 dep-load %llu  DSMEM dep-load %llu  DSMEM atomic/iter %llu  smem atomic/iter %llu (cycles)\n",
           cs, cudaGetErrorString(e), r[0], r[1], r[2], r[3], r[4], r[5], r[6]);
  }
  // launch overhead: events around empty cluster launches
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = 16; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(16); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = 200 * 1024; cfg.attrs = a; cfg.numAttrs = 1;
  for (int rep = 0; rep < 5; rep++) {
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k, (const uint32_t*)chain, out, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("event-timed cluster launch with iters=0: %.1f us\n", ms * 1e3);
  }
  return 0;
}
