// Trial overhead of the small-graph path: stream-ordered pool alloc + cluster
// launch, versus one CUDA graph launch holding the alloc node and the kernel.
#include <cstdio>
__global__ void __launch_bounds__(512, 1) kemp(int* p, int src) { if (threadIdx.x == 0 && blockIdx.x == 0) p[0] = src; }
int main() {
  cudaFuncSetAttribute(kemp, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(kemp, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaMemPool_t pool; cudaMemPoolProps props{}; props.allocType = cudaMemAllocationTypePinned; props.location.type = cudaMemLocationTypeDevice; props.location.id = 0;
  cudaMemPoolCreate(&pool, &props); unsigned long long keep = ~0ull; cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = 16; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(16); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 200 * 1024; cfg.stream = s; cfg.attrs = a; cfg.numAttrs = 1;
  void* prev = nullptr;
  float tot = 0;
  for (int rep = 0; rep < 30; rep++) {
    if (prev) cudaFreeAsync(prev, s);
    int* p;
    cudaEventRecord(e0, s);
    cudaMallocFromPoolAsync((void**)&p, 1 << 20, pool, s);
    cudaLaunchKernelEx(&cfg, kemp, p, rep);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    prev = p;
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep >= 10) tot += ms;
  }
  cudaFreeAsync(prev, s); cudaStreamSynchronize(s);
  printf("stream: pool alloc + cluster launch: %.2f us\n", tot / 20 * 1e3);
  // graph
  cudaGraph_t g; cudaGraphExec_t ge;
  int* gp = nullptr;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  cudaMallocAsync((void**)&gp, 1 << 20, s);
  cudaLaunchKernelEx(&cfg, kemp, gp, 0);
  cudaStreamEndCapture(s, &g);
  cudaError_t err = cudaGraphInstantiate(&ge, g, 0);
  printf("instantiate: %s\n", cudaGetErrorString(err));
  cudaGraphNode_t nodes[8]; size_t nn = 8; cudaGraphGetNodes(g, nodes, &nn);
  cudaGraphNode_t kn = nullptr;
  for (size_t i = 0; i < nn; i++) { cudaGraphNodeType t; cudaGraphNodeGetType(nodes[i], &t); if (t == cudaGraphNodeTypeKernel) kn = nodes[i]; }
  tot = 0;
  for (int rep = 0; rep < 30; rep++) {
    cudaKernelNodeParams kp; cudaGraphKernelNodeGetParams(kn, &kp);
    int src = rep; void* args[] = {&gp, &src}; kp.kernelParams = args;
    cudaGraphExecKernelNodeSetParams(ge, kn, &kp);
    cudaEventRecord(e0, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaFreeAsync(gp, s);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep >= 10) tot += ms;
  }
  cudaStreamSynchronize(s);
  printf("graph: alloc node + cluster kernel: %.2f us (%s)\n", tot / 20 * 1e3, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
