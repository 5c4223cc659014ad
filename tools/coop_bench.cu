// coop_bench.cu -- cost of cooperative launch and grid barriers on B200 (graph-replayed).
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ void atomic_barrier(unsigned* count, unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vg = gen;
    const unsigned g = *vg;
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *count = 0;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*vg == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

template <int MODE>  // 0 empty, 1 two cg grid syncs, 2 two atomic barriers
__global__ void __launch_bounds__(640, 1) k(unsigned* ws, int* out) {
  extern __shared__ char sm[];
  if (MODE == 1) { cg::this_grid().sync(); cg::this_grid().sync(); }
  if (MODE == 2) { atomic_barrier(ws, ws + 1); atomic_barrier(ws, ws + 1); }
  if (threadIdx.x == 0 && out) out[blockIdx.x] = sm[0];
}

template <int MODE>
float run(int G, bool coop, unsigned* ws, int* out) {
  cudaStream_t s; cudaStreamCreate(&s);
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G); cfg.blockDim = dim3(640); cfg.dynamicSmemBytes = 120 * 1024; cfg.stream = s;
  cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeCooperative; a[0].val.cooperative = 1;
  cfg.attrs = a; cfg.numAttrs = coop ? 1 : 0;
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 200; ++i) cudaLaunchKernelEx(&cfg, k<MODE>, ws, out);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, s); for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s); cudaEventRecord(e1, s);
  cudaStreamSynchronize(s);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("err %s\n", cudaGetErrorString(err));
  return ms * 1e3f / 1000.f;
}

int main() {
  unsigned* ws; int* out; cudaMalloc(&ws, 64); cudaMemset(ws, 0, 64); cudaMalloc(&out, 4096);
  for (int G : {5, 148}) {
    printf("G=%3d empty normal %.2f us | empty coop %.2f us | coop + 2 cg syncs %.2f us | normal + 2 atomic %.2f us | coop + 2 atomic %.2f us\n",
           G, run<0>(G, false, ws, out), run<0>(G, true, ws, out), run<1>(G, true, ws, out),
           run<2>(G, false, ws, out), run<2>(G, true, ws, out));
  }
  return 0;
}
