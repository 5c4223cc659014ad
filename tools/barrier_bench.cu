// barrier_bench.cu -- per-barrier cost on B200 for the fused step's grid barriers: cooperative
// groups grid.sync(), a release/acquire counter barrier (one atomic arrive, one polled word),
// and the hardware cluster barrier (G <= 16), each with and without 29 KB of global stores per
// CTA before the barrier (the quantized codes the next phase reads).  640 threads x 1 CTA / SM.
// Time = (globaltimer after NB barriers - before) / NB, CTA 0, median of 5 launches.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// counter barrier: monotonically increasing 32-bit counter, target = (arrival / G + 1) * G
__device__ __forceinline__ void counter_barrier(unsigned* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
    const unsigned target = (old / gridDim.x + 1) * gridDim.x;
    for (int spin = 0; spin < (1 << 22) && static_cast<int>(ld_acquire(ctr) - target) < 0; ++spin) {
    }
  }
  __syncthreads();
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int NB = 16;
template <int MODE, bool STORES>  // 0 cg grid.sync, 1 counter barrier, 2 cluster barrier
__global__ void __launch_bounds__(640, 1) k(unsigned* ctr, unsigned* sink, unsigned long long* t) {
  const unsigned long long t0 = gtimer();
  for (int i = 0; i < NB; ++i) {
    if (STORES) {  // 12 coalesced 4-B stores per thread (29 KB per CTA), like the codes
#pragma unroll
      for (int u = 0; u < 12; ++u) sink[(static_cast<size_t>(i & 1) * 12 + u) * gridDim.x * 640 + blockIdx.x * 640 + threadIdx.x] = i + u;
    }
    if (MODE == 0) cg::this_grid().sync();
    else if (MODE == 1) counter_barrier(ctr);
    else cluster_barrier();
  }
  const unsigned long long t1 = gtimer();
  if (threadIdx.x == 0 && blockIdx.x == 0) *t = t1 - t0;
}

template <int MODE, bool STORES>
double run(int G, unsigned* ctr, unsigned* sink, unsigned long long* t) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(640);
  cudaLaunchAttribute a[1];
  if (MODE == 2) {
    cudaFuncSetAttribute(k<MODE, STORES>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = G;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
  } else {
    a[0].id = cudaLaunchAttributeCooperative;
    a[0].val.cooperative = 1;
  }
  cfg.attrs = a;
  cfg.numAttrs = 1;
  std::vector<double> v;
  for (int r = 0; r < 7; ++r) {
    cudaMemset(ctr, 0, 64);  // the counter barrier's targets assume a multiple of G
    if (cudaLaunchKernelEx(&cfg, k<MODE, STORES>, ctr, sink, t) != cudaSuccess) return -1;
    cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
    if (r >= 2) v.push_back(h / 1e3 / NB);
  }
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

int main() {
  unsigned *ctr, *sink;
  unsigned long long* t;
  cudaMalloc(&ctr, 64);
  cudaMemset(ctr, 0, 64);
  cudaMalloc(&sink, 2ull * 12 * 148 * 640 * 4);
  cudaMalloc(&t, 8);
  for (int G : {6, 16, 148}) {
    printf("G=%3d  grid.sync %.2f / +stores %.2f us | counter barrier %.2f / +stores %.2f us", G,
           run<0, false>(G, ctr, sink, t), run<0, true>(G, ctr, sink, t), run<1, false>(G, ctr, sink, t),
           run<1, true>(G, ctr, sink, t));
    if (G <= 16) printf(" | cluster barrier %.2f / +stores %.2f us", run<2, false>(G, ctr, sink, t), run<2, true>(G, ctr, sink, t));
    printf("\n");
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return 0;
}
