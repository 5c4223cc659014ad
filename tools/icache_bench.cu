// icache_bench.cu -- cost of executing straight-line code for the first time in a launch
// (instruction fetch from L2) vs the second time (warm instruction cache), on every SM.
// A block of NI dependent-free integer ops (NI * 16 B of SASS) is run twice per launch;
// clock64 stamps around each pass (CTA 0, warp 0).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

template <int NI>
__global__ void __launch_bounds__(128, 1) straight(unsigned* out, long long* ts, int reps) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, a4 = a0 + 1u, a5 = a0 + 9u, a6 = a0 * 11u, a7 = a0 ^ 77u;
  for (int r = 0; r < reps; ++r) {
    long long t0 = clock64();
    asm volatile("" ::: "memory");
#pragma unroll
    for (int i = 0; i < NI / 8; ++i) {
      asm volatile("add.u32 %0, %0, %1;" : "+r"(a0) : "r"(a1));
      asm volatile("xor.b32 %0, %0, %1;" : "+r"(a4) : "r"(a5));
      asm volatile("xor.b32 %0, %0, %1;" : "+r"(a1) : "r"(a2));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(a5) : "r"(a6));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(a2) : "r"(a3));
      asm volatile("xor.b32 %0, %0, %1;" : "+r"(a6) : "r"(a7));
      asm volatile("xor.b32 %0, %0, %1;" : "+r"(a3) : "r"(a0));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(a7) : "r"(a4));
    }
    asm volatile("" ::: "memory");
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0 && r < 4) ts[r] = t1 - t0;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
}

template <int NI>
void run(int grid) {
  unsigned* out;
  long long* ts;
  cudaMalloc(&out, 1 << 22);
  cudaMalloc(&ts, 64);
  long long h[4];
  for (int it = 0; it < 3; ++it) {
    cudaMemset(ts, 0, 64);
    straight<NI><<<grid, 128>>>(out, ts, 2);
    cudaDeviceSynchronize();
  }
  cudaMemcpy(h, ts, 32, cudaMemcpyDeviceToHost);
  printf("NI=%5d (%6d B of SASS)  grid %3d : pass1 %7lld cyc  pass2 %7lld cyc  (%.1f vs %.1f cyc per 128-B line)\n",
         NI, NI * 16, grid, h[0], h[1], h[0] / (NI * 16 / 128.0), h[1] / (NI * 16 / 128.0));
  cudaFree(out);
  cudaFree(ts);
}

int main() {
  for (int g : {1, 148}) {
    run<256>(g);
    run<1024>(g);
    run<4096>(g);
  }
  return 0;
}
