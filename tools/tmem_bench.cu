// tmem_bench.cu -- tcgen05.ld / tcgen05.st throughput per SM (B200, sm_100a).
// One CTA per SM, W warps; warp w reads TMEM lane quarter (w & 3), columns
// [32 (w >> 2) .. +32) of a 512-column allocation, x32 per instruction.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2604_25306_b200/csrc/ptx.cuh"

using namespace qf;

template <int MODE>  // 0: ld x32 + wait each, 1: 2 x ld x32 then wait, 2: st x32 + wait
__global__ void tbench(uint32_t* out, long long* cyc, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) { tmem_alloc(&slot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot + ((static_cast<uint32_t>(warp & 3) * 32) << 16) + 32 * ((warp >> 2) & 7);
  uint32_t acc = 0, r[32], r2[32];
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
      tmem_ld32(base, r); tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += r[i];
    } else if (MODE == 1) {
      tmem_ld32(base, r); tmem_ld32(base + 256, r2); tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += r[i] ^ r2[i];
    } else {
      r[it & 31] = acc;
      tmem_st32(base, r); tmem_wait_st();
      acc += r[(it + 3) & 31];
    }
  }
  long long t1 = clock64();
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(slot, 512);
}

template <int MODE>
void run(int warps, const char* name) {
  const int sms = 148, iters = 2048;
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, sms * 1024 * 4); cudaMalloc(&cyc, sms * 8);
  tbench<MODE><<<sms, warps * 32>>>(out, cyc, iters);
  tbench<MODE><<<sms, warps * 32>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
  const double loads = (MODE == 1 ? 2.0 : 1.0) * iters * warps;  // warp-instructions of 32x32b.x32 (4 KB each)
  printf("%-28s warps %2d: %8.1f cyc/iter  %7.1f B/clk/SM  err=%s\n", name, warps, avg / iters,
         loads * 4096.0 / avg, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16}) run<0>(w, "ld x32 + wait");
  for (int w : {4, 8, 16}) run<1>(w, "2x ld x32 + wait");
  for (int w : {4, 8, 16}) run<2>(w, "st x32 + wait");
  return 0;
}
