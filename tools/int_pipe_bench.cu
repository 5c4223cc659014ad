// int_pipe_bench.cu -- INT32 pipe throughput microbenchmark for the integer
// softmax (SURVEY build step 1): per-SM throughput of the SASS instructions the
// ShiftExp2/requant/release sequences compile to.  One CTA per SM, 16 warps,
// 8 independent dependency chains per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
#define ITERS 4096

template <int OP>
__global__ void bench(uint32_t* out, long long* cyc, uint32_t seed) {
  uint32_t a[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = seed * (threadIdx.x + 1) + c * 7919u;
  const uint32_t k1 = seed | 1u, k2 = seed >> 3;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      uint32_t x = a[c], d;
      if (OP == 0) {        // IADD3 (3-input add)
        asm volatile("{.reg .u32 t; add.u32 t, %1, %2; add.u32 %0, t, %3;}" : "=r"(d) : "r"(x), "r"(k1), "r"(k2));
      } else if (OP == 1) { // IMAD (mad.lo)
        asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(k1), "r"(k2));
      } else if (OP == 2) { // IMAD.HI
        asm volatile("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(k1), "r"(k2));
      } else if (OP == 3) { // IMAD.WIDE
        uint64_t w;
        asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w) : "r"(x), "r"(k1));
        d = static_cast<uint32_t>(w) ^ static_cast<uint32_t>(w >> 32);
      } else if (OP == 4) { // SHF (funnel shift clamp)
        asm volatile("shf.r.clamp.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(k2), "r"(k1));
      } else if (OP == 5) { // LOP3
        asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(x), "r"(k1), "r"(k2));
      } else if (OP == 6) { // I2IP pack
        asm volatile("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(k1), "r"(k2));
      } else if (OP == 7) { // 3-input max
        asm volatile("max.s32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(k1));
      } else {              // the ShiftExp2 + requant element (8 ops incl. pack/max halves)
        const uint32_t d1 = x + (0u - k1) + k2;
        const uint32_t q1 = __umulhi(d1, 2196u * 1024u + 7u);
        const uint32_t num = q1 * 2049u + (x + k2 - k1);
        const uint32_t y = __funnelshift_rc(num, 0u, q1);
        d = __umulhi(y, 383778816u) + x;
      }
      a[c] = d;
    }
  }
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc ^= a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
double run(const char* name, int sms, int threads, uint32_t* out, long long* cyc) {
  bench<OP><<<sms, threads>>>(out, cyc, 12345u);
  bench<OP><<<sms, threads>>>(out, cyc, 12345u);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double ops = double(threads) * ITERS * CH;  // thread-ops per SM
  const double per_clk = ops / mx;
  printf("%-28s %7.1f thread-ops/clk/SM  (%5.2f warp-instr/clk/SMSP)\n", name, per_clk, per_clk / 32 / 4);
  return per_clk;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 512;
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(uint32_t) * sms * threads);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  printf("SMs %d, %d threads/SM, %d chains/thread\n", sms, threads, CH);
  run<0>("IADD3 (3-input add)", sms, threads, out, cyc);
  run<1>("IMAD (mad.lo)", sms, threads, out, cyc);
  run<2>("IMAD.HI (mad.hi)", sms, threads, out, cyc);
  run<3>("IMAD.WIDE (+LOP3)", sms, threads, out, cyc);
  run<4>("SHF (shf.r.clamp)", sms, threads, out, cyc);
  run<5>("LOP3", sms, threads, out, cyc);
  run<6>("I2IP (cvt.pack.sat)", sms, threads, out, cyc);
  run<7>("IMNMX (max.s32)", sms, threads, out, cyc);
  double e = run<8>("ShiftExp2+requant element", sms, threads, out, cyc);
  printf("=> elements/clk/SM %.1f (x5 ops each as written)\n", e);
  return 0;
}
