// peaks_bench.cu -- measured roofline denominators for bench.py (VERDICT r1 "Measured
// roofline denominators") and the division microbenchmark of SURVEY 8(f) N4:
//   1. tcgen05.mma.cta_group::1.kind::i8 throughput (M = 128, N = 256, K = 32 per
//      instruction, SS operands, s32 accumulators in TMEM), one issuing thread per SM;
//   2. the integer softmax element mix exactly as the attention kernel compiles it
//      (row max VIMNMX + shift_exp2_requant<FASTQ> + cvt.pack.sat, 32 independent
//      elements per thread, 16 warps per SM = the softmax warps of configuration 0);
//   3. the quotient q = floor(x / s_inv) of Alg. 2 (eq:q_div P:L822 vs
//      eq:q_mulshift P:L831-835): a runtime integer division (nvcc lowers it to
//      I2F/MUFU.RCP/F2I + fix-ups on sm_100a) against the exact one-IMAD.HI magic the
//      kernel uses, against the paper's literal mul+shift (M = round(2^32 / s_inv)).
// Prints one JSON object.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I include -I paper_2604_25306_b200/csrc tools/peaks_bench.cu -o tools/peaks_bench -lcuda
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "qflash_attn_kernel.cuh"

using namespace qf;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

// ------------------------------------------------------------ 1. tcgen05 kind::i8
__global__ void __launch_bounds__(128, 1) mma_peak(long long* out, int iters) {
  __shared__ __align__(1024) uint8_t sA[128 * 32];
  __shared__ __align__(1024) uint8_t sB[256 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 128 * 32 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sA)[i] = 0x01020304u * i;
  for (int i = threadIdx.x; i < 256 * 32 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sB)[i] = 0x05060708u ^ i;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(&slot, 512);
    tmem_relinquish();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc_i8(128, 256, 0, 0);
    const uint64_t da = make_smem_desc(smem_u32(sA), 16, 256, 6);  // SW32, 32-byte rows
    const uint64_t db = make_smem_desc(smem_u32(sB), 16, 256, 6);
    const long long c0 = clock64();
    const long long t0 = globaltimer_ns();
    for (int i = 0; i < iters; ++i) mma_i8_ss(tbase + (i & 1) * 256, da, db, idesc, i > 1 ? 1u : 0u);
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[2 * blockIdx.x] = clock64() - c0;
    out[2 * blockIdx.x + 1] = globaltimer_ns() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

// ------------------------------------------------------------ 2. softmax element mix
constexpr int kElems = 32;
__global__ void __launch_bounds__(512, 1) elem_mix(IntParams prm, uint32_t* sink, long long* out, int iters) {
  uint32_t s[kElems];
#pragma unroll
  for (int e = 0; e < kElems; ++e) s[e] = (threadIdx.x * 977u + e * 131u) & 0xFFFFu;
  uint32_t acc = 0;
  const long long c0 = clock64();
  const long long t0 = globaltimer_ns();
  const uint32_t one = 1u, s_inv = static_cast<uint32_t>(prm.s_inv);
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    // (2)(3) row max (the kernel's VIMNMX3 over the thread's columns)
    int32_t tmax = INT32_MIN;
#pragma unroll
    for (int e = 0; e < kElems; ++e) tmax = max(tmax, static_cast<int32_t>(s[e]));
    const int32_t m_new = tmax + (it & 7);
    const uint32_t mu = static_cast<uint32_t>(m_new), nmu = static_cast<uint32_t>(-m_new), c3 = s_inv - mu;
    // (5)(6) P = Requant(ShiftExp2(S - m_new)), packed 4 per word
#pragma unroll
    for (int e = 0; e < kElems; e += 4)
      acc ^= pack4_sat_s8(shift_exp2_requant<true, false>(static_cast<int32_t>(s[e]), mu, nmu, c3, one, prm),
                          shift_exp2_requant<true, true>(static_cast<int32_t>(s[e + 1]), mu, nmu, c3, one, prm),
                          shift_exp2_requant<true, false>(static_cast<int32_t>(s[e + 2]), mu, nmu, c3, one, prm),
                          shift_exp2_requant<true, true>(static_cast<int32_t>(s[e + 3]), mu, nmu, c3, one, prm));
  }
  const long long c1 = clock64();
  const long long t1 = globaltimer_ns();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = c1 - c0;
    out[2 * blockIdx.x + 1] = t1 - t0;
  }
}

// ------------------------------------------------------------ 3. quotient forms
template <int FORM>
__global__ void __launch_bounds__(512, 1) quotient(uint32_t divisor, uint32_t magic, uint32_t* sink,
                                                   long long* out, int iters) {
  uint32_t x[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) x[e] = threadIdx.x * 4099u + e * 65537u;
  uint32_t acc = 0;
  const long long c0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const uint32_t v = (x[e] + it) & 0x3FFFFFu;  // d in [0, 2^22)
      uint32_t q;
      if (FORM == 0) {
        q = v / divisor;  // eq:q_div, loop-invariant divisor: nvcc hoists the reciprocal
      } else if (FORM == 1) {
        // eq:q_div with a divisor that differs per element and iteration: the full
        // division sequence (reciprocal + multiply + correction) per quotient
        q = v / (divisor + static_cast<uint32_t>((it & 3) + e));
      } else {
        q = __umulhi(v, magic);  // one IMAD.HI (the kernel's exact magic / eq:q_mulshift)
      }
      acc += q;
    }
  }
  const long long c1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) out[blockIdx.x] = c1 - c0;
}

int main() {
  int sms = 0, clk_khz = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  long long* d_out;
  uint32_t* d_sink;
  CK(cudaMalloc(&d_out, 2 * sms * sizeof(long long)));
  CK(cudaMalloc(&d_sink, sms * 512 * sizeof(uint32_t)));
  std::vector<long long> h(2 * sms);
  auto span_ns = [&](int n) {
    long long mx = 0;
    for (int b = 0; b < n; ++b) mx = h[2 * b + 1] > mx ? h[2 * b + 1] : mx;
    return mx;
  };
  auto mean_cyc = [&](int n, int stride) {
    double s = 0;
    for (int b = 0; b < n; ++b) s += static_cast<double>(h[stride * b]);
    return s / n;
  };

  // 1. tensor core
  const int mma_iters = 40000;
  mma_peak<<<sms, 128>>>(d_out, 256);
  CK(cudaDeviceSynchronize());
  mma_peak<<<sms, 128>>>(d_out, mma_iters);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h.data(), d_out, 2 * sms * sizeof(long long), cudaMemcpyDeviceToHost));
  const double mma_ops = 2.0 * 128 * 256 * 32 * static_cast<double>(mma_iters) * sms;
  const double mma_ns = static_cast<double>(span_ns(sms));
  const double mma_cyc = mean_cyc(sms, 2);
  const double mma_tops = mma_ops / (mma_ns * 1e-9) / 1e12;
  const double macs_per_clk = 128.0 * 256 * 32 * mma_iters / mma_cyc;

  // 2. softmax element mix (FASTQ constants of a typical scale: s_q = s_k = 0.055, d = 64)
  IntParams prm{};
  prm.s_inv = 1834;
  prm.q_magic = static_cast<uint32_t>(((1ull << 32) + 1833) / 1834);
  prm.q_shift = 0;
  prm.m_p = 283;
  prm.r_p = 12;
  prm.one = 1;
  const int el_iters = 20000;
  elem_mix<<<sms, 512>>>(prm, d_sink, d_out, 64);
  CK(cudaDeviceSynchronize());
  elem_mix<<<sms, 512>>>(prm, d_sink, d_out, el_iters);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h.data(), d_out, 2 * sms * sizeof(long long), cudaMemcpyDeviceToHost));
  const double elems = static_cast<double>(kElems) * el_iters * 512.0 * sms;
  const double el_ns = static_cast<double>(span_ns(sms));
  const double el_cyc = mean_cyc(sms, 2);
  const double el_per_s = elems / (el_ns * 1e-9);
  const double el_per_clk_sm = kElems * static_cast<double>(el_iters) * 512.0 / el_cyc;

  // 3. quotient forms
  const int q_iters = 4096;
  double qrate[3];
  for (int f = 0; f < 3; ++f) {
    for (int rep = 0; rep < 2; ++rep) {
      if (f == 0) quotient<0><<<sms, 512>>>(1834u, 0u, d_sink, d_out, rep ? q_iters : 16);
      else if (f == 1) quotient<1><<<sms, 512>>>(1834u, 0u, d_sink, d_out, rep ? q_iters : 16);
      else quotient<2><<<sms, 512>>>(1834u, prm.q_magic, d_sink, d_out, rep ? q_iters : 16);
      CK(cudaDeviceSynchronize());
    }
    CK(cudaMemcpy(h.data(), d_out, sms * sizeof(long long), cudaMemcpyDeviceToHost));
    qrate[f] = 16.0 * q_iters * 512.0 / mean_cyc(sms, 1);  // quotients per clock per SM
  }

  printf("{\"sms\": %d, \"clock_attr_mhz\": %.0f,\n", sms, clk_khz / 1e3);
  printf(" \"int8_tops\": %.1f, \"int8_macs_per_clk_sm\": %.0f, \"int8_source\": \"measured: tools/peaks_bench.cu, "
         "tcgen05.mma.cta_group::1.kind::i8 M128 N256 K32 back to back on every SM (%d per SM), SS operands\",\n",
         mma_tops, macs_per_clk, mma_iters);
  printf(" \"alu_elems_per_s\": %.4e, \"alu_elems_per_clk_sm\": %.2f, \"alu_source\": \"measured: tools/peaks_bench.cu, "
         "the kernel's element mix (VIMNMX row max + shift_exp2_requant<FASTQ> + cvt.pack.sat), 16 warps x 32 "
         "independent elements per SM; peak = 10 ops x this rate\",\n",
         el_per_s, el_per_clk_sm);
  printf(" \"quotient_per_clk_sm\": {\"div_invariant_divisor\": %.2f, \"div_opaque_divisor\": %.2f, "
         "\"imad_hi_magic\": %.2f, \"speedup_vs_opaque_div\": %.2f, \"speedup_vs_invariant_div\": %.2f}}\n",
         qrate[0], qrate[1], qrate[2], qrate[2] / qrate[1], qrate[2] / qrate[0]);
  return 0;
}
