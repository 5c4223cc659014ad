// qflash_quant.cu -- per-tensor int8 quantizer (Eq. 2) and the
// dequantizer, HBM-bound streaming kernels for sm_100a.
//
// Quantization of T tensors (T = 1, or 3 for fused Q/K/V) is two launches:
//   1. amax: each block reduces max|x| (fmaxf with |.| source modifier: one
//      FMNMX per element) and atomically maxes s_b = fl32(amax_b / 127) into the
//      caller's pre-zeroed scale slot.  fl32 division is monotone, so the slot
//      ends at fl32(max_b amax_b / 127) = fl32(amax / 127).  Grids are sized to
//      ~8 blocks per SM in total, so each slot sees a few hundred atomics.
//   2. quantize: x^ = sat8(roundf(fl32(x / s))) (readings R1, R2) with s = 1/127
//      when the slot is 0 (R3).  Exact fast path: q = RN(x * RN(1/s)) is within
//      2^-15 of fl32(x / s) for |x / s| <= 128, so whenever q is farther than
//      0.5 - 2^-14 from a half-integer, rint(q) == roundf(fl32(x / s)); the
//      remaining elements (probability ~2^-13) take the IEEE division.  Block 0
//      of tensor 0 can also derive the attention's integer constants from the
//      final s_q, s_k (qflash_quantize_qkv_prepare) so the step needs no extra
//      launch.
// 16 elements per thread and iteration (64 B of fp32 in flight, one 16-B store).
//
// Single-pass variant (quantize_fused_kernel, three tensors): when every
// thread's share of Q, K and V fits in registers (<= 4 16-byte vectors per
// tensor), a cooperative grid (2 CTAs per SM) loads its share once, reduces the
// per-CTA amax, exchanges the partials through the caller's workspace around one
// grid barrier, and quantizes from registers: HBM is read once, one launch, no
// memset, no atomics.  Larger tensors take the two-pass path above.
//
// The attention, dequantize and second quantize launches use programmatic
// dependent launch (their prologue and launch latency overlap the previous
// grid's tail); every PDL-launched kernel calls griddep_wait() before its first
// global access.  Measured on B200 (tools/gpu_pdl_ab.sh): A3 b8 step 23.9 ->
// 23.0-23.4 us, A4 b8 35.5 -> 33.0 us, A1 b1 15.8 -> 14.6-15.0 us.
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "ptx.cuh"
#include "qflash_common.cuh"
#include "qflash_params.cuh"
#include "qflash_quant_elem.cuh"

namespace qf {

constexpr int kQThreads = 256;
constexpr int kDqTableOffset = kWsDqTableOffset;  // workspace bytes of the 256-entry dequant table
static_assert(kQThreads == 256, "one thread per dequant-table entry");
constexpr int kQElems = 16;  // elements per thread per iteration

template <typename T>
struct Load16;  // 16 consecutive elements widened (exactly) to fp32
template <>
struct Load16<float> {
  __device__ static void load(const void* base, int64_t i, float* o) {
    const float4* p = reinterpret_cast<const float4*>(base) + 4 * i;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 v = __ldg(p + k);
      o[4 * k] = v.x; o[4 * k + 1] = v.y; o[4 * k + 2] = v.z; o[4 * k + 3] = v.w;
    }
  }
  __device__ static float load1(const void* base, int64_t i) {
    return __ldg(reinterpret_cast<const float*>(base) + i);
  }
};
template <>
struct Load16<__nv_bfloat16> {
  __device__ static void load(const void* base, int64_t i, float* o) {
    const uint4* p = reinterpret_cast<const uint4*>(base) + 2 * i;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint4 v = __ldg(p + k);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        o[8 * k + 2 * e] = __uint_as_float(w[e] << 16);
        o[8 * k + 2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
      }
    }
  }
  __device__ static float load1(const void* base, int64_t i) {
    const uint16_t b = reinterpret_cast<const uint16_t*>(base)[i];
    return __uint_as_float(static_cast<uint32_t>(b) << 16);
  }
};
template <>
struct Load16<__half> {
  __device__ static void load(const void* base, int64_t i, float* o) {
    const uint4* p = reinterpret_cast<const uint4*>(base) + 2 * i;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint4 v = __ldg(p + k);
      const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __half22float2(h[e]);  // exact widening
        o[8 * k + 2 * e] = f.x;
        o[8 * k + 2 * e + 1] = f.y;
      }
    }
  }
  __device__ static float load1(const void* base, int64_t i) {
    return __half2float(reinterpret_cast<const __half*>(base)[i]);
  }
};

__device__ __forceinline__ const void* pick(const QuantTensors& t, int i) {
  return i == 0 ? t.x[0] : (i == 1 ? t.x[1] : t.x[2]);
}
__device__ __forceinline__ int8_t* pick_q(const QuantTensors& t, int i) {
  return i == 0 ? t.xq[0] : (i == 1 ? t.xq[1] : t.xq[2]);
}
__device__ __forceinline__ float* pick_s(const QuantTensors& t, int i) {
  return i == 0 ? t.scale[0] : (i == 1 ? t.scale[1] : t.scale[2]);
}

template <typename T>
__global__ void __launch_bounds__(kQThreads) amax_kernel(QuantTensors t, int64_t numel) {
  griddep_launch();  // let the quantize pass be scheduled early (it waits for us)
  const int ti = blockIdx.y;
  const void* x = pick(t, ti);
  const int64_t nv = numel / kQElems;
  float m[4] = {0.f, 0.f, 0.f, 0.f};
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nv; i += stride) {
    float v[kQElems];
    Load16<T>::load(x, i, v);
#pragma unroll
    for (int k = 0; k < kQElems; ++k) m[k & 3] = fmaxf(m[k & 3], fabsf(v[k]));
  }
  for (int64_t i = nv * kQElems + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < numel;
       i += stride)
    m[0] = fmaxf(m[0], fabsf(Load16<T>::load1(x, i)));
  float mm = fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o));
  __shared__ float red[kQThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mm;
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = red[0];
#pragma unroll
    for (int w = 1; w < kQThreads / 32; ++w) b = fmaxf(b, red[w]);
    // s_b = fl32(amax_b / 127) is monotone in amax_b; non-negative floats order
    // like their bit patterns, so an unsigned atomicMax on the bits is a float max.
    const float sb = __fdiv_rn(b, 127.0f);
    atomicMax(reinterpret_cast<unsigned int*>(pick_s(t, ti)), __float_as_uint(sb));
  }
}

template <typename T>
__global__ void __launch_bounds__(kQThreads)
    quantize_kernel(QuantTensors t, int64_t numel, IntParams* prm_out, int32_t head_dim) {
  griddep_wait();    // programmatic launch: the amax pass must be complete
  griddep_launch();
  const int ti = blockIdx.y;
  const void* x = pick(t, ti);
  int8_t* xq = pick_q(t, ti);
  float s = *reinterpret_cast<volatile float*>(pick_s(t, ti));
  if (s == 0.0f) s = 1.0f / 127.0f;  // all-zero tensor (R3)
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *pick_s(t, ti) = s;
    if (prm_out != nullptr && ti == 0) {
      // integer constants of the attention from the final s_q, s_k
      float sq = *reinterpret_cast<volatile float*>(t.scale[0]);
      float sk = *reinterpret_cast<volatile float*>(t.scale[1]);
      if (sq == 0.0f) sq = 1.0f / 127.0f;
      if (sk == 0.0f) sk = 1.0f / 127.0f;
      IntParams p;
      const int st = derive_core(sq, sk, head_dim, &p, nullptr);
      if (st != QFLASH_OK) {
        memset(&p, 0, sizeof(p));
        p.status = st;
      }
      *prm_out = p;
    }
  }
  if (blockIdx.x == 0 && ti == 2 && prm_out != nullptr) {
    // dequantization table of the fused attention epilogue: fl32(s_V * i), i = -128..127
    // (the same IEEE multiply as dequantize_kernel)
    reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(prm_out) + kDqTableOffset)[threadIdx.x] =
        __float_as_uint(__fmul_rn(s, static_cast<float>(static_cast<int>(threadIdx.x) - 128)));
  }
  const float r = __frcp_rn(s);
  const int64_t nv = numel / kQElems;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nv; i += stride) {
    float v[kQElems];
    Load16<T>::load(x, i, v);
    reinterpret_cast<uint4*>(xq)[i] = quant16(v, s, r);
  }
  for (int64_t i = nv * kQElems + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < numel;
       i += stride) {
    const int32_t v = quant_one(Load16<T>::load1(x, i), s, r);
    xq[i] = static_cast<int8_t>(max(-128, min(127, v)));
  }
}

// ----------------------------------------------------------- fused single pass
// Cooperative grid (2 CTAs x 256 threads per SM, 128 registers per thread).  Thread g of
// the grid owns the 16-byte vectors g, g + T, ..., g + (VPT-1) T of every tensor
// (coalesced), keeps them in registers across one grid barrier, and quantizes
// them with the global scale: one launch, HBM read once, no memset, no atomics.
constexpr int kFThreads = 256;
static_assert(kFThreads == 256, "one thread per dequant-table entry");
constexpr int kFBlocksPerSM = 2;

template <typename T>
__device__ __forceinline__ void widen16(const uint4& v, float* f);  // 16 B -> 16/sizeof(T) floats
template <>
__device__ __forceinline__ void widen16<float>(const uint4& v, float* f) {
  f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
  f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
}
template <>
__device__ __forceinline__ void widen16<__nv_bfloat16>(const uint4& v, float* f) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    f[2 * e] = __uint_as_float(w[e] << 16);
    f[2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
  }
}
template <>
__device__ __forceinline__ void widen16<__half>(const uint4& v, float* f) {
  const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 x = __half22float2(h[e]);
    f[2 * e] = x.x;
    f[2 * e + 1] = x.y;
  }
}

template <typename T, int VPT>
__global__ void __launch_bounds__(kFThreads, kFBlocksPerSM)
    quantize_fused_kernel(QuantTensors t, int64_t numel, float* partial, IntParams* prm_out,
                          int32_t head_dim) {
  namespace cg = cooperative_groups;
  constexpr int kE = 16 / sizeof(T);  // elements per 16-byte vector
  __shared__ float red[3][kFThreads / 32];
  __shared__ float sc[3];
  griddep_wait();
  const int64_t T_all = static_cast<int64_t>(gridDim.x) * kFThreads;
  const int64_t g = static_cast<int64_t>(blockIdx.x) * kFThreads + threadIdx.x;
  const int64_t nvec = numel / kE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  uint4 v[3][VPT];
  float m[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const uint4* src = reinterpret_cast<const uint4*>(pick(t, i));
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int64_t idx = g + u * T_all;
      v[i][u] = idx < nvec ? __ldg(src + idx) : make_uint4(0u, 0u, 0u, 0u);
    }
  }
  // tail elements (numel % kE): thread 0 of block 0 folds them into its amax
  // here and re-reads them for quantization after the barrier (<= 7 scalars)
  const int ntail = static_cast<int>(numel - nvec * kE);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      float f[kE];
      widen16<T>(v[i][u], f);
#pragma unroll
      for (int e = 0; e < kE; ++e) m[i] = fmaxf(m[i], fabsf(f[e]));
    }
    if (g == 0) {
      for (int e = 0; e < ntail; ++e) m[i] = fmaxf(m[i], fabsf(Load16<T>::load1(pick(t, i), nvec * kE + e)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m[i] = fmaxf(m[i], __shfl_xor_sync(0xffffffffu, m[i], o));
    if (lane == 0) red[i][warp] = m[i];
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    float b = 0.f;
#pragma unroll
    for (int w = 0; w < kFThreads / 32; ++w) b = fmaxf(b, red[threadIdx.x][w]);
    partial[threadIdx.x * gridDim.x + blockIdx.x] = b;
  }
  __threadfence();
  cg::this_grid().sync();
  // (no griddep_launch here: an early trigger measured ~1 us slower on A3 b8 -- the
  // attention grid is launched at our exit, still with its prologue overlapped)
  // per-tensor scale s = fl32(amax / 127) (R3: 1/127 for an all-zero tensor)
  if (warp < 3) {
    float b = 0.f;
    for (int j = lane; j < static_cast<int>(gridDim.x); j += 32) b = fmaxf(b, __ldcg(&partial[warp * gridDim.x + j]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
    if (lane == 0) {
      float s = __fdiv_rn(b, 127.0f);
      if (s == 0.0f) s = 1.0f / 127.0f;
      sc[warp] = s;
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && prm_out != nullptr) {
    // dequantization table of the fused attention epilogue: fl32(s_V * i), i = -128..127
    reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(prm_out) + kDqTableOffset)[threadIdx.x] =
        __float_as_uint(__fmul_rn(sc[2], static_cast<float>(static_cast<int>(threadIdx.x) - 128)));
  }
  if (g == 0) {
    for (int i = 0; i < 3; ++i) *pick_s(t, i) = sc[i];
    if (prm_out != nullptr) {
      IntParams p;
      const int st = derive_core(sc[0], sc[1], head_dim, &p, nullptr);
      if (st != QFLASH_OK) {
        memset(&p, 0, sizeof(p));
        p.status = st;
      }
      *prm_out = p;
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float s = sc[i];
    const float r = __frcp_rn(s);
    int8_t* xq = pick_q(t, i);
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int64_t idx = g + u * T_all;
      float f[16];
      widen16<T>(v[i][u], f);
      if constexpr (kE == 4) {
        // 4 elements -> one 32-bit store
        int32_t q[4];
        bool bad = false;
#pragma unroll
        for (int e = 0; e < 4; ++e) q[e] = quant_fast(f[e], r, bad);
        if (bad) {
#pragma unroll
          for (int e = 0; e < 4; ++e) q[e] = quant_exact(f[e], s);
        }
        uint32_t hi, lo;
        asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(q[3]), "r"(q[2]));
        asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(lo) : "r"(q[1]), "r"(q[0]), "r"(hi));
        if (idx < nvec) reinterpret_cast<uint32_t*>(xq)[idx] = lo;
      } else {
        int32_t q[8];
        bool bad = false;
#pragma unroll
        for (int e = 0; e < 8; ++e) q[e] = quant_fast(f[e], r, bad);
        if (bad) {
#pragma unroll
          for (int e = 0; e < 8; ++e) q[e] = quant_exact(f[e], s);
        }
        uint32_t w[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          uint32_t hi, lo;
          asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(q[4 * k + 3]), "r"(q[4 * k + 2]));
          asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(lo) : "r"(q[4 * k + 1]), "r"(q[4 * k]), "r"(hi));
          w[k] = lo;
        }
        if (idx < nvec) reinterpret_cast<uint2*>(xq)[idx] = make_uint2(w[0], w[1]);
      }
    }
    if (g == 0) {
      for (int e = 0; e < ntail; ++e)
        xq[nvec * kE + e] = static_cast<int8_t>(
            max(-128, min(127, quant_one(Load16<T>::load1(pick(t, i), nvec * kE + e), s, r))));
    }
  }
}

__global__ void __launch_bounds__(kQThreads)
    dequantize_kernel(const int8_t* __restrict__ xq, float scale, const float* __restrict__ scale_dev,
                      int64_t numel, float* __restrict__ y) {
  griddep_wait();  // programmatic launch: the producer of xq / scale must be complete
  const float s = scale_dev ? *scale_dev : scale;
  // 4 int8 per thread per step: one 4-B load and one 16-B store, both coalesced
  const int64_t n4 = numel / 4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += 2 * stride) {
    const uint32_t w0 = __ldg(reinterpret_cast<const uint32_t*>(xq) + i);
    const int64_t i2 = i + stride;
    const uint32_t w1 = i2 < n4 ? __ldg(reinterpret_cast<const uint32_t*>(xq) + i2) : 0u;
    reinterpret_cast<float4*>(y)[i] =
        make_float4(__fmul_rn(s, static_cast<float>(static_cast<int8_t>(w0 & 0xFF))),
                    __fmul_rn(s, static_cast<float>(static_cast<int8_t>((w0 >> 8) & 0xFF))),
                    __fmul_rn(s, static_cast<float>(static_cast<int8_t>((w0 >> 16) & 0xFF))),
                    __fmul_rn(s, static_cast<float>(static_cast<int8_t>(w0 >> 24))));
    if (i2 < n4)
      reinterpret_cast<float4*>(y)[i2] =
          make_float4(__fmul_rn(s, static_cast<float>(static_cast<int8_t>(w1 & 0xFF))),
                      __fmul_rn(s, static_cast<float>(static_cast<int8_t>((w1 >> 8) & 0xFF))),
                      __fmul_rn(s, static_cast<float>(static_cast<int8_t>((w1 >> 16) & 0xFF))),
                      __fmul_rn(s, static_cast<float>(static_cast<int8_t>(w1 >> 24))));
  }
  for (int64_t i = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < numel; i += stride)
    y[i] = __fmul_rn(s, static_cast<float>(xq[i]));
}

// ------------------------------------------------------- per-head granularity (N1)
// Problems are (batch, window, head) with the head fastest: head = problem mod H.
// Grid: x = problem, y = chunk of 1024 16-byte vectors of that problem, so every
// block sees one head.  Pass 1: block amax -> atomicMax of s = fl32(amax / 127)
// into scales[t * H + head] (pre-zeroed; fl32 division is monotone).  Pass 2:
// quantize with the head's final scale (0 -> 1/127, R3).
constexpr int kPHVec = 4;  // vectors per thread per block

__device__ __forceinline__ int head_of(int p, int H, uint32_t h_magic) {
  if (H == 1) return 0;  // ceil(2^32 / 1) does not fit the 32-bit magic
  const int q = static_cast<int>(__umulhi(static_cast<uint32_t>(p), h_magic));
  return p - q * H;
}

__global__ void __launch_bounds__(kQThreads)
    amax_per_head_kernel(QuantTensors t, int64_t vec_per_problem, int H, uint32_t h_magic) {
  const int ti = blockIdx.z;
  const int p = blockIdx.x;
  const float4* x = reinterpret_cast<const float4*>(pick(t, ti)) + static_cast<int64_t>(p) * vec_per_problem;
  float m = 0.f;
  const int64_t v0 = static_cast<int64_t>(blockIdx.y) * kQThreads * kPHVec + threadIdx.x;
#pragma unroll
  for (int u = 0; u < kPHVec; ++u) {
    const int64_t i = v0 + u * kQThreads;
    if (i < vec_per_problem) {
      const float4 v = __ldg(x + i);
      m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float red[kQThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = red[0];
#pragma unroll
    for (int w = 1; w < kQThreads / 32; ++w) b = fmaxf(b, red[w]);
    const float sb = __fdiv_rn(b, 127.0f);
    atomicMax(reinterpret_cast<unsigned int*>(pick_s(t, ti)) + head_of(p, H, h_magic), __float_as_uint(sb));
  }
}

__global__ void __launch_bounds__(kQThreads)
    quantize_per_head_kernel(QuantTensors t, int64_t vec_per_problem, int H, uint32_t h_magic) {
  const int ti = blockIdx.z;
  const int p = blockIdx.x;
  const int h = head_of(p, H, h_magic);
  float s = *reinterpret_cast<volatile float*>(pick_s(t, ti) + h);
  if (s == 0.0f) s = 1.0f / 127.0f;  // all-zero head (R3)
  if (p == h && blockIdx.y == 0 && threadIdx.x == 0) pick_s(t, ti)[h] = s;
  const float r = __frcp_rn(s);
  const float4* x = reinterpret_cast<const float4*>(pick(t, ti)) + static_cast<int64_t>(p) * vec_per_problem;
  uint32_t* xq = reinterpret_cast<uint32_t*>(pick_q(t, ti)) + static_cast<int64_t>(p) * vec_per_problem;
  const int64_t v0 = static_cast<int64_t>(blockIdx.y) * kQThreads * kPHVec + threadIdx.x;
#pragma unroll
  for (int u = 0; u < kPHVec; ++u) {
    const int64_t i = v0 + u * kQThreads;
    if (i < vec_per_problem) {
      const float4 v = __ldg(x + i);
      int32_t q[4];
      bool bad = false;
      q[0] = quant_fast(v.x, r, bad);
      q[1] = quant_fast(v.y, r, bad);
      q[2] = quant_fast(v.z, r, bad);
      q[3] = quant_fast(v.w, r, bad);
      if (bad) {
        q[0] = quant_exact(v.x, s);
        q[1] = quant_exact(v.y, s);
        q[2] = quant_exact(v.z, s);
        q[3] = quant_exact(v.w, s);
      }
      uint32_t hi, lo;
      asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(q[3]), "r"(q[2]));
      asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(lo) : "r"(q[1]), "r"(q[0]), "r"(hi));
      xq[i] = lo;
    }
  }
}

// Per-head integer constants: thread h derives head h's constants from
// (s_q[h], s_k[h]) with derive_core (the fp64 expression of qflash_derive_params)
// into table + kHeadPrmStride h; thread 0 then writes the header: status (first
// failing head's), and q_shift / s_inv / m_p chosen so that the kernel's fast-path
// test is true iff every head takes the fast quotient / requant path.
__global__ void derive_per_head_kernel(const float* __restrict__ scales, int H, int32_t d,
                                       char* __restrict__ ws) {
  __shared__ int fast_all, status;
  if (threadIdx.x == 0) {
    fast_all = 1;
    status = 0;
  }
  __syncthreads();
  for (int h = threadIdx.x; h < H; h += blockDim.x) {
    IntParams p;
    const int st = derive_core(scales[h], scales[H + h], d, &p, nullptr);
    if (st != QFLASH_OK) {
      memset(&p, 0, sizeof(p));
      p.status = st;
      atomicCAS(&status, 0, st);
    } else if (!(p.q_shift == 0 && static_cast<uint64_t>(p.s_inv) * static_cast<uint64_t>(p.m_p) < (1ull << 32))) {
      atomicAnd(&fast_all, 0);
    }
    *reinterpret_cast<IntParams*>(ws + kHeadPrmOffset + kHeadPrmStride * h) = p;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    IntParams hdr;
    memset(&hdr, 0, sizeof(hdr));
    hdr.status = status;
    hdr.q_shift = fast_all ? 0 : 1;
    hdr.s_inv = 1;
    hdr.m_p = 1;
    hdr.one = 1;
    *reinterpret_cast<IntParams*>(ws) = hdr;
  }
}

__global__ void __launch_bounds__(kQThreads)
    dequantize_per_head_kernel(const int8_t* __restrict__ xq, const float* __restrict__ scales,
                               int64_t vec_per_problem, int H, uint32_t h_magic, float* __restrict__ y) {
  const int p = blockIdx.x;
  const float s = scales[head_of(p, H, h_magic)];
  const uint32_t* src = reinterpret_cast<const uint32_t*>(xq) + static_cast<int64_t>(p) * vec_per_problem;
  float4* dst = reinterpret_cast<float4*>(y) + static_cast<int64_t>(p) * vec_per_problem;
  const int64_t v0 = static_cast<int64_t>(blockIdx.y) * kQThreads * kPHVec + threadIdx.x;
#pragma unroll
  for (int u = 0; u < kPHVec; ++u) {
    const int64_t i = v0 + u * kQThreads;
    if (i < vec_per_problem) {
      const uint32_t w = __ldg(src + i);
      dst[i] = make_float4(__fmul_rn(s, static_cast<float>(static_cast<int8_t>(w & 0xFF))),
                           __fmul_rn(s, static_cast<float>(static_cast<int8_t>((w >> 8) & 0xFF))),
                           __fmul_rn(s, static_cast<float>(static_cast<int8_t>((w >> 16) & 0xFF))),
                           __fmul_rn(s, static_cast<float>(static_cast<int8_t>(w >> 24))));
    }
  }
}

cudaError_t launch_quantize_per_head(const QuantTensors& t, int ntensors, int64_t P,
                                     int64_t vec_per_problem, int H, cudaStream_t stream) {
  const uint32_t hm = static_cast<uint32_t>(((1ull << 32) + H - 1) / H);
  for (int i = 0; i < ntensors; ++i) {
    cudaError_t e = cudaMemsetAsync(t.scale[i], 0, sizeof(float) * H, stream);
    if (e != cudaSuccess) return e;
  }
  dim3 grid(static_cast<unsigned>(P),
            static_cast<unsigned>((vec_per_problem + kQThreads * kPHVec - 1) / (kQThreads * kPHVec)),
            ntensors);
  amax_per_head_kernel<<<grid, kQThreads, 0, stream>>>(t, vec_per_problem, H, hm);
  quantize_per_head_kernel<<<grid, kQThreads, 0, stream>>>(t, vec_per_problem, H, hm);
  return cudaGetLastError();
}

cudaError_t launch_derive_per_head(const float* scales, int H, int32_t d, void* ws, cudaStream_t stream) {
  derive_per_head_kernel<<<1, 128, 0, stream>>>(scales, H, d, static_cast<char*>(ws));
  return cudaGetLastError();
}

cudaError_t launch_dequantize_per_head(const int8_t* xq, const float* scales, int64_t P,
                                       int64_t vec_per_problem, int H, float* y, cudaStream_t stream) {
  const uint32_t hm = static_cast<uint32_t>(((1ull << 32) + H - 1) / H);
  dim3 grid(static_cast<unsigned>(P),
            static_cast<unsigned>((vec_per_problem + kQThreads * kPHVec - 1) / (kQThreads * kPHVec)));
  dequantize_per_head_kernel<<<grid, kQThreads, 0, stream>>>(xq, scales, vec_per_problem, H, hm, y);
  return cudaGetLastError();
}

static int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// Launch with programmatic stream serialization (PDL): the kernel may be
// scheduled while its stream predecessor drains and calls griddep_wait()
// before touching global memory.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, int threads,
                              cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Blocks per tensor: enough 256-thread blocks for one pass over the data, capped
// at ~8 resident blocks per SM in total over the `ntensors` tensors.
static int stream_grid(int64_t thread_items, int ntensors) {
  int64_t blocks = (thread_items + kQThreads - 1) / kQThreads;
  const int64_t cap = static_cast<int64_t>(num_sms()) * 8 / ntensors;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return static_cast<int>(blocks);
}

// Single-pass fused launch (three tensors) when every thread's share fits in
// registers (<= 4 vectors per tensor).  Returns cudaErrorNotSupported (nothing
// enqueued) otherwise.
template <typename T, int VPT>
static cudaError_t launch_fused_vpt(const QuantTensors& t, int64_t numel, float* partial,
                                    IntParams* prm_out, int32_t head_dim, int blocks,
                                    cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(blocks));
  cfg.blockDim = dim3(kFThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, quantize_fused_kernel<T, VPT>, t, numel, partial, prm_out, head_dim);
}

template <typename T>
static cudaError_t launch_fused_t(const QuantTensors& t, int ntensors, int64_t numel,
                                  float* partial, IntParams* prm_out, int32_t head_dim,
                                  cudaStream_t stream) {
  if (ntensors != 3) return cudaErrorNotSupported;
  constexpr int kE = 16 / sizeof(T);
  const int64_t nvec = numel / kE;
  // blocks: as few as needed at <= 4 vectors per thread, capped at full occupancy
  const int64_t cap = static_cast<int64_t>(num_sms()) * kFBlocksPerSM;
  int64_t blocks = (nvec + kFThreads - 1) / kFThreads;  // VPT = 1
  int vpt = 1;
  while (blocks > cap && vpt < 4) {
    ++vpt;
    blocks = (nvec + static_cast<int64_t>(kFThreads) * vpt - 1) / (static_cast<int64_t>(kFThreads) * vpt);
  }
  if (blocks > cap) return cudaErrorNotSupported;
  if (blocks < 1) blocks = 1;
  if (blocks > kWsMaxPartialCtas) return cudaErrorNotSupported;  // partials end before the table
  switch (vpt) {
    case 1: return launch_fused_vpt<T, 1>(t, numel, partial, prm_out, head_dim, static_cast<int>(blocks), stream);
    case 2: return launch_fused_vpt<T, 2>(t, numel, partial, prm_out, head_dim, static_cast<int>(blocks), stream);
    case 3: return launch_fused_vpt<T, 3>(t, numel, partial, prm_out, head_dim, static_cast<int>(blocks), stream);
    default: return launch_fused_vpt<T, 4>(t, numel, partial, prm_out, head_dim, static_cast<int>(blocks), stream);
  }
}

// dtype: 0 f32, 1 bf16, 2 f16.  Requires 16-byte aligned x and xq (checked by host).
// `partial` (device, >= 3 * #SMs floats) enables the single-pass fused kernel.
cudaError_t launch_quantize(const QuantTensors& t, int ntensors, int dtype, int64_t numel,
                            IntParams* prm_out, int32_t head_dim, cudaStream_t stream,
                            float* partial) {
  static int fused_mode = -1;  // QFLASH_QUANT_FUSED=0 disables the single-pass kernel
  if (fused_mode < 0) {
    const char* env = getenv("QFLASH_QUANT_FUSED");
    fused_mode = (env != nullptr && env[0] == '0') ? 0 : 1;
  }
  if (fused_mode == 1 && partial != nullptr && numel > 0) {
    cudaError_t e = cudaErrorNotSupported;
    switch (dtype) {
      case 0: e = launch_fused_t<float>(t, ntensors, numel, partial, prm_out, head_dim, stream); break;
      case 1: e = launch_fused_t<__nv_bfloat16>(t, ntensors, numel, partial, prm_out, head_dim, stream); break;
      case 2: e = launch_fused_t<__half>(t, ntensors, numel, partial, prm_out, head_dim, stream); break;
    }
    if (e != cudaErrorNotSupported) return e;
  }
  const bool contiguous = ntensors == 3 && t.scale[1] == t.scale[0] + 1 && t.scale[2] == t.scale[0] + 2;
  if (contiguous) {
    cudaError_t e = cudaMemsetAsync(t.scale[0], 0, 3 * sizeof(float), stream);
    if (e != cudaSuccess) return e;
  } else {
    for (int i = 0; i < ntensors; ++i) {
      cudaError_t e = cudaMemsetAsync(t.scale[i], 0, sizeof(float), stream);
      if (e != cudaSuccess) return e;
    }
  }
  dim3 grid(stream_grid((numel + kQElems - 1) / kQElems, ntensors), ntensors);
  switch (dtype) {
    case 0:
      amax_kernel<float><<<grid, kQThreads, 0, stream>>>(t, numel);
      return launch_pdl((pdl_mask() & 4) != 0, quantize_kernel<float>, grid, kQThreads, stream, t, numel, prm_out, head_dim);
    case 1:
      amax_kernel<__nv_bfloat16><<<grid, kQThreads, 0, stream>>>(t, numel);
      return launch_pdl((pdl_mask() & 4) != 0, quantize_kernel<__nv_bfloat16>, grid, kQThreads, stream, t, numel, prm_out,
                        head_dim);
    case 2:
      amax_kernel<__half><<<grid, kQThreads, 0, stream>>>(t, numel);
      return launch_pdl((pdl_mask() & 4) != 0, quantize_kernel<__half>, grid, kQThreads, stream, t, numel, prm_out, head_dim);
    default:
      return cudaErrorInvalidValue;
  }
}

// amax of three fp32 tensors (blockIdx.y = tensor) -> amax[t] (zeroed by the host
// first): block max, then an unsigned atomicMax on the bits (non-negative floats
// order like their bit patterns).  Used by sharded quantization:
// local amax -> MAX all-reduce -> qflash_forward_fused_amax.
__global__ void __launch_bounds__(kQThreads) amax3_kernel(const float* __restrict__ q,
                                                         const float* __restrict__ k,
                                                         const float* __restrict__ v, int64_t numel,
                                                         unsigned int* amax) {
  const float* x = blockIdx.y == 0 ? q : (blockIdx.y == 1 ? k : v);
  const int64_t nv = numel >> 2;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  float m0 = 0.f, m1 = 0.f;
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + stride < nv; i += 2 * stride) {
    const float4 a = __ldg(x4 + i), b = __ldg(x4 + i + stride);
    m0 = fmaxf(m0, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))));
    m1 = fmaxf(m1, fmaxf(fmaxf(fabsf(b.x), fabsf(b.y)), fmaxf(fabsf(b.z), fabsf(b.w))));
  }
  if (i < nv) {
    const float4 a = __ldg(x4 + i);
    m0 = fmaxf(m0, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))));
  }
  for (int64_t j = nv * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < numel; j += stride)
    m0 = fmaxf(m0, fabsf(x[j]));
  float mm = fmaxf(m0, m1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o));
  __shared__ float red[kQThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mm;
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = red[0];
#pragma unroll
    for (int w = 1; w < kQThreads / 32; ++w) b = fmaxf(b, red[w]);
    atomicMax(amax + blockIdx.y, __float_as_uint(b));
  }
}

cudaError_t launch_amax3(const float* q, const float* k, const float* v, int64_t numel, float* amax,
                         cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(amax, 0, 3 * sizeof(float), stream);
  if (e != cudaSuccess || numel == 0) return e;
  dim3 grid(stream_grid((numel + 7) / 8, 3), 3);
  amax3_kernel<<<grid, kQThreads, 0, stream>>>(q, k, v, numel, reinterpret_cast<unsigned int*>(amax));
  return cudaGetLastError();
}

cudaError_t launch_dequantize(const int8_t* xq, float scale, const float* scale_dev, int64_t numel,
                              float* y, cudaStream_t stream) {
  dim3 grid(stream_grid((numel + 15) / 16, 1));
  return launch_pdl((pdl_mask() & 2) != 0, dequantize_kernel, grid, kQThreads, stream, xq, scale, scale_dev, numel, y);
}

}  // namespace qf
