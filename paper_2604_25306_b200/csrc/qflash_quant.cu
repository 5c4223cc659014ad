// qflash_quant.cu -- per-tensor int8 quantizer (Eq. 2) and the
// dequantizer, HBM-bound streaming kernels for sm_100a.
//
// Quantization of T tensors (T = 1, or 3 for fused Q/K/V) is two launches:
//   1. amax: every block reduces max|x| (as IEEE bit patterns, so NaN
//      propagates) and atomically maxes s_b = fl32(amax_b / 127) into the
//      caller's scale slot (pre-zeroed).  fl32 division is monotone, so the
//      slot ends at fl32(max_b amax_b / 127) = fl32(amax / 127).
//   2. quantize: x^ = sat8(roundf(__fdiv_rn(x, s))), with s = 1/127 when the
//      slot is 0 (all-zero tensor, reading R3).  Block 0 writes 1/127 back in
//      that case; every block treats 0 and 1/127 identically, so the write is
//      race-free.
// Loads are 16-byte vectors, grid-strided over a grid sized to the SM count.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "qflash_common.cuh"

namespace qf {

constexpr int kQThreads = 256;


template <typename T>
struct Vec;  // 16-byte vector of T widened to fp32
template <>
struct Vec<float> {
  static constexpr int kN = 4;
  __device__ static void load(const void* base, int64_t i, float* out) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(base) + i);
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
  }
  __device__ static float load1(const void* base, int64_t i) {
    return __ldg(reinterpret_cast<const float*>(base) + i);
  }
};
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int kN = 8;
  __device__ static void load(const void* base, int64_t i, float* out) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(base) + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      out[2 * k] = __uint_as_float(w[k] << 16);
      out[2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
    }
  }
  __device__ static float load1(const void* base, int64_t i) {
    const uint16_t b = reinterpret_cast<const uint16_t*>(base)[i];
    return __uint_as_float(static_cast<uint32_t>(b) << 16);
  }
};
template <>
struct Vec<__half> {
  static constexpr int kN = 8;
  __device__ static void load(const void* base, int64_t i, float* out) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(base) + i);
    const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __half22float2(h[k]);  // exact widening
      out[2 * k] = f.x;
      out[2 * k + 1] = f.y;
    }
  }
  __device__ static float load1(const void* base, int64_t i) {
    return __half2float(reinterpret_cast<const __half*>(base)[i]);
  }
};

__device__ __forceinline__ uint32_t abs_bits(float x) { return __float_as_uint(x) & 0x7FFFFFFFu; }

// scale from amax (as stored in the slot): fl32(amax / 127); 0 stays 0 here.
__device__ __forceinline__ float scale_of_amax_bits(uint32_t amax_bits) {
  return __fdiv_rn(__uint_as_float(amax_bits), 127.0f);
}

template <typename T>
__global__ void __launch_bounds__(kQThreads) amax_kernel(QuantTensors t, int64_t numel) {
  const int ti = blockIdx.y;
  const void* x = t.x[ti];
  constexpr int kN = Vec<T>::kN;
  const int64_t nvec = numel / kN;
  uint32_t m = 0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nvec; i += stride) {
    float v[kN];
    Vec<T>::load(x, i, v);
#pragma unroll
    for (int k = 0; k < kN; ++k) m = max(m, abs_bits(v[k]));
  }
  for (int64_t i = nvec * kN + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < numel; i += stride)
    m = max(m, abs_bits(Vec<T>::load1(x, i)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ uint32_t red[kQThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t b = red[0];
    for (int w = 1; w < kQThreads / 32; ++w) b = max(b, red[w]);
    // s_b = fl32(amax_b / 127) is monotone in amax_b; non-negative floats
    // (and NaN, whose bits exceed +inf) order like their bit patterns.
    const float sb = scale_of_amax_bits(b);
    atomicMax(reinterpret_cast<unsigned int*>(t.scale[ti]), __float_as_uint(sb));
  }
}

__device__ __forceinline__ int32_t quant_one(float x, float s) {
  float r = roundf(__fdiv_rn(x, s));  // IEEE division, half away from zero (R1, R2)
  r = fminf(fmaxf(r, -128.0f), 127.0f);
  return static_cast<int32_t>(r);
}

template <typename T>
__global__ void __launch_bounds__(kQThreads) quantize_kernel(QuantTensors t, int64_t numel) {
  const int ti = blockIdx.y;
  const void* x = t.x[ti];
  int8_t* xq = t.xq[ti];
  float s = *reinterpret_cast<volatile float*>(t.scale[ti]);
  if (s == 0.0f) s = 1.0f / 127.0f;  // all-zero tensor (R3)
  if (blockIdx.x == 0 && threadIdx.x == 0) *t.scale[ti] = s;
  constexpr int kN = Vec<T>::kN;
  const int64_t nvec = numel / kN;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nvec; i += stride) {
    float v[kN];
    Vec<T>::load(x, i, v);
    uint32_t w[kN / 4];
#pragma unroll
    for (int k = 0; k < kN / 4; ++k) {
      const int32_t a = quant_one(v[4 * k], s), b = quant_one(v[4 * k + 1], s);
      const int32_t c = quant_one(v[4 * k + 2], s), d = quant_one(v[4 * k + 3], s);
      w[k] = (static_cast<uint32_t>(a) & 0xFFu) | ((static_cast<uint32_t>(b) & 0xFFu) << 8) |
             ((static_cast<uint32_t>(c) & 0xFFu) << 16) | (static_cast<uint32_t>(d) << 24);
    }
    if constexpr (kN == 4)
      reinterpret_cast<uint32_t*>(xq)[i] = w[0];
    else
      reinterpret_cast<uint2*>(xq)[i] = make_uint2(w[0], w[1]);
  }
  for (int64_t i = nvec * kN + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < numel; i += stride)
    xq[i] = static_cast<int8_t>(quant_one(Vec<T>::load1(x, i), s));
}

__global__ void __launch_bounds__(kQThreads)
    dequantize_kernel(const int8_t* __restrict__ xq, float scale, const float* __restrict__ scale_dev,
                      int64_t numel, float* __restrict__ y) {
  const float s = scale_dev ? *scale_dev : scale;
  const int64_t nvec = numel / 16;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nvec; i += stride) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(xq) + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    float4* dst = reinterpret_cast<float4*>(y) + 4 * i;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int32_t b0 = static_cast<int8_t>(w[k] & 0xFF), b1 = static_cast<int8_t>((w[k] >> 8) & 0xFF);
      const int32_t b2 = static_cast<int8_t>((w[k] >> 16) & 0xFF), b3 = static_cast<int8_t>(w[k] >> 24);
      dst[k] = make_float4(__fmul_rn(s, static_cast<float>(b0)), __fmul_rn(s, static_cast<float>(b1)),
                           __fmul_rn(s, static_cast<float>(b2)), __fmul_rn(s, static_cast<float>(b3)));
    }
  }
  for (int64_t i = nvec * 16 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < numel; i += stride)
    y[i] = __fmul_rn(s, static_cast<float>(xq[i]));
}

static int stream_grid(int64_t work_items) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  int64_t blocks = (work_items + kQThreads - 1) / kQThreads;
  const int64_t cap = static_cast<int64_t>(sms) * 8;  // 8 x 256 threads per SM
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return static_cast<int>(blocks);
}

// dtype: 0 f32, 1 bf16, 2 f16.  Requires 16-byte aligned x and xq (checked by host).
cudaError_t launch_quantize(const QuantTensors& t, int ntensors, int dtype, int64_t numel,
                            cudaStream_t stream) {
  for (int i = 0; i < ntensors; ++i) {
    cudaError_t e = cudaMemsetAsync(t.scale[i], 0, sizeof(float), stream);
    if (e != cudaSuccess) return e;
  }
  const int vec = (dtype == 0) ? 4 : 8;
  dim3 grid(stream_grid((numel + vec - 1) / vec), ntensors);
  switch (dtype) {
    case 0:
      amax_kernel<float><<<grid, kQThreads, 0, stream>>>(t, numel);
      quantize_kernel<float><<<grid, kQThreads, 0, stream>>>(t, numel);
      break;
    case 1:
      amax_kernel<__nv_bfloat16><<<grid, kQThreads, 0, stream>>>(t, numel);
      quantize_kernel<__nv_bfloat16><<<grid, kQThreads, 0, stream>>>(t, numel);
      break;
    case 2:
      amax_kernel<__half><<<grid, kQThreads, 0, stream>>>(t, numel);
      quantize_kernel<__half><<<grid, kQThreads, 0, stream>>>(t, numel);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_dequantize(const int8_t* xq, float scale, const float* scale_dev, int64_t numel,
                              float* y, cudaStream_t stream) {
  dim3 grid(stream_grid((numel + 15) / 16));
  dequantize_kernel<<<grid, kQThreads, 0, stream>>>(xq, scale, scale_dev, numel, y);
  return cudaGetLastError();
}

}  // namespace qf
