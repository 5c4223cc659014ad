// qflash_quant_elem.cuh -- the per-element exact quantizer of Eq. 2 (readings R1,
// R2): x^ = sat8(roundf(fl32(x / s))), shared by the quantize kernels
// (qflash_quant.cu) and the fused-step prologue of the attention kernel.
#pragma once
#include <cstdint>

namespace qf {

// roundf(fl32(x / s)) exactly (see the header comment).  Fast path on the exact
// product x r (r = RN(1/s), so x r = (x / s)(1 + d), |d| <= 2^-24): t = RN(x r +
// 1.5*2^23) is rint(x r) + 1.5*2^23 for |x r| < 2^22 (no FRND/F2I); the FFMA
// x r - rint(x r) flags `bad` when x r is within 2^-14 of a half-integer, where
// x / s and fl32(x / s) could round differently (|x r - x / s| < 2^-16 for
// |x / s| < 2^8; beyond 2^8 every value saturates to +-127 / -128 anyway).  Domain:
// |x / s| < 2^22, which every caller guarantees (s = fl32(amax / 127) of the same
// values, so |x / s| <= 127 (1 + 2^-22)); a non-finite r (subnormal s) always takes
// the exact path.  FFMA + FADD + FFMA + FSETP + IADD.
__device__ __forceinline__ int32_t quant_fast(float x, float r, bool& bad) {
  const float t = __fmaf_rn(x, r, 12582912.0f);                 // 1.5 * 2^23
  const float fi = __fadd_rn(t, -12582912.0f);                  // rint(x r), exact
  // written as !(|.| < c) so that a NaN residual also takes the exact path: r = +Inf
  // when s < 2^-128 (a subnormal scale), where x r is NaN / Inf
  bad |= !(fabsf(__fmaf_rn(x, r, -fi)) < 0.49993896484375f);   // 0.5 - 2^-14
  return static_cast<int32_t>(__float_as_uint(t) - 0x4B400000u);  // int(rint(x r))
}
// the exact definition: IEEE division then round half away from zero (R1, R2)
__device__ __forceinline__ int32_t quant_exact(float x, float s) {
  return static_cast<int32_t>(roundf(__fdiv_rn(x, s)));
}
__device__ __forceinline__ int32_t quant_one(float x, float s, float r) {
  bool bad = false;
  const int32_t v = quant_fast(x, r, bad);
  return bad ? quant_exact(x, s) : v;
}
// 16 elements -> 16 int8 (uint4), one warp-voted exact pass if any lane needs it.
__device__ __forceinline__ uint4 quant16(const float* f, float s, float r) {
  int32_t v[16];
  bool bad = false;
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = quant_fast(f[k], r, bad);
  if (__any_sync(__activemask(), bad)) {
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = quant_exact(f[k], s);
  }
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t hi, lo;
    asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(v[4 * k + 3]), "r"(v[4 * k + 2]));
    asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(lo) : "r"(v[4 * k + 1]), "r"(v[4 * k]), "r"(hi));
    w[k] = lo;
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

}  // namespace qf
