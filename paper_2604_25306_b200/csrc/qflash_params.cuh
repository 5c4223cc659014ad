// qflash_params.cuh -- derivation of the integer constants of one attention call
// from the per-tensor scales (Alg. 1 Require P:L151, Alg. 2, Eq. 9-10)
// plus the division-free realisation constants the kernel uses.  Compiled for
// the host (qflash_derive_params / the host-scale path) and the device (the
// dscale path and the fused quantize kernel) from this one source.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../include/qflash.h"
#include "qflash_common.cuh"

namespace qf {
// ------------------------------------------------------------------------
// Constant derivation, shared by the host path and the one-thread device
// kernel.  fp64 operations are written with explicit round-to-nearest
// intrinsics on the device (no FMA contraction) and plain operators on the
// host (compiled with -ffp-contract=off), so both evaluate the identical IEEE
// expression ((s_q * s_k) * log2e) / sqrt(d) of Alg. 1.
__host__ __device__ inline double dmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
__host__ __device__ inline double ddiv(double a, double b) {
#ifdef __CUDA_ARCH__
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}
__host__ __device__ inline double dsqrt(double a) {
#ifdef __CUDA_ARCH__
  return __dsqrt_rn(a);
#else
  return std::sqrt(a);
#endif
}

using u128 = unsigned __int128;

// floor(N / D) and N mod D for 1 <= D < 2^26, N < 2^58, quotient < 2^33: an fp64
// estimate (relative error < 2^-51, so within 1 of the quotient) corrected by the
// exact 64-bit remainder.  Replaces the ~100-instruction software u64 division
// on the device's constant-derivation critical path; checked against '/' for
// every D of the domain by tools/udiv_check.cpp.
__host__ __device__ inline uint64_t udiv_small(uint64_t N, uint64_t D, uint64_t* rem) {
#ifdef __CUDA_ARCH__
  const double est = __dmul_rz(__ull2double_rn(N), __drcp_rn(__ull2double_rn(D)));
#else
  const double est = static_cast<double>(N) * (1.0 / static_cast<double>(D));
#endif
  uint64_t q = static_cast<uint64_t>(est);
  int64_t r = static_cast<int64_t>(N - q * D);
  if (r < 0) {
    --q;
    r += static_cast<int64_t>(D);
  } else if (r >= static_cast<int64_t>(D)) {
    ++q;
    r -= static_cast<int64_t>(D);
  }
  *rem = static_cast<uint64_t>(r);
  return q;
}

// smallest L with 2^L >= x (x >= 1)
__host__ __device__ inline int ceil_log2(uint64_t x) {
#ifdef __CUDA_ARCH__
  return x <= 1 ? 0 : 64 - __clzll(x - 1);
#else
  int L = 0;
  while ((uint64_t(1) << L) < x) ++L;
  return L;
#endif
}
// sqrt(d) of Alg. 1's s = s_q s_k log2(e) / sqrt(d): the device uses the
// correctly rounded fp64 constants for the supported d (identical to IEEE sqrt).
__host__ __device__ inline double sqrt_head_dim(int32_t d) {
#ifdef __CUDA_ARCH__
  if (d == 32) return 5.65685424949238058190;   // RN(sqrt(32)) = 0x4016A09E667F3BCD
  if (d == 64) return 8.0;
  if (d == 128) return 11.3137084989847611638;  // RN(sqrt(128)) = 0x4026A09E667F3BCD
  return dsqrt(static_cast<double>(d));
#else
  return std::sqrt(static_cast<double>(d));
#endif
}

__host__ __device__ inline int derive_core(float s_q, float s_k, int32_t d, qf::IntParams* o,
                                           qflash_int_params* pub) {
  if (!(s_q > 0.0f) || !(s_k > 0.0f) || !isfinite(s_q) || !isfinite(s_k))
    return QFLASH_ERR_SCALE_RANGE;
  const double log2e = 1.4426950408889634;
  const double x = dmul(dmul(static_cast<double>(s_q), static_cast<double>(s_k)), log2e);
  // x / 8 is the exact scaling x * 2^-3 (x is a normal fp64 number)
  const double s = d == 64 ? dmul(x, 0.125) : ddiv(x, sqrt_head_dim(d));
  if (!(s >= ldexp(1.0, -24)) || !(s <= 0.5)) return QFLASH_ERR_SCALE_RANGE;
#ifdef __CUDA_ARCH__
  const int64_t s_inv = llround(__drcp_rn(s));   // RN(1/s), round half away (R1)
#else
  const int64_t s_inv = llround(ddiv(1.0, s));  // round half away (R1)
#endif
  const double ratio = dmul(s, 127.0);          // s / s_P, s_P = 1/127 (R8)
  int e = 0;
  (void)frexp(ratio, &e);
  const int32_t n = e - 1;                      // floor(log2 ratio)   (Eq. 9)
  const int32_t r_p = 8 - n;                    // r = b - n           (Eq. 9)
  const int64_t m_p = llround(ldexp(ratio, r_p));  // round(ratio 2^r) (Eq. 10)

  const uint64_t D = static_cast<uint64_t>(s_inv);
  // q1 = floor(t / s_inv) for t < 2^25 (t = m - S + s_inv, the kernel's range).
  uint32_t q_magic;
  int32_t q_shift;
  {
    uint64_t r0;
    const uint64_t m0 = udiv_small(uint64_t(1) << 32, D, &r0);
    const uint64_t m = m0 + (r0 != 0 ? 1 : 0);  // ceil(2^32 / D)
    const uint64_t err = m * D - (uint64_t(1) << 32);
    // fast form: exact for t < 27 s_inv (q1 <= 26); beyond, the estimate is
    // >= the true quotient (>= 26) and the shifted value is < 2^26, so y = 0
    // exactly as in the oracle.
    if (D <= (uint64_t(1) << 22) && (27 * D) * err < (uint64_t(1) << 32)) {
      q_magic = static_cast<uint32_t>(m);
      q_shift = 0;
    } else {
      const int L = ceil_log2(D);
      const int sh = L > 7 ? L - 7 : 0;           // L <= 25: 2^(32 + sh) < 2^51
      uint64_t rr;
      const uint64_t mm0 = udiv_small(uint64_t(1) << (32 + sh), D, &rr);
      const uint64_t mm = mm0 + (rr != 0 ? 1 : 0);
      q_magic = static_cast<uint32_t>(mm);
      q_shift = sh;
    }
  }
  // P = floor(y M_P / 2^r_P) = umulhi(y << p_pre, p_mul)
  const int32_t p_pre = r_p < 10 ? 10 - r_p : 0;
  const uint64_t p_mul = static_cast<uint64_t>(m_p) << (32 - r_p - p_pre);
  const int64_t p_max = (s_inv * m_p) >> r_p;
  // release: floor(n / s_inv) for n < 2^56
  uint64_t rel_magic;
  int32_t rel_shift;
  {
    // ceil(2^(64 + sh) / D) by two 64-bit long-division steps (exact):
    // 2^(32 + sh) = q1 D + r1, then r1 2^32 = q2 D + r2 (r1 < D < 2^25).
    const int L = ceil_log2(D);
    const int sh = L > 8 ? L - 8 : 0;
    const uint64_t A = uint64_t(1) << (32 + sh);
    uint64_t r1, r2;
    const uint64_t q1 = udiv_small(A, D, &r1);
    const uint64_t q2 = udiv_small(r1 << 32, D, &r2);
    rel_magic = (q1 << 32) + q2 + (r2 != 0 ? 1 : 0);
    rel_shift = sh;
  }
  if (o) {
    o->status = 0;
    o->s_inv = static_cast<int32_t>(s_inv);
    o->q_magic = q_magic;
    o->q_shift = q_shift;
    o->p_mul = static_cast<uint32_t>(p_mul);
    o->p_pre = p_pre;
    o->rel_magic_lo = static_cast<uint32_t>(rel_magic);
    o->rel_magic_hi = static_cast<uint32_t>(rel_magic >> 32);
    o->rel_shift = rel_shift;
    o->p_max = static_cast<int32_t>(p_max);
    o->r_p = r_p;
    o->m_p = static_cast<int32_t>(m_p);
    o->n = n;
    o->one = 1;
    o->zero = 0;
    o->pad[0] = 0;
    o->s = s;
  }
  if (pub) {
    pub->s = s;
    pub->s_inv = static_cast<int32_t>(s_inv);
    pub->n = n;
    pub->r_p = r_p;
    pub->m_p = static_cast<int32_t>(m_p);
    pub->q_magic = q_magic;
    pub->q_shift = q_shift;
    pub->p_mul = static_cast<uint32_t>(p_mul);
    pub->p_pre = p_pre;
    pub->p_max = static_cast<int32_t>(p_max);
    pub->rel_magic = rel_magic;
    pub->rel_shift = rel_shift;
  }
  return QFLASH_OK;
}

}  // namespace qf
