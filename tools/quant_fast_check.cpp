// quant_fast_check.cpp -- host check of the kernel's fast element quantizer
// (paper_2604_25306_b200/csrc/qflash_quant_elem.cuh, compiled here for the host with
// the CUDA rounding intrinsics mapped to their IEEE host equivalents: fmaf is the
// correctly rounded fused multiply-add, like __fmaf_rn).  Claim checked: whenever
// quant_fast does not flag `bad`, sat8(its result) == sat8(roundf(fl32(x / s))), the
// exact definition of Eq. 2 (readings R1, R2); the flagged cases take quant_exact.
// Inputs: for 400 scales s = fl32(amax / 127), every float with |x| <= amax within
// +-48 ulps of each half-integer boundary (k + 1/2) s, k = -130..129, plus random x.
//   g++ -O2 -std=c++17 -ffp-contract=off tools/quant_fast_check.cpp -o /tmp/qfc && /tmp/qfc
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>

#define __device__
#define __forceinline__ inline
static inline float __fmaf_rn(float a, float b, float c) { return std::fmaf(a, b, c); }
static inline float __fadd_rn(float a, float b) { return a + b; }
static inline float __fdiv_rn(float a, float b) { return a / b; }
static inline uint32_t __float_as_uint(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}
struct uint4 {
  uint32_t x, y, z, w;
};
static inline uint4 make_uint4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) { return {a, b, c, d}; }
static inline unsigned __activemask() { return 1u; }
static inline bool __any_sync(unsigned, bool b) { return b; }
#include "../paper_2604_25306_b200/csrc/qflash_quant_elem.cuh"

static inline int sat8(int v) { return v > 127 ? 127 : (v < -128 ? -128 : v); }

int main() {
  std::mt19937_64 rng(2604);
  std::uniform_real_distribution<double> ue(-9.0, 2.0);  // amax in [2^-9 ... 2^2] x 127
  long long checked = 0, flagged = 0, wrong = 0;
  for (int si = 0; si < 412; ++si) {
    // amax = 127 2^-k every fourth scale: s is a power of two, so exact ties occur;
    // the last 12 scales are subnormal (amax ~ 1e-38 .. 1e-43: r = 1/s overflows to
    // +Inf below s = 2^-128, where every element must be flagged for the exact path)
    const float amax = si >= 400 ? std::ldexp(1.7f, -126 - 2 * (si - 400))
                       : si % 4 == 0 ? std::ldexp(127.0f, -(si % 20))
                                     : static_cast<float>(std::exp2(ue(rng)) * 127.0);
    const float s = amax / 127.0f;  // fl32(amax / 127), as the quantize kernels compute it
    const float r = 1.0f / s;                           // __frcp_rn
    auto check = [&](float x) {
      if (!(std::fabs(x) <= amax)) return;  // the callers' domain: |x| <= amax
      bool bad = false;
      const int v = qf::quant_fast(x, r, bad);
      ++checked;
      if (std::isinf(r) && !bad) {
        if (wrong < 10) printf("r = inf not flagged: s=%a x=%a\n", s, x);
        ++wrong;
        return;
      }
      if (bad) {
        ++flagged;
        return;
      }
      const int ref = sat8(static_cast<int>(std::roundf(x / s)));
      if (sat8(v) != ref) {
        if (wrong < 10) printf("mismatch s=%a x=%a fast=%d exact=%d\n", s, x, v, ref);
        ++wrong;
      }
    };
    for (int k = -130; k <= 129; ++k) {
      float b = static_cast<float>((k + 0.5) * static_cast<double>(s));
      for (int u = 0; u < 48; ++u) b = std::nextafterf(b, -INFINITY);
      for (int u = 0; u < 97; ++u, b = std::nextafterf(b, INFINITY)) check(b);
    }
    std::uniform_real_distribution<float> ux(-1.1f * amax, 1.1f * amax);
    for (int i = 0; i < 20000; ++i) check(ux(rng));
    check(0.0f);
    check(-0.0f);
    check(amax);
    check(-amax);
  }
  printf("quant_fast: %lld inputs, %lld flagged for the exact path, %lld mismatches\n", checked,
         flagged, wrong);
  return wrong != 0;
}
