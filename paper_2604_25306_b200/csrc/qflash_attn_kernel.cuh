// qflash_attn_kernel.cuh -- the fused integer-only attention kernel (Algorithm 1
// of arxiv 2604.25306) for B200 / sm_100a, as a template included by
// the instantiation units (qflash_attention.cu, qflash_attention_dbg.cu).
//
// A CTA (one per SM, persistent) runs QT independent "groups"; each group walks
// its own sequence of 128-row query tiles (B_r = 128 = the tcgen05 M; TMEM lane
// r = tile row r) with its own TMA producer warp, MMA issuer warp, shared-memory
// ring, TMEM region and mbarriers.  Two groups (QT = 2) ping-pong: while one
// group's softmax warps wait for its P V / Q K^T round trip on the tensor core,
// the other group's warps compute, so the integer ALUs stay busy.
//
// Warps 0..3 are control warps: warp g (< QT) is group g's TMA producer, warp
// 2 + g (< 2 + QT) its MMA issuer; warp 2 also allocates TMEM and warp 3 loads
// the reciprocal table of step (11) before taking their roles.  Then QT x CS
// softmax warpgroups: group g's CS warpgroups split every KV tile's B_c key
// columns (B_c / CS per thread) and the d output columns; thread = (query row,
// column slice).  Per KV tile j a softmax thread
//   (2)(3) loads its S columns from TMEM (tcgen05.ld 32x32b), takes their row max
//          (VIMNMX3) and combines it with the group's other warpgroups through
//          shared memory (one named barrier per group);
//   (4)    alpha = ShiftExp2(m_old - m_new);
//   (5)(6) P = Requant(ShiftExp2(S - m_new)), packed 4 x int8 per TMEM column
//          (cvt.pack.sat) and stored over the consumed S columns;
//   (7)(8) ScaleRelease of its O columns and l once P V_{j-1} has landed;
//   then arrives on the group's p_full barrier, which releases the MMA warp to
//   issue O += P [V_j | 1] (the ones block makes TMEM column d the row sum l).
// After the last KV tile: (11) O = floor(O / l), saturated, 16-byte row stores.
//
// Tiling (NSEG):
//   NSEG = 1  "generic": tile = (problem, 128-row query block).
//   NSEG > 1  "row-packed": query rows of all problems are flattened and cut into
//             128-row tiles spanning up to NSEG problems (segments).  Segment s
//             gets its own Q tile, loaded by TMA with row coordinates shifted by
//             -s N so rows of other problems fall out of range and are zero-filled;
//             S = sum_s Q_s K_{s,j}^T then holds every row's scores against its
//             own problem's keys.  P is stored once per segment (own segment: the
//             row's P, others: zeros) and O = sum_s P_s [V_{s,j} | 1].
//
// The production instantiations (DBG = false) execute no floating-point
// instruction (tests/test_abi_cpu.py audits the SASS).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include <cooperative_groups.h>

#include "ptx.cuh"
#include "qflash_common.cuh"
#include "qflash_params.cuh"
#include "qflash_quant_elem.cuh"

namespace qf {

// ----------------------------------------------------------------------------
// Reciprocal table for step (11): kRecip[i] = floor(2^62 / (2^31 + (2i+1) 2^20)),
// the reciprocal of the midpoint of the i-th of 1024 buckets of a normalised
// l in [2^31, 2^32).  Built at compile time (no runtime division anywhere).
struct RecipTable {
  uint32_t v[1024];
};
constexpr RecipTable make_recip_table() {
  RecipTable t{};
  for (int i = 0; i < 1024; ++i) {
    const unsigned long long den = (1ull << 31) + ((2ull * i + 1ull) << 20);
    t.v[i] = static_cast<uint32_t>((1ull << 62) / den);
  }
  return t;
}
static __device__ const RecipTable g_recip = make_recip_table();

constexpr int kMaxStages = 3;  // K/V ring stages reserved in the barrier layout
#ifndef QF_KV_STAGES_C1
#define QF_KV_STAGES_C1 2  // K/V ring depth of configuration 1 (3 measured: no gain, r2_experiments.md)
#endif
constexpr int kBlockR = 128;

// Sleep (ns) between barrier probes of the waits off the critical path
// (experiment builds override with -D).
#ifndef QF_KVR
#define QF_KVR 4
#endif
#ifndef QF_SLEEP_CORR
#define QF_SLEEP_CORR 0  // > 0: correction warps poll with test_wait + nanosleep(ns)
#endif
#ifndef QF_SLEEP_PROD
#define QF_SLEEP_PROD 0  // > 0: producers poll with test_wait + nanosleep(ns) instead of a suspended try_wait
#endif
#ifndef QF_PRE_PROXY_FENCE
#define QF_PRE_PROXY_FENCE 1  // fused prologue: writer-side proxy fence before the second barrier
#endif
#ifndef QF_NO_CODE_STORE
#define QF_NO_CODE_STORE 0  // timing experiment only: quantize without storing the codes (wrong output)
#endif
#ifndef QF_EVICT_FIRST
#define QF_EVICT_FIRST 0  // 1: L2 evict-first policy on the fused step's fp32 input loads / output stores
#endif
#ifndef QF_SLEEP_SOFT
#define QF_SLEEP_SOFT 0
#endif

// TMA producer waits on consumer-release barriers.  nanosleep-polling measured ~65 K
// loop iterations per producer warp over an L14 launch (the sleep returns almost at
// once), i.e. ~8 % of the kernel's issued instructions on SMSPs 0 / 1; the suspended
// try_wait parks the warp until the phase flips.
QF_DEV void prod_wait(uint64_t* bar, uint32_t parity) {
  if (QF_SLEEP_PROD > 0) mbar_wait_sleep(bar, parity, QF_SLEEP_PROD);
  else mbar_wait(bar, parity);
}

QF_DEV void corr_wait(uint64_t* bar, uint32_t parity) {
  if (QF_SLEEP_CORR > 0) mbar_wait_sleep(bar, parity, QF_SLEEP_CORR);
  else mbar_wait(bar, parity);
}

__host__ __device__ constexpr uint32_t tmem_cols_pow2(int cols) {
  return cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
}
template <int D>
__host__ __device__ constexpr uint32_t swizzle_layout() {
  return D == 32 ? 6u : D == 64 ? 4u : 2u;  // UMMA layout: SW32 / SW64 / SW128
}

// ---------------------------------------------------------------- configuration
template <int D, int BC, int NSEG, int CS, int QT>
struct Cfg {
  // CS = 1 ("row owner"): per group one softmax warpgroup (thread = row, all B_c
  // columns) plus one correction warpgroup (ScaleRelease of O and l, step 11).
  static constexpr bool kRC = CS == 1;
  static constexpr int kNWG = kRC ? 2 * QT : CS * QT;  // softmax (+ correction) warpgroups
  static constexpr int kCtl = 4;                  // control warps
  static constexpr int kThreads = 32 * kCtl + 128 * kNWG;
  static constexpr int kGroupThreads = 128 * CS;  // softmax threads of one group
  static constexpr int kCW = BC / CS;             // key columns per thread
  static constexpr int kOW = D / CS;              // O columns per thread
  // TMEM per group: kNumS S buffers of BC columns (P_s of KV tile j aliases S
  // buffer j: segment s at columns [s BC/4, (s+1) BC/4)), then O (D columns),
  // l (column D) and 15 copies of l from the ones block.
  static constexpr int kNumS = (QT == 1 && 2 * BC + D + 16 <= 512) ? 2 : 1;
  // Separate P region (CS = 2, QT = 2, generic tiles, when TMEM allows): P lives
  // in its own B_c/4 columns instead of aliasing S, so the next Q K^T may overwrite
  // S as soon as the softmax warps have read it (s_empty), overlapping the round
  // trip with the P arithmetic and the release instead of following P V.
  static constexpr bool kSepP =
      CS == 2 && QT == 2 && NSEG == 1 && QT * (BC + BC / 4 + D + 16) <= 512;
  static constexpr int kPCol = kNumS * BC;                         // P region (kSepP)
  static constexpr int kOCol = kNumS * BC + (kSepP ? BC / 4 : 0);  // O (+ l, ones copies)
  static constexpr int kGroupCols = kOCol + D + 16;
  static constexpr uint32_t kTmemCols = tmem_cols_pow2(QT * kGroupCols);
  // shared memory (offsets from the 1024-aligned base)
  static constexpr int kQBytes = kBlockR * D;
  static constexpr int kKVBytes = BC * D;
  // K/V ring depth: 3 for configuration 1 with generic tiles (the load of K/V tile j + 2
  // starts once P V_{j-1} has released its stage, a round earlier than with 2), else 2
  static constexpr int kSt = (QT == 2 && CS == 2 && NSEG == 1) ? QF_KV_STAGES_C1 : 2;
  static constexpr int kGroupSmem = 2 * NSEG * kQBytes + 2 * kSt * NSEG * kKVBytes;
  static constexpr int kQ = 0;                               // [2][NSEG] (+ g kGroupSmem)
  static constexpr int kK = 2 * NSEG * kQBytes;              // [kSt][NSEG]
  static constexpr int kV = kK + kSt * NSEG * kKVBytes;      // [kSt][NSEG]
  static constexpr int kOnes = QT * kGroupSmem;              // second MN atom of [V | 1]
  static constexpr int kBarsPerGroup = 2 * kMaxStages + 4 + kNumS + 7;
  static constexpr int kBar = kOnes + BC * D;
  static constexpr int kTmemSlot = kBar + QT * kBarsPerGroup * 8;
  static constexpr int kRed = (kTmemSlot + 16 + 15) / 16 * 16;  // [QT][2][CS][128] int32
  static constexpr int kRecip = kRed + QT * 2 * CS * 128 * 4;   // [1024] u32 + [256] dequant
  static constexpr int kPrm = kRecip + 1280 * 4;                // IntParams (fused step)
  static constexpr int kScratch = kPrm + 128;                    // [3][32] f32 + [3] scales
  static constexpr int kTotal = kScratch + 512;
  static constexpr int kAlloc = kTotal + 1024;                  // slack for 1024-B alignment
  static_assert(QT * kGroupCols <= 512, "TMEM budget");
  static_assert(NSEG * (BC / 4) <= BC, "P segments must fit in one S buffer");
  static_assert(kCW == 16 || kCW == 32 || kCW == 64 || (kRC && kCW == 128), "columns per thread");
  static_assert(kOW % 8 == 0, "O columns per thread");
};

template <int D, int BC, int NSEG, int CS, int QT>
constexpr bool config_fits() {
  return (QT * (((QT == 1 && 2 * BC + D + 16 <= 512) ? 2 : 1) * BC + D + 16) <= 512) &&
         (BC / CS == 16 || BC / CS == 32 || BC / CS == 64 || (CS == 1 && BC == 128)) &&
         ((D / CS) % 8 == 0) &&
         (NSEG * (BC / 4) <= BC) &&
         (QT * (2 * NSEG * kBlockR * D + 2 * ((QT == 2 && CS == 2 && NSEG == 1) ? QF_KV_STAGES_C1 : 2) * NSEG * BC * D) +
              BC * D + 8 * QT * (2 * kMaxStages + 4 + 2 + 7) +
              QT * 2 * CS * 512 + 5120 + 640 + 2048 <=
          227 * 1024);
}

// Group barriers (8 B each): kv_full[kMaxStages], kv_empty[kMaxStages], q_full[2],
// q_empty[2], s_full[kNumS], p_full, o_full.
template <int NUMS>
struct GroupBars {
  uint64_t* base;
  QF_DEV uint64_t* kv_full(int s) const { return base + s; }
  QF_DEV uint64_t* kv_empty(int s) const { return base + kMaxStages + s; }
  QF_DEV uint64_t* q_full(int b) const { return base + 2 * kMaxStages + b; }
  QF_DEV uint64_t* q_empty(int b) const { return base + 2 * kMaxStages + 2 + b; }
  QF_DEV uint64_t* s_full(int b) const { return base + 2 * kMaxStages + 4 + b; }
  // p_full(1) and rel_full are used by the row-owner roles (CS = 1) (alpha_full: slot kept
  // for the layout; the alpha hand-off uses named barriers),
  // where the softmax warpgroup may run one KV tile ahead of its consumers: the
  // double-buffered barriers (index it & 1, parity (it >> 1) & 1) never overrun.
  QF_DEV uint64_t* p_full(int b = 0) const { return base + 2 * kMaxStages + 4 + NUMS + b; }
  QF_DEV uint64_t* o_full() const { return base + 2 * kMaxStages + 6 + NUMS; }
  QF_DEV uint64_t* alpha_full(int b) const { return base + 2 * kMaxStages + 7 + NUMS + b; }
  QF_DEV uint64_t* rel_full() const { return base + 2 * kMaxStages + 9 + NUMS; }
  QF_DEV uint64_t* s_empty() const { return base + 2 * kMaxStages + 10 + NUMS; }  // kSepP
};


// TMEM column (within an S buffer) of the packed P of warpgroup c, segment s:
// CW >= 32 "own range" (inside the warpgroup's own S columns), CW = 16 contiguous.
template <int BC, int CW>
__host__ __device__ constexpr int p_col(int c, int s) {
  return CW >= 32 ? c * CW + s * (CW / 4) : s * (BC / 4) + c * (CW / 4);
}
// ... and of the 8 columns (32 keys) consumed by K-step kk of the P V MMA.
template <int BC, int CW>
__host__ __device__ constexpr int p_col_k(int kk, int s) {
  return CW >= 32 ? p_col<BC, CW>((32 * kk) / CW, s) + (((32 * kk) % CW) / 32) * 8
                  : s * (BC / 4) + 8 * kk;
}

// ---------------------------------------------------------------- the math

// ShiftExp2 + requantization of one score (steps 5-6 for one element).
//   d1 = m + s_inv - S  (>= s_inv),  q1 = floor(d1 / s_inv) = q + 1  (exact magic)
//   y  = (q1 s_inv + S + s_inv - m) >> q1  ==  ((r >> 1) + s_inv) >> q   (Alg. 2)
//   P  = floor(y M_P / 2^r_P)                                            (Eq. 10)
// Per element: 2 IADD3 + SHF (+ SHF) on the ALU pipe, IMAD.HI + IMAD (+ IMAD) on
// the FMA pipe.  ALT = true computes u = S + (s_inv - m) with IMAD instead of
// IADD3, so alternating the forms balances the two pipes.
template <bool FASTQ, bool ALT>
QF_DEV int32_t shift_exp2_requant(int32_t S, uint32_t m, uint32_t nm, uint32_t c3, uint32_t one,
                                  const IntParams& p) {
  const uint32_t s_inv = static_cast<uint32_t>(p.s_inv);
  const uint32_t d1 = iadd3(m, static_cast<uint32_t>(-S), s_inv);
  uint32_t q1 = umulhi(d1, p.q_magic);
  if constexpr (!FASTQ) q1 >>= p.q_shift;
  uint32_t u;
  if constexpr (ALT) {
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(u) : "r"(static_cast<uint32_t>(S)), "r"(one), "r"(c3));
  } else {
    u = iadd3(static_cast<uint32_t>(S), s_inv, nm);
  }
  const uint32_t num = q1 * s_inv + u;
  uint32_t y = shr_clamp(num, q1);
  if constexpr (FASTQ) {
    // y M_P < 2^32 (host-checked: s_inv M_P < 2^32): IMAD + SHF instead of IMAD.HI
    return static_cast<int32_t>((y * static_cast<uint32_t>(p.m_p)) >> p.r_p);
  } else {
    y <<= p.p_pre;
    return static_cast<int32_t>(umulhi(y, p.p_mul));
  }
}

// alpha = ShiftExp2(m_old - m_new) (step 4) -- same formula, x = m_old - m_new <= 0.
template <bool FASTQ>
QF_DEV int32_t shift_exp2(int32_t x, const IntParams& p) {
  const uint32_t d1 = static_cast<uint32_t>(p.s_inv - x);
  uint32_t q1 = umulhi(d1, p.q_magic);
  if constexpr (!FASTQ) q1 >>= p.q_shift;
  const uint32_t num = q1 * static_cast<uint32_t>(p.s_inv) + static_cast<uint32_t>(x + p.s_inv);
  return static_cast<int32_t>(shr_clamp(num, q1));
}

// floor(alpha 2^32 / s_inv) for 0 <= alpha <= s_inv < 2^25, exactly, via the
// 64-bit release magic (floor(n / s_inv) = hi64(n mg) >> rel_shift, n < 2^56):
// hi64((alpha 2^32) (mh 2^32 + ml)) = alpha mh + hi32(alpha ml).
QF_DEV uint64_t alpha_over_sinv_2p32(uint32_t alpha, const IntParams& p) {
  const uint64_t hi = static_cast<uint64_t>(alpha) * p.rel_magic_hi + __umulhi(alpha, p.rel_magic_lo);
  return hi >> p.rel_shift;
}

// Fast exact ScaleRelease (Eq. 14 realised per P:L408, reading R10):
// floor(X alpha / s_inv) for |X| <= bound.  With B = (bound >> k) + 1, 2^k <= s_inv,
// X' = X + B s_inv lies in [1, 3 bound + s_inv); whenever X' s_inv < 2^32 (the
// per-launch threshold `rel_lthr` on l guarantees it),
//   floor(X alpha / s_inv) = floor(X' alpha / s_inv) - B alpha = hi(X' A_c) - B alpha,
// A_c = floor(alpha 2^32 / s_inv) + 1: the ceiling error X' (A_c 2^-32 - alpha / s_inv)
// < 1 / s_inv cannot cross an integer (the fraction of X' alpha / s_inv is a
// multiple of 1 / s_inv).  alpha = s_inv (identity) uses A = 2^32 - 1:
// hi(X' (2^32 - 1)) = X' - 1, corrected by +1.  Per element: IADD3 + IMAD.HI (with
// the addend folded in).
struct BiasedRelease {
  uint32_t bias;  // B s_inv
  uint32_t mul;   // A_c (or 2^32 - 1 for identity rows)
  uint32_t add;   // -B alpha (+1 for identity rows)
  QF_DEV uint32_t apply(uint32_t X) const {
    uint32_t r;
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(X + bias), "r"(mul), "r"(add));
    return r;
  }
};
QF_DEV BiasedRelease make_biased_release(int32_t alpha, uint32_t bound, const IntParams& p,
                                         int sinv_log2) {
  const uint32_t B = (bound >> sinv_log2) + 1u;
  const bool ident = alpha == p.s_inv;
  BiasedRelease r;
  r.bias = B * static_cast<uint32_t>(p.s_inv);
  r.mul = ident ? 0xFFFFFFFFu : static_cast<uint32_t>(alpha_over_sinv_2p32(alpha, p)) + 1u;
  r.add = (0u - B * static_cast<uint32_t>(alpha)) + (ident ? 1u : 0u);
  return r;
}

// A = min(floor(alpha 2^31 / s_inv), 2^31 - 1): per-row constant of the general release.
QF_DEV int32_t release_factor(int32_t alpha, const IntParams& p) {
  uint64_t a = alpha_over_sinv_2p32(static_cast<uint32_t>(alpha), p) >> 1;
  if (a > 0x7FFFFFFFull) a = 0x7FFFFFFFull;
  return static_cast<int32_t>(a);
}
// General exact ScaleRelease of one accumulator: q0 = floor(X A / 2^31) is within
// one of the answer; the remainder X alpha - q0 s_inv (exact mod 2^32, true value
// in [-s_inv, 2 s_inv)) corrects it.
QF_DEV int32_t scale_release(int32_t X, int32_t alpha, int32_t A, int32_t s_inv) {
  int32_t q0 = mul_shr31(X, A);
  const int32_t rem = X * alpha - q0 * s_inv;
  q0 += (rem >= s_inv) ? 1 : 0;
  q0 += rem >> 31;  // -1 if rem < 0
  return q0;
}

// Step (11): floor(O / l) exactly.  R = kRecip[...] approximates 2^(62-k)/l to
// 2^-11; q0 = floor(O R / 2^(62-k)) is within one of the answer because
// |O / l| < 2^11; the remainder corrects it.
struct Recip {
  int32_t R;
  int32_t sh;
  int32_t l;
};
QF_DEV Recip make_recip(int32_t l, const uint32_t* table) {
  const int32_t k = __clz(l);                         // l >= 2  =>  1 <= k <= 30
  const uint32_t ln = static_cast<uint32_t>(l) << k;  // [2^31, 2^32)
  Recip r;
  r.R = static_cast<int32_t>(table[(ln >> 21) & 1023u]);
  r.sh = 30 - k;
  r.l = l;
  return r;
}
QF_DEV int32_t floor_div(int32_t O, const Recip& r, bool& bad) {
  int32_t q0 = __mulhi(O, r.R) >> r.sh;
  const int32_t rem = O - q0 * r.l;
  q0 += (rem >= r.l) ? 1 : 0;
  q0 += rem >> 31;  // -1 if rem < 0
  bad |= (rem >= 2 * r.l) | (rem < -r.l);
  return q0;
}
QF_DEV int32_t floor_div_exact(int32_t O, int32_t l) {
  int64_t d = l;
  int64_t qq = 0, acc = 0;
  const bool neg = O < 0;
  const uint64_t un = neg ? static_cast<uint64_t>(-(static_cast<int64_t>(O) + 1)) : static_cast<uint64_t>(O);
#pragma unroll 1
  for (int b = 31; b >= 0; --b) {
    acc = (acc << 1) | static_cast<int64_t>((un >> b) & 1u);
    if (acc >= d) {
      acc -= d;
      qq |= (1ll << b);
    }
  }
  return static_cast<int32_t>(neg ? ~qq : qq);  // floor(O/l) = ~floor(~O/l) for O < 0
}

QF_DEV void sts32(uint32_t addr, int32_t v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
QF_DEV int32_t lds32(uint32_t addr) {
  int32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

// Persistent tile iterator (identical in every role of a group); no runtime
// division: the host supplies the magics and the stride quotient/remainder.
//   generic (NSEG = 1): tile t = problem * T_r + qt, rows [128 qt, 128 qt + 128).
//   row-packed:         tile t = flattened rows [128 t, 128 t + 128) of [P N].
// Group g of CTA b visits tiles b + g G, then steps by QT G.
template <int NSEG>
struct TileIter {
  int problem;  // first problem of the tile
  int off;      // row of tile row 0 inside `problem`
  int rows;     // live tile rows [0, rows)
  int nseg;     // problems the tile spans (1..NSEG)
  int i;        // tiles visited by this group
  __device__ void fill(const AttnArgs& a) {
    if constexpr (NSEG == 1) {
      rows = min(kBlockR, a.N - off);
      nseg = 1;
    } else {
      const int64_t left = static_cast<int64_t>(a.P - problem) * a.N - off;
      rows = left < kBlockR ? static_cast<int>(left) : kBlockR;
      const int last = off + rows - 1;
      nseg = 1 + (last >= a.N ? 1 : 0);
      if constexpr (NSEG > 2) nseg += (last >= 2 * a.N ? 1 : 0) + (last >= 3 * a.N ? 1 : 0);
    }
  }
  __device__ void init(const AttnArgs& a, uint32_t t) {
    i = 0;
    if constexpr (NSEG == 1) {
      problem = a.Tr == 1 ? static_cast<int>(t) : static_cast<int>(__umulhi(t, a.tr_magic));
      off = (static_cast<int>(t) - problem * a.Tr) * kBlockR;
    } else {
      const uint64_t row0 = static_cast<uint64_t>(t) * kBlockR;
      problem = static_cast<int>(__umul64hi(row0, a.n_magic));  // floor(row0 / N), exact
      off = static_cast<int>(row0 - static_cast<uint64_t>(problem) * a.N);
    }
    if (problem < a.P) fill(a);
  }
  __device__ bool valid(const AttnArgs& a) const { return problem < a.P; }
  __device__ void next(const AttnArgs& a) {
    ++i;
    problem += a.g_div;
    off += a.g_mod;
    const int lim = NSEG == 1 ? a.Tr * kBlockR : a.N;
    if (off >= lim) {
      off -= lim;
      ++problem;
    }
    if (problem < a.P) fill(a);
  }
};

// Bring-up timeline: clock64() stamps of CTA 0, group 0, first tile (DBG only).
#define QF_TS(slot)                                         \
  do {                                                      \
    if constexpr (DBG) {                                    \
      if (args.dbg_t != nullptr && (slot) < 128)            \
        args.dbg_t[(slot)] = clock64();                     \
    }                                                       \
  } while (0)

// ---------------------------------------------------------------- softmax role
// Masked 8-column groups: column group k of a thread is fully valid, partial
// (the ragged edge), or absent; `valid` is warp-uniform so the branches are too.
// Per-head granularity: the constants of head h = problem mod H
// (problems are (batch, window, head) with the head fastest), read per tile.
struct RowConsts {
  uint32_t s_inv;
  int sinv_log2;
  int32_t rel_lthr;
};
QF_DEV RowConsts row_consts(const IntParams& prm, int Tc) {
  RowConsts r;
  r.s_inv = static_cast<uint32_t>(prm.s_inv);
  r.sinv_log2 = 31 - __clz(prm.s_inv);
  // fast-release threshold on l: (3 * 128 (l + 2 T_c) + s_inv) s_inv < 2^32, i.e.
  // 384 (l + 2 T_c) + s_inv <= floor((2^32 - 1) / s_inv) (64-bit magic, n < 2^56)
  const uint64_t mg = (static_cast<uint64_t>(prm.rel_magic_hi) << 32) | prm.rel_magic_lo;
  const uint64_t A = __umul64hi(0xFFFFFFFFull, mg) >> prm.rel_shift;
  const int64_t t = (static_cast<int64_t>(A) - static_cast<int64_t>(r.s_inv)) / 384 - 2 * Tc;
  r.rel_lthr = t < 0 ? -1 : (t > 0x7FFFFFFF ? 0x7FFFFFFF : static_cast<int32_t>(t));
  return r;
}
QF_DEV int head_of(const AttnArgs& a, uint32_t problem) {
  // problem mod H (H = 1: the 32-bit magic ceil(2^32 / 1) does not exist)
  const uint32_t q = a.H == 1 ? problem : __umulhi(problem, a.h_magic);
  return static_cast<int>(problem - q * static_cast<uint32_t>(a.H));
}
QF_DEV IntParams head_params(const AttnArgs& a, const IntParams* table, int problem) {
  return *reinterpret_cast<const IntParams*>(reinterpret_cast<const char*>(table) +
                                             kHeadPrmStride * head_of(a, static_cast<uint32_t>(problem)));
}

// tcgen05.ld of W consecutive 32-bit TMEM columns of this warp's lanes (no wait).
template <int W>
QF_DEV void tmem_ld_cols(uint32_t taddr, uint32_t* r) {
  if constexpr (W == 8) tmem_ld8(taddr, r);
  else if constexpr (W == 16) tmem_ld16(taddr, r);
  else if constexpr (W == 32) tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(r));
  else tmem_ld<W>(taddr, r);
}

// Max of N int32 values as a tree of 3-input maxima (VIMNMX3): dependency depth
// ceil(log3 N) instead of the N / 2 of a running max (a 16-deep chain for 32 columns).
template <int N>
QF_DEV int32_t tree_max(const int32_t* v) {
  if constexpr (N == 1) {
    return v[0];
  } else if constexpr (N == 2) {
    return max(v[0], v[1]);
  } else {
    constexpr int M = (N + 2) / 3;
    int32_t t[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const int32_t a = v[3 * i];
      const int32_t b = 3 * i + 1 < N ? v[3 * i + 1] : a;
      const int32_t c = 3 * i + 2 < N ? v[3 * i + 2] : a;
      t[i] = max(a, max(b, c));
    }
    return tree_max<M>(t);
  }
}

// Row max over the first `valid` of W columns (valid warp-uniform; <= 0: none).
template <int W>
QF_DEV int32_t row_max_masked(const uint32_t* s, int valid) {
  int32_t t = INT32_MIN;
  if (valid >= W) {
    t = tree_max<W>(reinterpret_cast<const int32_t*>(s));
  } else {
#pragma unroll
    for (int k = 0; k < W / 8; ++k) {
      if (8 * k + 8 <= valid) {
#pragma unroll
        for (int e = 8 * k; e < 8 * k + 8; ++e) t = max(t, static_cast<int32_t>(s[e]));
      } else if (8 * k < valid) {
#pragma unroll
        for (int e = 8 * k; e < 8 * k + 8; ++e)
          if (e < valid) t = max(t, static_cast<int32_t>(s[e]));
      }
    }
  }
  return t;
}

// Steps (5)(6) for W <= 32 columns: P = Requant(ShiftExp2(S - m_new)) packed 4 per
// word into pw[W / 4]; columns >= hv (warp-uniform) get P = 0; hv <= 0 leaves pw.
template <int W, bool FASTQ>
QF_DEV void p_pack(const uint32_t* sc, int hv, uint32_t mu, uint32_t nmu, uint32_t c3, uint32_t one,
                   const IntParams& prm, uint32_t* pw) {
  if (hv >= W) {
#pragma unroll
    for (int e = 0; e < W; e += 4)
      pw[e / 4] = pack4_sat_s8(
          shift_exp2_requant<FASTQ, false>(static_cast<int32_t>(sc[e]), mu, nmu, c3, one, prm),
          shift_exp2_requant<FASTQ, true>(static_cast<int32_t>(sc[e + 1]), mu, nmu, c3, one, prm),
          shift_exp2_requant<FASTQ, false>(static_cast<int32_t>(sc[e + 2]), mu, nmu, c3, one, prm),
          shift_exp2_requant<FASTQ, true>(static_cast<int32_t>(sc[e + 3]), mu, nmu, c3, one, prm));
  } else {
#pragma unroll
    for (int k = 0; k < W / 8; ++k) {
      if (8 * k + 8 <= hv) {
#pragma unroll
        for (int e = 8 * k; e < 8 * k + 8; e += 4)
          pw[e / 4] = pack4_sat_s8(
              shift_exp2_requant<FASTQ, false>(static_cast<int32_t>(sc[e]), mu, nmu, c3, one, prm),
              shift_exp2_requant<FASTQ, true>(static_cast<int32_t>(sc[e + 1]), mu, nmu, c3, one, prm),
              shift_exp2_requant<FASTQ, false>(static_cast<int32_t>(sc[e + 2]), mu, nmu, c3, one, prm),
              shift_exp2_requant<FASTQ, true>(static_cast<int32_t>(sc[e + 3]), mu, nmu, c3, one, prm));
      } else if (8 * k < hv) {
#pragma unroll
        for (int e = 8 * k; e < 8 * k + 8; e += 4) {
          int32_t pv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int32_t x = shift_exp2_requant<FASTQ, false>(static_cast<int32_t>(sc[e + u]), mu, nmu, c3, one, prm);
            pv[u] = (e + u < hv) ? x : 0;
          }
          pw[e / 4] = pack4_sat_s8(pv[0], pv[1], pv[2], pv[3]);
        }
      }
    }
  }
}

// ---- Scale Accumulation (Eq. 13; the rejected alternative of App. B.1)
// X <- X alpha + Y s_inv in int64 with two's-complement wrap (the oracle's int64 cast of
// the exact int128 value); flags bit 0: the exact value left int64, bit 1: it left int32
// (an int32-accumulator kernel would have overflowed).
QF_DEV int64_t acc_update(int64_t X, int32_t alpha, int32_t Y, int32_t s_inv, uint32_t& flags) {
  const __int128 v = static_cast<__int128>(X) * alpha + static_cast<__int128>(Y) * s_inv;
  if (v > static_cast<__int128>(INT64_MAX) || v < static_cast<__int128>(INT64_MIN)) flags |= 1u;
  if (v > static_cast<__int128>(INT32_MAX) || v < static_cast<__int128>(INT32_MIN)) flags |= 2u;
  return static_cast<int64_t>(static_cast<unsigned __int128>(v));
}
// floor(a / b) for b > 0, integer-only restoring division (no FP lowering of `/`).
QF_DEV int64_t floor_div64(int64_t a, int64_t b) {
  const bool neg = a < 0;
  uint64_t un = neg ? static_cast<uint64_t>(-(a + 1)) : static_cast<uint64_t>(a);  // ~a for a < 0
  const uint64_t d = static_cast<uint64_t>(b);
  uint64_t q = 0, r = 0;
#pragma unroll 1
  for (int i = 63; i >= 0; --i) {
    r = (r << 1) | ((un >> i) & 1u);
    if (r >= d) {
      r -= d;
      q |= (1ull << i);
    }
  }
  return neg ? static_cast<int64_t>(~q) : static_cast<int64_t>(q);  // floor(a/b) = ~floor(~a/b), a < 0
}

// ---- FP softmax of the V2 ablation (N4): P = rint(127 exp2(s (S - m))) in fp32 --
QF_DEV float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <int W>
QF_DEV void p_pack_fp(const uint32_t* sc, int hv, int32_t m_new, float s_f, uint32_t* pw) {
#pragma unroll
  for (int e = 0; e < W; e += 4) {
    int32_t v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float p = ex2_approx(static_cast<float>(static_cast<int32_t>(sc[e + u]) - m_new) * s_f);
      v[u] = (e + u < hv) ? __float2int_rn(127.0f * p) : 0;
    }
    pw[e / 4] = pack4_sat_s8(v[0], v[1], v[2], v[3]);
  }
}

// Step (11) for one row's OW output columns [c OW, c OW + OW): O = floor(O / l)
// saturated to int8 (R14), stored as int8 and/or dequantized fp32 (DQ row) at
// flattened output row `orow` (row-packed tiles included).
template <int D, int OW, bool FMUL = false>
QF_DEV void normalize_store(const AttnArgs& args, int64_t orow, int c, const uint32_t* o, uint32_t lraw,
                            const uint32_t* recip, float sv = 0.f) {
  const Recip rc = make_recip(static_cast<int32_t>(lraw), recip);
  bool bad = false;
  uint32_t w[OW / 4];
#pragma unroll
  for (int e = 0; e < OW; e += 4)
    w[e / 4] = pack4_sat_s8(floor_div(static_cast<int32_t>(o[e]), rc, bad),
                            floor_div(static_cast<int32_t>(o[e + 1]), rc, bad),
                            floor_div(static_cast<int32_t>(o[e + 2]), rc, bad),
                            floor_div(static_cast<int32_t>(o[e + 3]), rc, bad));
  if (bad) {  // (theoretical) quotient outside the table's exact range: long division
#pragma unroll
    for (int e = 0; e < OW; e += 4)
      w[e / 4] = pack4_sat_s8(floor_div_exact(static_cast<int32_t>(o[e]), rc.l),
                              floor_div_exact(static_cast<int32_t>(o[e + 1]), rc.l),
                              floor_div_exact(static_cast<int32_t>(o[e + 2]), rc.l),
                              floor_div_exact(static_cast<int32_t>(o[e + 3]), rc.l));
  }
  if (args.out != nullptr) {
    int8_t* dst = args.out + orow * D + c * OW;
    if constexpr (OW == 8) {
      *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
    } else {
#pragma unroll
      for (int e = 0; e < OW / 16; ++e)
        reinterpret_cast<uint4*>(dst)[e] = make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
    }
  }
  if (args.out_f32 != nullptr) {
    // fused dequantization y = s_V * O^ (DQ row): the fp32 bit pattern of every
    // int8 value comes from a 256-entry table the quantize kernel computed with
    // the same IEEE multiply as qflash_dequantize -- the attention kernel itself
    // stays integer-only.
    const uint32_t dqt = smem_u32(recip + 1024);
    const uint64_t ypol = QF_EVICT_FIRST ? l2_evict_first_policy() : 0ull;  // y is written once
    uint32_t* ydst = reinterpret_cast<uint32_t*>(args.out_f32 + orow * D + c * OW);
#pragma unroll
    for (int e = 0; e < OW / 4; ++e) {
      uint32_t y4[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if constexpr (FMUL) {  // per-head scales (fused per-head step): y = fl32(s_V[h] x^)
          const int32_t x = static_cast<int32_t>(static_cast<int8_t>((w[e] >> (8 * b)) & 0xFFu));
          y4[b] = __float_as_uint(__fmul_rn(sv, static_cast<float>(x)));
        } else {
          y4[b] = static_cast<uint32_t>(lds32(dqt + ((((w[e] >> (8 * b)) & 0xFFu) ^ 0x80u) << 2)));
        }
      }
      if (QF_EVICT_FIRST) stg_ef(reinterpret_cast<uint4*>(ydst) + e, make_uint4(y4[0], y4[1], y4[2], y4[3]), ypol);
      else reinterpret_cast<uint4*>(ydst)[e] = make_uint4(y4[0], y4[1], y4[2], y4[3]);
    }
  }
}

template <int D, int BC, int NSEG, int CS, int QT, bool DBG, bool FASTQ, bool PH = false, int VAR = 0,
          int FQ_PH = 0>
__device__ __forceinline__ void softmax_role(const AttnArgs& args, const IntParams& prm_k,
                                             uint32_t tmem_group, GroupBars<Cfg<D, BC, NSEG, CS, QT>::kNumS> gb,
                                             uint32_t red_group, const uint32_t* recip, int g,
                                             int c, int quarter, int lane, const IntParams* head_tab = nullptr) {
  using C = Cfg<D, BC, NSEG, CS, QT>;
  constexpr int CW = C::kCW;
  constexpr int OW = C::kOW;
  const int N = args.N;
  const int Tc = args.Tc;
  const int row = quarter * 32 + lane;  // TMEM lane == tile row
  const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
  const uint32_t tS0 = tmem_group + lane_off;  // S buffer b at + b * BC
  const uint32_t tO = tS0 + C::kOCol;
  const uint32_t tP = tS0 + C::kPCol;  // kSepP
  const int c0 = c * CW;  // first key column of this thread
  const bool dbg_on = DBG && blockIdx.x == 0 && g == 0;
  const bool ts_warp = dbg_on && c == 0 && quarter == 0 && lane == 0;
  const RowConsts rck = row_consts(prm_k, Tc);  // per-tensor constants (PH: per tile below)

  TileIter<NSEG> ti;
  ti.init(args, blockIdx.x + g * gridDim.x);
  int it0 = 0;  // KV iterations of this group so far
  uint64_t* tables_bar = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(const_cast<uint32_t*>(recip)) -
                                                     C::kRecip + C::kTmemSlot + 8);
  bool tables_ready = false;
  for (; ti.valid(args); ti.next(args)) {
    const bool dbg = dbg_on && ti.i == 0;
    const bool live = row < ti.rows;  // padded rows of the last tile do no work
    const bool warp_live = quarter * 32 < ti.rows;
    int seg = 0;  // this row's problem = ti.problem + seg
    if constexpr (NSEG > 1) {
      const int x = ti.off + row;
      seg = (x >= N ? 1 : 0);
      if constexpr (NSEG > 2) seg += (x >= 2 * N ? 1 : 0) + (x >= 3 * N ? 1 : 0);
    }
    const int nseg = ti.nseg;
    int32_t m = -(1 << 21);  // m^(0) = -2^21
    IntParams prm_t;
    RowConsts rct = rck;
    if constexpr (PH) {
      prm_t = head_params(args, head_tab, ti.problem + seg);
      rct = row_consts(prm_t, Tc);
    }
    const IntParams& prm = PH ? prm_t : prm_k;
    const uint32_t s_inv = PH ? rct.s_inv : rck.s_inv;
    const int sinv_log2 = PH ? rct.sinv_log2 : rck.sinv_log2;
    const int32_t rel_lthr = PH ? rct.rel_lthr : rck.rel_lthr;
    // Ablation variants (VAR > 0): P V_j lands fresh in TMEM every KV tile and is folded
    // into register accumulators of this thread's O columns and l --
    //   VAR 1 (Eq. 13, N3): int64, O <- O alpha + PV s_inv (flags: int64 / int32 overflow);
    //   VAR 2 (V3, N4): fp32, O <- O (alpha / s_inv) + PV  (integer exp, FP accumulation);
    //   VAR 3 (V2, N4): fp32, O <- O alpha_f + PV           (FP exp2 softmax, int8 P V).
    constexpr bool kAcc = VAR == 1;
    constexpr bool kFp = VAR >= 2;
    int64_t o64[kAcc ? OW : 1];
    float of[kFp ? OW : 1];
    int64_t l64 = 0;
    float lf = 0.f;
    int32_t alpha_prev = 0;
    float alpha_prev_f = 0.f;
    uint32_t acc_flags = 0;
    if constexpr (kAcc) {
#pragma unroll
      for (int e = 0; e < OW; ++e) o64[e] = 0;
    }
    if constexpr (kFp) {
#pragma unroll
      for (int e = 0; e < OW; ++e) of[e] = 0.f;
    }
    const float s_f = static_cast<float>(prm.s);              // VAR 3: real logit scale (log2 domain)
    const float rinv_f = 1.0f / static_cast<float>(s_inv);   // VAR 2: 1 / s_inv
    auto acc_fold = [&](int32_t al, float al_f) {
      if constexpr (VAR == 0) return;
      if (!warp_live) return;
      uint32_t o[OW], lc;
      tmem_ld_cols<OW>(tO + c * OW, o);
      tmem_ld1(tO + D + c, lc);  // an unreleased copy of rowsum(P_j) from the ones block
      tmem_wait_ld();
      if constexpr (kAcc) {  // O <- O alpha + PV s_inv, l <- l alpha + rowsum(P) s_inv
        uint32_t f = 0;
#pragma unroll
        for (int e = 0; e < OW; ++e)
          o64[e] = acc_update(o64[e], al, static_cast<int32_t>(o[e]), static_cast<int32_t>(s_inv), f);
        l64 = acc_update(l64, al, static_cast<int32_t>(lc), static_cast<int32_t>(s_inv), f);
        if (live) acc_flags |= f;  // padding rows of the last query tile do not count
      } else {
        const float a = VAR == 2 ? static_cast<float>(al) * rinv_f : al_f;
#pragma unroll
        for (int e = 0; e < OW; ++e) of[e] = fmaf(of[e], a, static_cast<float>(static_cast<int32_t>(o[e])));
        lf = fmaf(lf, a, static_cast<float>(static_cast<int32_t>(lc)));
      }
    };

    for (int j = 0; j < Tc; ++j) {
      const int it = it0 + j;
      const int sb = (C::kNumS == 2) ? (it & 1) : 0;
      const uint32_t tS = tS0 + sb * BC;
      if (QF_SLEEP_SOFT > 0)
        mbar_wait_sleep(gb.s_full(sb), (C::kNumS == 2 ? (it >> 1) : it) & 1, QF_SLEEP_SOFT);
      else
        mbar_wait(gb.s_full(sb), (C::kNumS == 2 ? (it >> 1) : it) & 1);
      tc_fence_after();
      if (dbg && ts_warp && j < 7) QF_TS(40 + 8 * j);
      // columns of this thread that exist in KV tile j (ragged last tile, R16)
      const int valid = min(BC, N - j * BC) - c0;
      // S columns of this thread: CW <= 32 stay in registers for the P pass;
      // CW = 64 is loaded whole for the max and reloaded per 32-column chunk.
      constexpr int HW = CW < 32 ? CW : 32;  // chunk width
      constexpr int NH = CW / HW;            // chunks
      uint32_t s[CW];
      int32_t tmax = INT32_MIN;
      if (warp_live && valid > 0) {
        if constexpr (CW == 16) {
          tmem_ld16(tS + c0, s);
        } else {
#pragma unroll
          for (int h = 0; h < NH; ++h) tmem_ld32(tS + c0 + 32 * h, *reinterpret_cast<uint32_t(*)[32]>(s + 32 * h));
        }
        tmem_wait_ld();
        if (dbg && ts_warp && j < 7) QF_TS(60 + j);
        if constexpr (DBG) {
          if (args.dbg_s != nullptr && dbg && j == 0)
            for (int e = 0; e < CW; ++e) args.dbg_s[row * BC + c0 + e] = static_cast<int32_t>(s[e]);
        }
        tmax = row_max_masked<CW>(s, valid);
        if (dbg && ts_warp && j < 7) QF_TS(70 + j);
      }
      // (2)(3) combine the partial maxima of the group's CS warpgroups
      if constexpr (CS > 1) {
        const uint32_t rb = red_group + static_cast<uint32_t>((it & 1) * (CS * 128) * 4);
        sts32(rb + static_cast<uint32_t>((c * 128 + row) * 4), tmax);
        // only the CS warps that share this warp's TMEM lane quarter (the same 32
        // rows) exchange maxima, and only their S / P columns alias: one named
        // barrier per (group, lane quarter) of CS x 32 threads
        named_bar_sync(1 + g * 4 + quarter, CS * 32);
#pragma unroll
        for (int h = 0; h < CS; ++h)
          if (h != c) tmax = max(tmax, lds32(rb + static_cast<uint32_t>((h * 128 + row) * 4)));
      }
      if (dbg && ts_warp && j < 7) QF_TS(41 + 8 * j);
      const int32_t m_new = max(m, tmax);
      // (4) alpha = ShiftExp2(m_old - m_new)
      const int32_t alpha = shift_exp2<FASTQ>(m - m_new, prm);
      float alpha_f = 0.f;  // VAR 3: exp2(s (m_old - m_new)) in fp32
      if constexpr (VAR == 3) alpha_f = ex2_approx(static_cast<float>(m - m_new) * s_f);

      // (5)(6) P = Requant(ShiftExp2(S - m_new)), 4 x int8 per TMEM column.
      const uint32_t mu = static_cast<uint32_t>(m_new);
      const uint32_t nmu = static_cast<uint32_t>(-m_new);
      const uint32_t c3 = s_inv - mu;
      const uint32_t one = static_cast<uint32_t>(prm.one);
      // Computed in chunks of HW <= 32 columns (CW = 64 reloads each chunk from
      // TMEM); all P words are stored after the last chunk's S load.  Layout of
      // the packed P of segment s in the S buffer (kernel_p_col): CW >= 32 puts
      // each warpgroup's P inside its own S columns ("own range", no other
      // warpgroup reads them); CW = 16 packs the row contiguously, which is safe
      // because every warpgroup's S loads completed before the max exchange.
      uint32_t pk[CW / 4];
#pragma unroll
      for (int e = 0; e < CW / 4; ++e) pk[e] = 0u;
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const int hv = valid - h * HW;  // valid columns of this chunk (warp-uniform)
        if (warp_live && hv > 0) {
          uint32_t sc[HW];
          if constexpr (NH == 1) {
#pragma unroll
            for (int e = 0; e < HW; ++e) sc[e] = s[e];
          } else {
            tmem_ld32(tS + c0 + 32 * h, *reinterpret_cast<uint32_t(*)[32]>(sc));
            tmem_wait_ld();
          }
          if constexpr (VAR == 3)
            p_pack_fp<HW>(sc, hv, m_new, s_f, pk + h * (HW / 4));
          else
            p_pack<HW, FASTQ>(sc, hv, mu, nmu, c3, one, prm, pk + h * (HW / 4));
        }
      }
      if constexpr (C::kSepP) {
        // every S read of this warp is done: the next Q K^T may overwrite S; P goes
        // to its own region once P V_{j-1} has read the previous P (o_full)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(gb.s_empty());
        if (j > 0) {
          mbar_wait(gb.o_full(), (it - 1) & 1);
          tc_fence_after();
        }
        tmem_st<CW / 4>(tP + c * (CW / 4), pk);
      } else if (nseg == 1) {
        tmem_st<CW / 4>(tS + p_col<BC, CW>(c, 0), pk);
      } else {
        // segment s gets this row's P if the row belongs to it, zeros otherwise
#pragma unroll
        for (int sg = 0; sg < NSEG; ++sg) {
          if (sg < nseg) {
            uint32_t z[CW / 4];
#pragma unroll
            for (int e = 0; e < CW / 4; ++e) z[e] = (seg == sg && live) ? pk[e] : 0u;
            tmem_st<CW / 4>(tS + p_col<BC, CW>(c, sg), z);
          }
        }
      }
      if (dbg && ts_warp && j < 7) QF_TS(44 + 8 * j);

      // (7)(8) ScaleRelease of O (this warpgroup's columns) and l (warpgroup 0)
      // once P V_{j-1} has landed -- after P_j so that P V_{j-1} completes behind
      // the P computation; skipped for j = 0 (O = l = 0) and for warps whose rows
      // all kept their maximum (alpha = s_inv is the identity, R10).  P V_j is
      // issued only after every warp's p_full arrival below, i.e. after the release.
      if constexpr (VAR != 0) {
        if (j > 0) {  // fold step j-1 (its alpha, its P V) before P V_j overwrites TMEM
          mbar_wait(gb.o_full(), (it - 1) & 1);
          tc_fence_after();
          acc_fold(alpha_prev, alpha_prev_f);
        }
        alpha_prev = alpha;
        alpha_prev_f = alpha_f;
      } else if (j > 0) {
        if constexpr (!C::kSepP) {
          mbar_wait(gb.o_full(), (it - 1) & 1);
          tc_fence_after();
        }
        if (dbg && ts_warp && j < 7) QF_TS(45 + 8 * j);
        if (warp_live && __any_sync(0xffffffffu, alpha != prm.s_inv)) {
          uint32_t o[OW];
          if constexpr (OW == 8) tmem_ld8(tO + c * OW, o);
          else if constexpr (OW == 16) tmem_ld16(tO + c * OW, o);
          else tmem_ld<OW>(tO + c * OW, o);
          // l for this warpgroup's bound: warpgroup 0 reads (and later rewrites)
          // column D, the released l; warpgroup c > 0 reads its own copy D + c of
          // the ones block, never released -- an upper bound of l, so a valid
          // bound -- because column D may already hold warpgroup 0's released l.
          uint32_t lcol;
          tmem_ld1(tO + D + c, lcol);
          tmem_wait_ld();
          if (dbg && ts_warp && j < 7) QF_TS(46 + 8 * j);
          // Fast exact path when every row of the warp has l <= rel_lthr
          // (bound |O| <= 128 (l + 2 T_c)).
          if (__all_sync(0xffffffffu, static_cast<int32_t>(lcol) <= rel_lthr)) {
            const uint32_t bound = 128u * (lcol + 2u * static_cast<uint32_t>(Tc));
            const BiasedRelease br = make_biased_release(alpha, bound, prm, sinv_log2);
#pragma unroll
            for (int e = 0; e < OW; ++e) o[e] = br.apply(o[e]);
            tmem_st<OW>(tO + c * OW, o);
            if (c == 0) tmem_st1(tO + D, br.apply(lcol));
          } else {
            const int32_t A = release_factor(alpha, prm);
#pragma unroll
            for (int e = 0; e < OW; ++e)
              o[e] = static_cast<uint32_t>(scale_release(static_cast<int32_t>(o[e]), alpha, A, prm.s_inv));
            tmem_st<OW>(tO + c * OW, o);
            if (c == 0)
              tmem_st1(tO + D, static_cast<uint32_t>(scale_release(static_cast<int32_t>(lcol), alpha, A, prm.s_inv)));
          }
          if (dbg && ts_warp && j < 7) QF_TS(47 + 8 * j);
        }
      }

      tmem_wait_st();
      if constexpr (DBG) {
        if (args.dbg_p != nullptr && dbg && j == 0) {
          if constexpr (CS > 1) named_bar_sync(1 + g * 4 + quarter, CS * 32);
          if (c == 0) {
            for (int kk = 0; kk < BC / 32; ++kk) {
              uint32_t pw[8];
              tmem_ld8(tS + p_col_k<BC, CW>(kk, 0), pw);
              tmem_wait_ld();
              for (int e = 0; e < 8; ++e) args.dbg_p[row * (BC / 4) + 8 * kk + e] = static_cast<int32_t>(pw[e]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(gb.p_full());
      if (dbg && ts_warp && j < 7) QF_TS(43 + 8 * j);
      m = m_new;
    }

    // (11) O_i = floor(O / l), saturated to int8 (R14); this warpgroup's O columns.
    const int itl = it0 + Tc - 1;
    mbar_wait(gb.o_full(), itl & 1);
    tc_fence_after();
    if (dbg && ts_warp) QF_TS(100);
    if (!tables_ready) {  // the step-(11) tables warp 3 loaded (complete long before)
      mbar_wait(tables_bar, 0);
      tables_ready = true;
    }
    if (dbg && ts_warp) QF_TS(103);
    if constexpr (VAR >= 2) {
      acc_fold(alpha_prev, alpha_prev_f);
      if (warp_live && live) {  // y = s_V O / l in fp32 (the FP variants' natural output)
        const float k = args.s_v / lf;
        float* ydst = args.out_f32 + (static_cast<int64_t>(ti.problem) * N + ti.off + row) * D + c * OW;
#pragma unroll
        for (int e = 0; e < OW; e += 4)
          *reinterpret_cast<float4*>(ydst + e) = make_float4(of[e] * k, of[e + 1] * k, of[e + 2] * k, of[e + 3] * k);
      }
      it0 += Tc;
      continue;
    }
    if constexpr (VAR == 1) {
      acc_fold(alpha_prev, 0.f);
      if (warp_live && live) {
        uint32_t w[OW / 4];
#pragma unroll
        for (int e = 0; e < OW; e += 4) {
          int32_t v4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            int64_t q = l64 > 0 ? floor_div64(o64[e + u], l64) : 0;  // oracle: l <= 0 -> 0
            v4[u] = static_cast<int32_t>(q > 127 ? 127 : (q < -128 ? -128 : q));
          }
          w[e / 4] = pack4_sat_s8(v4[0], v4[1], v4[2], v4[3]);
        }
        int8_t* dst = args.out + (static_cast<int64_t>(ti.problem) * N + ti.off + row) * D + c * OW;
#pragma unroll
        for (int e = 0; e < OW / 4; ++e) reinterpret_cast<uint32_t*>(dst)[e] = w[e];
      }
      if (warp_live) {
        const uint32_t f = __reduce_or_sync(0xffffffffu, acc_flags);
        if (lane == 0 && f != 0) atomicOr(args.acc_flags, static_cast<int32_t>(f));
      }
      it0 += Tc;
      continue;
    }
    if (warp_live) {
      uint32_t lraw;
      uint32_t o[OW];
      tmem_ld1(tO + D, lraw);
      if constexpr (OW == 8) tmem_ld8(tO + c * OW, o);
      else if constexpr (OW == 16) tmem_ld16(tO + c * OW, o);
      else tmem_ld<OW>(tO + c * OW, o);
      tmem_wait_ld();
      if (dbg && ts_warp) QF_TS(104);
      if constexpr (DBG) {
        if (args.dbg_o != nullptr && dbg) {
          for (int e = 0; e < OW; ++e) args.dbg_o[row * (D + 1) + c * OW + e] = static_cast<int32_t>(o[e]);
          if (c == 0) args.dbg_o[row * (D + 1) + D] = static_cast<int32_t>(lraw);
        }
      }
      if (live)  // the fused step dequantizes with an FMUL by s_V (per head: s_V[h]) kept in pad[0]
        normalize_store<D, OW, (FQ_PH != 0)>(args, static_cast<int64_t>(ti.problem) * N + ti.off + row, c,
                                               o, lraw, recip, __int_as_float(prm.pad[0]));
    }
    if (dbg && ts_warp) QF_TS(101);
    // The O/l loads above completed (wait::ld) before this thread's next p_full
    // arrival, so the next tile's first P V (which overwrites O) cannot race them.
    it0 += Tc;
  }
}

// ---------------------------------------------------------------- row-owner roles (CS = 1)
// Named barriers of the alpha hand-off (softmax warpgroup -> correction warpgroup of
// group g, double-buffered slot b), 128 + 128 threads each: ids 1..8 (0 = __syncthreads;
// the column-split configurations use 1..8 for their max exchange instead).
QF_DEV uint32_t rc_full_bar(int g, int b) { return 1u + 4u * g + b; }
QF_DEV uint32_t rc_free_bar(int g, int b) { return 3u + 4u * g + b; }
// Softmax warpgroup: thread = query row, all B_c key columns of every KV tile.
// No cross-warpgroup max exchange; alpha goes to the correction warpgroup
// through shared memory (a pair of named barriers), P (packed, contiguous per segment)
// over the S buffer once every S chunk of the row has been read.
template <int D, int BC, int NSEG, int QT, bool FASTQ>
__device__ __forceinline__ void softmax_rc_role(const AttnArgs& args, const IntParams& prm,
                                                uint32_t tmem_group,
                                                GroupBars<Cfg<D, BC, NSEG, 1, QT>::kNumS> gb,
                                                uint32_t alpha_buf, int g, int quarter, int lane) {
  using C = Cfg<D, BC, NSEG, 1, QT>;
  constexpr int NH = BC / 32;  // 32-column chunks
  const int N = args.N;
  const int Tc = args.Tc;
  const int row = quarter * 32 + lane;
  const uint32_t tS0 = tmem_group + (static_cast<uint32_t>(quarter * 32) << 16);
  const uint32_t s_inv = static_cast<uint32_t>(prm.s_inv);
  const uint32_t one = static_cast<uint32_t>(prm.one);
  TileIter<NSEG> ti;
  ti.init(args, blockIdx.x + g * gridDim.x);
  int it0 = 0;
  for (; ti.valid(args); ti.next(args)) {
    const bool live = row < ti.rows;
    const bool warp_live = quarter * 32 < ti.rows;
    int seg = 0;
    if constexpr (NSEG > 1) {
      const int x = ti.off + row;
      seg = (x >= N ? 1 : 0);
      if constexpr (NSEG > 2) seg += (x >= 2 * N ? 1 : 0) + (x >= 3 * N ? 1 : 0);
    }
    const int nseg = ti.nseg;
    int32_t m = -(1 << 21);  // m^(0) = -2^21
    for (int j = 0; j < Tc; ++j) {
      const int it = it0 + j;
      const int sb = (C::kNumS == 2) ? (it & 1) : 0;
      const uint32_t tS = tS0 + sb * BC;
      if (QF_SLEEP_SOFT > 0)
        mbar_wait_sleep(gb.s_full(sb), (C::kNumS == 2 ? (it >> 1) : it) & 1, QF_SLEEP_SOFT);
      else
        mbar_wait(gb.s_full(sb), (C::kNumS == 2 ? (it >> 1) : it) & 1);
      tc_fence_after();
      const int valid = min(BC, N - j * BC);  // ragged last KV tile (R16), warp-uniform
      // (2)(3) row max over the valid columns, two 32-column chunks per TMEM wait
      int32_t tmax = INT32_MIN;
      if (warp_live) {
#pragma unroll
        for (int h2 = 0; h2 < NH; h2 += 2) {
          uint32_t sc[64];
          tmem_ld32(tS + 32 * h2, *reinterpret_cast<uint32_t(*)[32]>(sc));
          if (h2 + 1 < NH) tmem_ld32(tS + 32 * h2 + 32, *reinterpret_cast<uint32_t(*)[32]>(sc + 32));
          tmem_wait_ld();
          constexpr int W = NH >= 2 ? 64 : 32;
          tmax = max(tmax, row_max_masked<W>(sc, valid - 32 * h2));
        }
      }
      const int32_t m_new = max(m, tmax);
      // (4) alpha = ShiftExp2(m_old - m_new), handed to the correction warpgroup
      const int32_t alpha = shift_exp2<FASTQ>(m - m_new, prm);
      // slot it & 1: free once the correction warpgroup read it at iteration it - 2
      // (named barriers, so that racecheck models both directions of the hand-off)
      if (it >= 2) named_bar_sync(rc_free_bar(g, it & 1), 256);
      sts32(alpha_buf + static_cast<uint32_t>(((it & 1) * 128 + row) * 4), alpha);
      named_bar_arrive(rc_full_bar(g, it & 1), 256);
      // (5)(6) P = Requant(ShiftExp2(S - m_new)), chunk by chunk (S reloaded)
      const uint32_t mu = static_cast<uint32_t>(m_new);
      const uint32_t nmu = static_cast<uint32_t>(-m_new);
      const uint32_t c3 = s_inv - mu;
      uint32_t pk[BC / 4];
#pragma unroll
      for (int e = 0; e < BC / 4; ++e) pk[e] = 0u;
      if (warp_live) {
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const int hv = valid - 32 * h;
          if (hv > 0) {
            uint32_t sc[32];
            tmem_ld32(tS + 32 * h, sc);
            tmem_wait_ld();
            p_pack<32, FASTQ>(sc, hv, mu, nmu, c3, one, prm, pk + 8 * h);
          }
        }
      }
      // every S chunk of this row is read: P of segment s -> columns [s B_c/4, +B_c/4)
      if (nseg == 1) {
        tmem_st<BC / 4>(tS, pk);
      } else {
#pragma unroll
        for (int sg = 0; sg < NSEG; ++sg) {
          if (sg < nseg) {
            uint32_t z[BC / 4];
#pragma unroll
            for (int e = 0; e < BC / 4; ++e) z[e] = (seg == sg && live) ? pk[e] : 0u;
            tmem_st<BC / 4>(tS + sg * (BC / 4), z);
          }
        }
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(gb.p_full(it & 1));
      m = m_new;
    }
    it0 += Tc;
  }
  // drain: the correction warpgroup's "consumed" arrivals of the last two iterations
  for (int it = max(it0 - 2, 0); it < it0; ++it) named_bar_sync(rc_free_bar(g, it & 1), 256);
}

// Correction warpgroup: thread = query row.  Per KV tile j >= 1 it releases the
// row's O (all d columns) and l with the alpha of tile j once P V_{j-1} has
// landed (Eq. 14, R10) -- concurrently with the softmax warpgroup's P work --
// then arrives on rel_full, which the MMA warp needs (with p_full) before
// P V_j.  After the last KV tile: step (11) and the stores (int8 and/or the
// fused dequantization), before the next tile's first rel_full arrival.
template <int D, int BC, int NSEG, int QT, int FQ>
__device__ __forceinline__ void correction_role(const AttnArgs& args, const IntParams& prm,
                                                uint32_t tmem_group,
                                                GroupBars<Cfg<D, BC, NSEG, 1, QT>::kNumS> gb,
                                                uint32_t alpha_buf, const uint32_t* recip, int g,
                                                int quarter, int lane) {
  using C = Cfg<D, BC, NSEG, 1, QT>;
  constexpr int OH = D < 32 ? D : 32;  // O columns per TMEM round trip
  const int N = args.N;
  const int Tc = args.Tc;
  const int row = quarter * 32 + lane;
  const uint32_t tO = tmem_group + (static_cast<uint32_t>(quarter * 32) << 16) + C::kOCol;
  const int sinv_log2 = 31 - __clz(prm.s_inv);
  int32_t rel_lthr;
  {
    const uint64_t mg = (static_cast<uint64_t>(prm.rel_magic_hi) << 32) | prm.rel_magic_lo;
    const uint64_t A = __umul64hi(0xFFFFFFFFull, mg) >> prm.rel_shift;
    const int64_t t = (static_cast<int64_t>(A) - static_cast<int64_t>(prm.s_inv)) / 384 - 2 * Tc;
    rel_lthr = t < 0 ? -1 : (t > 0x7FFFFFFF ? 0x7FFFFFFF : static_cast<int32_t>(t));
  }
  uint64_t* tables_bar = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(const_cast<uint32_t*>(recip)) -
                                                     C::kRecip + C::kTmemSlot + 8);
  bool tables_ready = false;
  TileIter<NSEG> ti;
  ti.init(args, blockIdx.x + g * gridDim.x);
  int it0 = 0;
  for (; ti.valid(args); ti.next(args)) {
    const bool live = row < ti.rows;
    const bool warp_live = quarter * 32 < ti.rows;
    for (int j = 0; j < Tc; ++j) {
      const int it = it0 + j;
      named_bar_sync(rc_full_bar(g, it & 1), 256);  // alpha of iteration it published
      const int32_t alpha = lds32(alpha_buf + static_cast<uint32_t>(((it & 1) * 128 + row) * 4));
      named_bar_arrive(rc_free_bar(g, it & 1), 256);  // slot it & 1 consumed
      if (j > 0) {
        corr_wait(gb.o_full(), (it - 1) & 1);
        tc_fence_after();
        if (warp_live && __any_sync(0xffffffffu, alpha != prm.s_inv)) {
          uint32_t lcol;
          uint32_t o[OH];
          tmem_ld1(tO + D, lcol);
          if constexpr (OH == 32) tmem_ld32(tO, *reinterpret_cast<uint32_t(*)[32]>(o));
          else tmem_ld<OH>(tO, o);
          tmem_wait_ld();
          if (__all_sync(0xffffffffu, static_cast<int32_t>(lcol) <= rel_lthr)) {
            const uint32_t bound = 128u * (lcol + 2u * static_cast<uint32_t>(Tc));
            const BiasedRelease br = make_biased_release(alpha, bound, prm, sinv_log2);
#pragma unroll
            for (int h = 0; h < D / OH; ++h) {
              if (h > 0) {
                if constexpr (OH == 32) tmem_ld32(tO + OH * h, *reinterpret_cast<uint32_t(*)[32]>(o));
                else tmem_ld<OH>(tO + OH * h, o);
                tmem_wait_ld();
              }
#pragma unroll
              for (int e = 0; e < OH; ++e) o[e] = br.apply(o[e]);
              tmem_st<OH>(tO + OH * h, o);
            }
            tmem_st1(tO + D, br.apply(lcol));
          } else {
            const int32_t A = release_factor(alpha, prm);
#pragma unroll
            for (int h = 0; h < D / OH; ++h) {
              if (h > 0) {
                if constexpr (OH == 32) tmem_ld32(tO + OH * h, *reinterpret_cast<uint32_t(*)[32]>(o));
                else tmem_ld<OH>(tO + OH * h, o);
                tmem_wait_ld();
              }
#pragma unroll
              for (int e = 0; e < OH; ++e)
                o[e] = static_cast<uint32_t>(scale_release(static_cast<int32_t>(o[e]), alpha, A, prm.s_inv));
              tmem_st<OH>(tO + OH * h, o);
            }
            tmem_st1(tO + D, static_cast<uint32_t>(scale_release(static_cast<int32_t>(lcol), alpha, A, prm.s_inv)));
          }
          tmem_wait_st();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(gb.rel_full());
    }
    // (11) O_i = floor(O / l), saturated (R14), stores
    mbar_wait(gb.o_full(), (it0 + Tc - 1) & 1);
    tc_fence_after();
    if (!tables_ready) {
      mbar_wait(tables_bar, 0);
      tables_ready = true;
    }
    if (warp_live) {
      uint32_t lraw;
      tmem_ld1(tO + D, lraw);
      tmem_wait_ld();
      const int64_t orow = static_cast<int64_t>(ti.problem) * N + ti.off + row;
#pragma unroll
      for (int h = 0; h < D / OH; ++h) {
        uint32_t o[OH];
        if constexpr (OH == 32) tmem_ld32(tO + OH * h, *reinterpret_cast<uint32_t(*)[32]>(o));
        else tmem_ld<OH>(tO + OH * h, o);
        tmem_wait_ld();
        if (live) normalize_store<D, OH, (FQ != 0)>(args, orow, h, o, lraw, recip, __int_as_float(prm.pad[0]));
      }
    }
    it0 += Tc;
  }
}

// ---------------------------------------------------------------- fused-step prologue
// Q0 for the fused step (FQ): every thread of the cooperative grid takes part.
//  1. per-tensor amax over a grid-stride share of Q, K, V (fp32, one FMNMX per
//     element), block reduce, per-CTA partial to global memory; grid barrier;
//  2. every CTA reduces the partials to the same s = fl32(amax / 127) (R2, R3),
//     derives the integer constants (derive_core, the fp64 expression of
//     qflash_derive_params) and the 256-entry dequant table fl32(s_V * i) into
//     shared memory (CTA 0 also publishes scales, constants and table);
//  3. quantizes its share (inputs re-read from L2) with the exact element
//     quantizer of qflash_quant.cu into the int8 buffers the TMA maps point at;
//     proxy fence + grid barrier, after which the attention roles start.
#ifdef QF_FQ_TIMING
// experiment builds: globaltimer stamps of CTA 0 in the workspace (bytes 6144..)
#define QF_FQ_TS_AT(a, k, b, t)                                                            \
  do {                                                                                     \
    if (blockIdx.x == (b) && threadIdx.x == (t))                                           \
      reinterpret_cast<long long*>(reinterpret_cast<char*>((a).prm_out) + 6144)[k] = globaltimer_ns(); \
  } while (0)
#else
#define QF_FQ_TS_AT(a, k, b, t) \
  do {                          \
  } while (0)
#endif
#define QF_FQ_TS(a, k) QF_FQ_TS_AT(a, k, 0, 0)
// per-CTA event ev (1..3) of the timing build: low 32 bits of globaltimer at bytes 6400..8176 (thread 0)
#ifdef QF_FQ_TIMING
#define QF_FQ_CTA(a, ev)                                                                                \
  do {                                                                                                  \
    if (threadIdx.x == 0 && blockIdx.x < 148)                                                           \
      reinterpret_cast<uint32_t*>(reinterpret_cast<char*>((a).prm_out) + 6400)[3 * blockIdx.x + (ev) - 1] = \
          static_cast<uint32_t>(globaltimer_ns());                                                      \
  } while (0)
#else
#define QF_FQ_CTA(a, ev) \
  do {                  \
  } while (0)
#endif
// Source float4 of output vector i (the [P, N, d] layout of tensor t) in the fused step's
// input: the same index for three separate tensors; for a packed QKV projection output
// [P / H, N, 3, H, d] (N2, dynamic quantization of the projection P:L703) the (n, h)
// transpose: problem p = b H + h, row n, lane k4 -> ((b N + n) 3 + t) H d/4 + h d/4 + k4.
template <int D, bool PACKED>
QF_DEV int64_t qkv_src_vec(const AttnArgs& a, int t, int64_t i) {
  constexpr int R = D / 4;  // float4 per row
  constexpr int kShift = D == 32 ? 3 : D == 64 ? 4 : 5;
  if constexpr (!PACKED) return i;
  const uint64_t row = static_cast<uint64_t>(i) >> kShift;  // p N + n
  const int k4 = static_cast<int>(i & (R - 1));
  const uint64_t p = a.N == 1 ? row : __umul64hi(row, a.qkv_n_magic);  // (ceil(2^64 / 1) overflows)
  const uint64_t n = row - p * static_cast<uint64_t>(a.N);
  const uint64_t b = a.qkv_H == 1 ? p : __umul64hi(p, a.qkv_h_magic);
  const uint64_t h = p - b * static_cast<uint64_t>(a.qkv_H);
  return static_cast<int64_t>(((b * a.N + n) * 3 + t) * (static_cast<uint64_t>(a.qkv_H) * R) + h * R + k4);
}

// The fused prologue's grid barrier: hardware cluster barrier for a one-cluster grid, else the
// cooperative-groups grid barrier (an out-of-line copy shared by both call sites was measured
// slower, profiles/r2_experiments.md §11).
static __device__ __forceinline__ void fused_grid_barrier(int cluster_grid) {
  if (cluster_grid) cluster_sync_all();
  else cooperative_groups::this_grid().sync();
}
// Code store of the fused prologue.
__device__ __forceinline__ void stg_code(uint32_t* p, uint32_t w) { *p = w; }
// Quantize one float4 (4 elements) -> 4 packed int8 codes (exact, see qflash_quant_elem.cuh).
// The exact definition, out of line: taken for ~1e-4 of the vectors (x r within 2^-14 of a
// half-integer), so its division sequence is one copy in the binary instead of one per
// unrolled element -- the prologue runs once per launch from a cold instruction cache, and
// the inlined copies made its quantize phase ~46 KB of mostly skipped code (ncu: the
// no_instructions stall led the fused step, profiles/r2_ncu_summary.md).
static __device__ __noinline__ uint32_t quant4_exact(float4 v, float s) {
  return pack4_sat_s8(quant_exact(v.x, s), quant_exact(v.y, s), quant_exact(v.z, s), quant_exact(v.w, s));
}
// Fast path only: `bad` flags a vector whose codes must come from quant4_exact.
__device__ __forceinline__ uint32_t quant4_fast(const float4& v, float r, bool& bad) {
  const int32_t q0 = quant_fast(v.x, r, bad);
  const int32_t q1 = quant_fast(v.y, r, bad);
  const int32_t q2 = quant_fast(v.z, r, bad);
  const int32_t q3 = quant_fast(v.w, r, bad);
  return pack4_sat_s8(q0, q1, q2, q3);
}
__device__ __forceinline__ uint32_t quant4(const float4& v, float s, float r) {
  bool bad = false;
  const uint32_t w = quant4_fast(v, r, bad);
  return bad ? quant4_exact(v, s) : w;
}
__device__ __forceinline__ float amax4(float m, const float4& v) {
  return fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
}

template <int D>
__device__ __forceinline__ void fused_quantize_prologue(const AttnArgs& a, float* scratch,
                                                       IntParams* sprm, uint32_t* dq_table) {

  constexpr int kVR = QF_KVR;  // register-resident 16-B vectors per tensor and thread
  QF_FQ_TS(a, 0);
  // Warp 0 moves no data: its lane 0 derives the integer constants (~1-2 us of
  // fp64 / 64-bit integer work) while warps 1.. quantize, off the critical path.
  const int nthr_blk = blockDim.x;
  const int ndata_blk = nthr_blk - 32;
  const bool data_thread = threadIdx.x >= 32;
  const int64_t nthr = static_cast<int64_t>(gridDim.x) * ndata_blk;
  const int64_t gtid = data_thread ? static_cast<int64_t>(blockIdx.x) * ndata_blk + threadIdx.x - 32
                                   : INT64_MAX / 2;
  const int64_t nvec = a.numel >> 2;
  // external amax (a.amax_in: e.g. MAX-all-reduced over the ranks that shard one
  // logical tensor): no amax pass, no barrier 1
  const bool ext = a.amax_in != nullptr;
  const bool resident = !ext && nvec <= kVR * nthr;  // the whole share stays in registers
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float m[3] = {0.f, 0.f, 0.f};
  float4 reg[3][kVR];
  if (ext) {
    if (threadIdx.x < 3) scratch[96 + threadIdx.x] = __ldcg(a.amax_in + threadIdx.x);
  } else {
  if (resident) {
    // every load of all three tensors in flight before the first reduction (packed
    // QKV input: the same loads with the (token, head) transpose of the addresses);
    // read once (registers keep them for the quantize pass): L2 evict-first
    const uint64_t pol = QF_EVICT_FIRST ? l2_evict_first_policy() : 0ull;
    auto load_all = [&](auto packed) {
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const float4* src = reinterpret_cast<const float4*>(a.xin[t]);
#pragma unroll
        for (int u = 0; u < kVR; ++u) {
          const int64_t i = gtid + u * nthr;
          reg[t][u] = i < nvec ? (QF_EVICT_FIRST ? ldg_stream_ef(src + qkv_src_vec<D, decltype(packed)::value>(a, t, i), pol)
                                                 : ldg_stream(src + qkv_src_vec<D, decltype(packed)::value>(a, t, i)))
                               : make_float4(0.f, 0.f, 0.f, 0.f);  // no L1 allocation
        }
      }
    };
    if (a.qkv_H == 0) load_all(std::false_type{});
    else load_all(std::true_type{});
#pragma unroll
    for (int t = 0; t < 3; ++t)
#pragma unroll
      for (int u = 0; u < kVR; ++u) m[t] = amax4(m[t], reg[t][u]);
  } else {
    auto stream_amax = [&](auto packed) {
      constexpr bool PK = decltype(packed)::value;
      for (int64_t i = gtid; i < nvec; i += 2 * nthr) {  // 6 16-B loads in flight
        float4 v[3][2];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const float4* src = reinterpret_cast<const float4*>(a.xin[t]);
          v[t][0] = __ldg(src + qkv_src_vec<D, PK>(a, t, i));
          v[t][1] = i + nthr < nvec ? __ldg(src + qkv_src_vec<D, PK>(a, t, i + nthr)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int t = 0; t < 3; ++t) m[t] = amax4(amax4(m[t], v[t][0]), v[t][1]);
      }
    };
    if (a.qkv_H == 0) stream_amax(std::false_type{});
    else stream_amax(std::true_type{});
  }
#pragma unroll
  for (int t = 0; t < 3; ++t) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m[t] = fmaxf(m[t], __shfl_xor_sync(0xffffffffu, m[t], o));
    if (lane == 0) scratch[t * 32 + warp] = m[t];
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    float b = 0.f;
    for (int w = 0; w < nthr_blk / 32; ++w) b = fmaxf(b, scratch[threadIdx.x * 32 + w]);
    a.partial[threadIdx.x * gridDim.x + blockIdx.x] = b;
  }
  QF_FQ_TS(a, 1);
#ifdef QF_FQ_TIMING_B1
  __syncthreads();
  QF_FQ_CTA(a, 1);
#endif
  // No per-thread __threadfence: both grid barriers order memory themselves
  // (grid.sync(): bar.sync, then the arriving thread's gpu-scope fence + atomic;
  // barrier.cluster arrive.release / wait.acquire).  Dropping the redundant
  // fences saved ~1 us of the A3 step (profiles/r1_cfg_ab.txt).  A flag barrier
  // (per-CTA tagged slots polled by every CTA, no atomics) was measured slower:
  // 2.8 us vs 1.3 us -- the polling traffic competes with the stragglers' loads.
  fused_grid_barrier(a.cluster_grid);
  QF_FQ_TS(a, 2);
#ifdef QF_FQ_TIMING_B1
  QF_FQ_CTA(a, 2);
#endif
  if (warp < 3) {
    float b = 0.f;
    float pv[5];  // gridDim.x <= 160: every partial load in flight at once
#pragma unroll
    for (int u = 0; u < 5; ++u) {
      const int j = lane + 32 * u;
      pv[u] = j < static_cast<int>(gridDim.x) ? __ldcg(&a.partial[warp * gridDim.x + j]) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 5; ++u) b = fmaxf(b, pv[u]);
    for (int j = lane + 160; j < static_cast<int>(gridDim.x); j += 32) b = fmaxf(b, __ldcg(&a.partial[warp * gridDim.x + j]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
    if (lane == 0) scratch[96 + warp] = b;
  }
  }  // !ext
  // 2. global scales (every CTA, identical): s = fl32(amax / 127), R3 for zeros
  __syncthreads();
  if (threadIdx.x < 3) {
    float sc = __fdiv_rn(scratch[96 + threadIdx.x], 127.0f);
    if (sc == 0.0f) sc = 1.0f / 127.0f;  // all-zero tensor (R3)
    scratch[100 + threadIdx.x] = sc;
  }
  __syncthreads();
  const float s3[3] = {scratch[100], scratch[101], scratch[102]};
#ifdef QF_FQ_TIMING_B1
  QF_FQ_CTA(a, 3);
#endif
  QF_FQ_TS_AT(a, 13, 0, 32);
  // the integer constants (one thread, ~1.3 us of fp64) overlap the quantization
  // of every other warp; the roles read *sprm only after the final __syncthreads
  if (threadIdx.x == 0) {
    IntParams p;
    const int st = derive_core(s3[0], s3[1], D, &p, nullptr);
    if (st != QFLASH_OK) {
      memset(&p, 0, sizeof(p));
      p.status = st;
    }
    p.pad[0] = __float_as_int(s3[2]);  // s_V for the epilogue's y = fl32(s_V O^)
    *sprm = p;
    QF_FQ_TS(a, 3);
    if (blockIdx.x == 0) {
      *a.prm_out = p;
      for (int t = 0; t < 3; ++t) a.scales_out[t] = s3[t];
    }
  } else if (threadIdx.x >= 32 && threadIdx.x < 32 + 256) {
    // dequant table of the epilogue: fl32(s_V * i), i = -128..127
    const int i = static_cast<int>(threadIdx.x) - 32 - 128;
    const uint32_t bits = __float_as_uint(__fmul_rn(s3[2], static_cast<float>(i)));
    dq_table[i + 128] = bits;
    if (blockIdx.x == 0) a.table_out[i + 128] = bits;
  }
  // 3. quantize this thread's share (registers, or an L2-resident re-read with
  // all three tensors' loads in flight per step, as in the amax pass)
  QF_FQ_TS_AT(a, 14, 0, 32);
  // Warp 0 holds no data (its lane 0 derived the constants): a warp-uniform skip, so it
  // reaches the second barrier without issuing the ~540 predicated-off instructions of
  // the unrolled quantize pass after the derivation.
  if (data_thread) {
  float r3[3];
#pragma unroll
  for (int t = 0; t < 3; ++t) r3[t] = __frcp_rn(s3[t]);
  QF_FQ_TS_AT(a, 15, 0, 32);
  if (resident) {
    // fast path for every register-resident vector (stored at once), then the rare
    // flagged vectors again through the out-of-line exact definition
    uint32_t badmask = 0;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      uint32_t* dst = reinterpret_cast<uint32_t*>(a.xq[t]);
#pragma unroll
      for (int u = 0; u < kVR; ++u) {
        const int64_t i = gtid + u * nthr;
        bool bad = false;
        const uint32_t w = quant4_fast(reg[t][u], r3[t], bad);
        if (i < nvec && !QF_NO_CODE_STORE) stg_code(dst + i, w);
        badmask |= (bad && i < nvec) ? (1u << (t * kVR + u)) : 0u;
      }
    }
    QF_FQ_TS_AT(a, 16, 0, 32);
    if (badmask != 0) {
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        uint32_t* dst = reinterpret_cast<uint32_t*>(a.xq[t]);
#pragma unroll
        for (int u = 0; u < kVR; ++u)
          if (badmask & (1u << (t * kVR + u))) dst[gtid + u * nthr] = quant4_exact(reg[t][u], s3[t]);
      }
    }
  } else {
    auto stream_quant = [&](auto packed) {
      constexpr bool PK = decltype(packed)::value;
      for (int64_t i = gtid; i < nvec; i += 2 * nthr) {
        const bool two = i + nthr < nvec;
        float4 v[3][2];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const float4* src = reinterpret_cast<const float4*>(a.xin[t]);
          // the inputs are read-only for the whole launch: the non-coherent path, as the amax
          // pass (measured 0.1-0.2 us per step faster than ld.global.cg, r2_experiments.md §16)
          v[t][0] = __ldg(src + qkv_src_vec<D, PK>(a, t, i));
          v[t][1] = two ? __ldg(src + qkv_src_vec<D, PK>(a, t, i + nthr)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          uint32_t* dst = reinterpret_cast<uint32_t*>(a.xq[t]);
          const uint32_t w0 = quant4(v[t][0], s3[t], r3[t]);
          const uint32_t w1 = quant4(v[t][1], s3[t], r3[t]);
          if (!QF_NO_CODE_STORE) {
            stg_code(dst + i, w0);
            if (two) stg_code(dst + i + nthr, w1);
          } else if ((w0 ^ w1) == 0x5a5a5a5au) {
            dst[i] = 0u;  // keeps the computation live in the timing experiment
          }
        }
      }
    };
    if (a.qkv_H == 0) stream_quant(std::false_type{});
    else stream_quant(std::true_type{});
  }
  }  // data_thread
  // int8 codes (generic-proxy stores) -> TMA loads of other CTAs after the barrier
  QF_FQ_TS(a, 4);
  QF_FQ_TS_AT(a, 6, 0, 32);
  if (QF_PRE_PROXY_FENCE) fence_proxy_async_global();
  QF_FQ_TS_AT(a, 7, 0, 32);
#if defined(QF_FQ_TIMING) && !defined(QF_FQ_TIMING_B1)
  __syncthreads();  // timing build: the stamp marks the CTA's last thread done
  QF_FQ_CTA(a, 1);
#endif
  fused_grid_barrier(a.cluster_grid);
#ifndef QF_FQ_TIMING_B1
  QF_FQ_CTA(a, 2);
#endif
  fence_proxy_async_global();
  QF_FQ_TS(a, 5);
#ifndef QF_FQ_TIMING_B1
  QF_FQ_CTA(a, 3);
#endif
  QF_FQ_TS_AT(a, 10, 0, 32);
}

// ---------------------------------------------------------------- fused per-head prologue
// Q0 with one scale per (tensor, head) for the
// fused per-head step (FQ + PH): the same grid-stride share as the per-tensor prologue,
// but each float4's amax goes to its head h = (vector / (N d/4)) mod H through shared-memory
// atomics, then one global atomicMax per (tensor, head) and CTA; after the grid barrier every
// CTA reads the 3H maxima, forms s = fl32(amax / 127) (R2, R3), derives the H constant sets
// (thread h: derive_core, the fp64 expression of qflash_derive_params) into the shared head
// table and quantizes with its head's scale.  After the second barrier CTA 0 re-zeroes the
// global accumulators for the next launch (the workspace must be zero before the first one).
// head area: [table 96 x 80 B][s 3 x 96][1/s 3 x 96][amax bits 3 x 96]
// Shared-memory max of one float4's amax into its head's slot (h < 0: nothing), aggregated
// over the warp when every lane has the same head (consecutive vectors of one problem): one
// atomic per warp instead of 32.  Called by all 32 lanes.
QF_DEV void ph_amax_add(uint32_t* slots, int h, float m) {
  const int h0 = __shfl_sync(0xffffffffu, h, 0);
  if (__all_sync(0xffffffffu, h == h0)) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && h0 >= 0) atomicMax(&slots[h0], __float_as_uint(m));
  } else if (h >= 0) {
    atomicMax(&slots[h], __float_as_uint(m));
  }
}
template <int D>
__device__ __forceinline__ void fused_quantize_prologue_ph(const AttnArgs& a, IntParams* sprm,
                                                          uint8_t* head_area) {
  constexpr int kVR = QF_KVR;
  IntParams* tab = reinterpret_cast<IntParams*>(head_area);  // stride kHeadPrmStride
  float* s_h = reinterpret_cast<float*>(head_area + kMaxHeads * kHeadPrmStride);
  float* r_h = s_h + 3 * kMaxHeads;
  uint32_t* am_h = reinterpret_cast<uint32_t*>(r_h + 3 * kMaxHeads);
  __shared__ int ph_fast, ph_status;
  const int H = a.H;
  const int ndata_blk = static_cast<int>(blockDim.x) - 32;
  const bool data_thread = threadIdx.x >= 32;
  const int64_t nthr = static_cast<int64_t>(gridDim.x) * ndata_blk;
  const int64_t gtid = data_thread ? static_cast<int64_t>(blockIdx.x) * ndata_blk + threadIdx.x - 32
                                   : INT64_MAX / 2;
  const int64_t nvec = a.numel >> 2;
  const bool resident = nvec <= kVR * nthr;
  auto head_vec = [&](int64_t i) {  // head of float4 vector i (i < 2^32)
    const uint64_t p = a.vp_magic == 0 ? static_cast<uint64_t>(i) : __umul64hi(static_cast<uint64_t>(i), a.vp_magic);
    return head_of(a, static_cast<uint32_t>(p));
  };
  for (int j = threadIdx.x; j < 3 * kMaxHeads; j += blockDim.x) am_h[j] = 0u;
  if (threadIdx.x == 0) {
    ph_fast = 1;
    ph_status = 0;
  }
  __syncthreads();
  float4 reg[3][kVR];
  if (resident) {
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const float4* src = reinterpret_cast<const float4*>(a.xin[t]);
#pragma unroll
      for (int u = 0; u < kVR; ++u) {
        const int64_t i = gtid + u * nthr;
        reg[t][u] = i < nvec ? ldg_stream(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int u = 0; u < kVR; ++u) {
      const int64_t i = gtid + u * nthr;
      const bool ok = i < nvec;
      const int h = ok ? head_vec(i) : -1;
#pragma unroll
      for (int t = 0; t < 3; ++t) ph_amax_add(am_h + t * kMaxHeads, h, ok ? amax4(0.f, reg[t][u]) : 0.f);
    }
  } else {
    // warp-uniform trip count (lanes hold consecutive vectors), so the aggregation's
    // shuffles see the full warp; kVR steps of all three tensors' loads in flight at once
    const int lane = threadIdx.x & 31;
    for (int64_t i0 = gtid; i0 - lane < nvec; i0 += kVR * nthr) {
      float4 v[3][kVR];
#pragma unroll
      for (int u = 0; u < kVR; ++u) {
        const int64_t i = i0 + u * nthr;
#pragma unroll
        for (int t = 0; t < 3; ++t)
          v[t][u] = i < nvec ? __ldg(reinterpret_cast<const float4*>(a.xin[t]) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kVR; ++u) {
        const int64_t i = i0 + u * nthr;
        const int h = i < nvec ? head_vec(i) : -1;
#pragma unroll
        for (int t = 0; t < 3; ++t) ph_amax_add(am_h + t * kMaxHeads, h, amax4(0.f, v[t][u]));
      }
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < 3 * H; j += blockDim.x) {
    const int t = j / H, h = j - t * H;  // (3 H <= 288 entries, once per CTA)
    const uint32_t v = am_h[t * kMaxHeads + h];
    if (v != 0u) atomicMax(&a.ph_amax[j], v);
  }
  if (a.cluster_grid) cluster_sync_all();
  else cooperative_groups::this_grid().sync();
  // scales (every CTA, identical): s = fl32(amax / 127), R3 for an all-zero head
  for (int j = threadIdx.x; j < 3 * H; j += blockDim.x) {
    const int t = j / H, h = j - t * H;
    float sc = __fdiv_rn(__uint_as_float(__ldcg(&a.ph_amax[j])), 127.0f);
    if (sc == 0.0f) sc = 1.0f / 127.0f;
    s_h[t * kMaxHeads + h] = sc;
    r_h[t * kMaxHeads + h] = __frcp_rn(sc);
    if (blockIdx.x == 0) a.scales_out[j] = sc;  // [3][H]: s_q[h], s_k[h], s_v[h]
  }
  __syncthreads();
  // constants of head h (one thread each, in parallel with the quantization below), s_V in
  // the spare word pad[0] for the epilogue's y = fl32(s_V[h] x^)
  if (threadIdx.x < H) {
    const int h = threadIdx.x;
    IntParams p;
    const int st = derive_core(s_h[h], s_h[kMaxHeads + h], D, &p, nullptr);
    if (st != QFLASH_OK) {
      memset(&p, 0, sizeof(p));
      p.status = st;
      atomicCAS(&ph_status, 0, st);
    } else if (!(p.q_shift == 0 && static_cast<uint64_t>(p.s_inv) * static_cast<uint64_t>(p.m_p) < (1ull << 32))) {
      atomicAnd(&ph_fast, 0);
    }
    p.pad[0] = __float_as_int(s_h[2 * kMaxHeads + h]);
    *reinterpret_cast<IntParams*>(reinterpret_cast<char*>(tab) + kHeadPrmStride * h) = p;
    if (blockIdx.x == 0)
      *reinterpret_cast<IntParams*>(reinterpret_cast<char*>(a.prm_out) + kHeadPrmOffset + kHeadPrmStride * h) = p;
  }
  // quantize this thread's share with its heads' scales
  if (resident) {
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      uint32_t* dst = reinterpret_cast<uint32_t*>(a.xq[t]);
#pragma unroll
      for (int u = 0; u < kVR; ++u) {
        const int64_t i = gtid + u * nthr;
        if (i < nvec) {
          const int h = head_vec(i);
          dst[i] = quant4(reg[t][u], s_h[t * kMaxHeads + h], r_h[t * kMaxHeads + h]);
        }
      }
    }
  } else {
    for (int64_t i = gtid; i < nvec; i += 2 * nthr) {  // 6 16-B loads in flight
      const bool two = i + nthr < nvec;
      float4 v[3][2];
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        v[t][0] = __ldcg(reinterpret_cast<const float4*>(a.xin[t]) + i);
        v[t][1] = two ? __ldcg(reinterpret_cast<const float4*>(a.xin[t]) + i + nthr) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      const int h0 = head_vec(i), h1 = two ? head_vec(i + nthr) : 0;
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        uint32_t* dst = reinterpret_cast<uint32_t*>(a.xq[t]);
        dst[i] = quant4(v[t][0], s_h[t * kMaxHeads + h0], r_h[t * kMaxHeads + h0]);
        if (two) dst[i + nthr] = quant4(v[t][1], s_h[t * kMaxHeads + h1], r_h[t * kMaxHeads + h1]);
      }
    }
  }
  __syncthreads();  // the head table and flags are complete
  if (threadIdx.x == 0) {
    // header: status, and whether EVERY head takes the fast quotient path (the kernel
    // picks one softmax instantiation for all heads)
    IntParams hdr;
    memset(&hdr, 0, sizeof(hdr));
    hdr.status = ph_status;
    hdr.q_shift = ph_fast ? 0 : 1;
    hdr.s_inv = 1;
    hdr.m_p = 1;
    hdr.one = 1;
    *sprm = hdr;
    if (blockIdx.x == 0) *a.prm_out = hdr;
  }
  fence_proxy_async_global();
  if (a.cluster_grid) cluster_sync_all();
  else cooperative_groups::this_grid().sync();
  fence_proxy_async_global();
  // every CTA read the accumulators before barrier 2: re-zero them for the next launch
  if (blockIdx.x == 0)
    for (int j = threadIdx.x; j < 3 * H; j += blockDim.x) a.ph_amax[j] = 0u;
}

// ---------------------------------------------------------------- the kernel
template <int D, int BC, int NSEG, int CS, int QT, bool DBG, int FQ = 0, bool PH = false, int VAR = 0>
__global__ void __launch_bounds__(Cfg<D, BC, NSEG, CS, QT>::kThreads, 1)
    qflash_attn_kernel(const __grid_constant__ CUtensorMap tm_q,
                       const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const AttnArgs args) {
  using C = Cfg<D, BC, NSEG, CS, QT>;
  constexpr uint32_t kTmemCols = C::kTmemCols;
  constexpr uint32_t kSwz = swizzle_layout<D>();
  constexpr int kNO = D + 16;  // extended PV width (O columns + ones block)
  constexpr uint32_t kIdescQK = make_idesc_i8(128, BC, 0, 0);
  constexpr uint32_t kIdescPV = make_idesc_i8(128, kNO, 0, 1);
  using Bars = GroupBars<C::kNumS>;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sOnes = smem + C::kOnes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kTmemSlot);
  uint32_t* recip = reinterpret_cast<uint32_t*>(smem + C::kRecip);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0 && blockIdx.x == 0) QF_TS(0);
  if constexpr (FQ) QF_FQ_TS(args, 8);
  if constexpr (DBG) {
    if (threadIdx.x == 0 && args.dbg_t != nullptr) args.dbg_t[128 + 2 * blockIdx.x] = globaltimer_ns();
  }
  const int Tc = args.Tc;

  // ------------------------------------------------------------- setup
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
    for (int g = 0; g < QT; ++g) {
      const Bars gb{bars + g * C::kBarsPerGroup};
      for (int s = 0; s < kMaxStages; ++s) {
        mbar_init(gb.kv_full(s), 1);
        mbar_init(gb.kv_empty(s), 1);
      }
      for (int b = 0; b < 2; ++b) {
        mbar_init(gb.q_full(b), 1);
        mbar_init(gb.q_empty(b), 1);
      }
      for (int b = 0; b < C::kNumS; ++b) mbar_init(gb.s_full(b), 1);
      for (int b = 0; b < 2; ++b) {
        mbar_init(gb.p_full(b), C::kGroupThreads / 32);
      }
      mbar_init(gb.o_full(), 1);
      mbar_init(gb.rel_full(), 4);
      mbar_init(gb.s_empty(), C::kGroupThreads / 32);
    }
    mbar_init(reinterpret_cast<uint64_t*>(smem + C::kTmemSlot + 8), 1);  // step-(11) tables loaded
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, kTmemCols);
    tmem_relinquish();
  }
  // ones block of the extended V operand (any layout: every byte is 1)
  for (int i = threadIdx.x; i < BC * D / 16; i += C::kThreads)
    reinterpret_cast<uint4*>(sOnes)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0 && blockIdx.x == 0) QF_TS(1);
  // Everything above overlaps the tail of the previous kernel (programmatic
  // dependent launch); every global access of this grid comes after the wait.
  // (Moving this setup behind the fused prologue's load issue instead was measured
  // 0.4 us slower per step, profiles/r2_experiments.md.)
  griddep_wait();
  IntParams* sprm = reinterpret_cast<IntParams*>(smem + C::kPrm);
  if constexpr (FQ && PH) {
    fused_quantize_prologue_ph<D>(args, sprm, smem + C::kTotal);
    __syncthreads();
  } else if constexpr (FQ) {
    fused_quantize_prologue<D>(args, reinterpret_cast<float*>(smem + C::kScratch), sprm, recip + 1024);
    __syncthreads();
  }
  const IntParams* dprm = FQ ? sprm : args.dev_prm;  // constants in memory, or nullptr (by value)

  if (warp < 2) {
    // ========================================================= TMA producer of group `warp`
    // Starts before the integer constants are read: the first Q tile and KV
    // stages load while the constants arrive; the device-derived status is
    // checked before the first wait on a consumer (empty) barrier, and an
    // out-of-range launch drains the loads already issued and stops.
    const int g = warp;
    if (g < QT && lane == 0) {
      const Bars gb{bars + g * C::kBarsPerGroup};
      uint8_t* sQ = smem + g * C::kGroupSmem + C::kQ;
      uint8_t* sK = smem + g * C::kGroupSmem + C::kK;
      uint8_t* sV = smem + g * C::kGroupSmem + C::kV;
      int nq = 0, nkv = 0;  // loads issued before the status check
      bool checked = false;
      auto status_ok = [&]() -> bool {
        if (checked) return true;
        checked = true;
        const int st = dprm != nullptr ? *reinterpret_cast<const volatile int32_t*>(&dprm->status)
                                       : args.prm.status;
        if (st == 0) return true;
        for (int b = 0; b < nq; ++b) mbar_wait(gb.q_full(b), 0);
        for (int b = 0; b < nkv; ++b) mbar_wait(gb.kv_full(b), 0);
        return false;
      };
      TileIter<NSEG> ti;
      ti.init(args, blockIdx.x + g * gridDim.x);
      int it = 0;
      bool ok = true;
      for (; ok && ti.valid(args); ti.next(args)) {
        const int qb = ti.i & 1;
        if (ti.i >= 2) {
          if (!(ok = status_ok())) break;
          prod_wait(gb.q_empty(qb), ((ti.i >> 1) - 1) & 1);
        }
        mbar_arrive_expect_tx(gb.q_full(qb), ti.nseg * C::kQBytes);
        // segment s: rows of problem + s land at their tile rows, every other
        // tile row is out of range (row < 0 or >= N) and zero-filled
        for (int s = 0; s < ti.nseg; ++s)
          tma_load_3d(sQ + (qb * NSEG + s) * C::kQBytes, &tm_q, gb.q_full(qb), 0,
                      ti.off - s * args.N, ti.problem + s);
        if (!checked) ++nq;
        for (int j = 0; j < Tc; ++j, ++it) {
          const int st = it % C::kSt;
          if (it >= C::kSt) {
            if (!(ok = status_ok())) break;
            prod_wait(gb.kv_empty(st), ((it / C::kSt) - 1) & 1);
          }
          if (ti.i == 0 && blockIdx.x == 0 && g == 0 && j < 7) QF_TS(5 + 4 * j);
          mbar_arrive_expect_tx(gb.kv_full(st), ti.nseg * 2 * C::kKVBytes);
          for (int s = 0; s < ti.nseg; ++s) {
            tma_load_3d(sK + (st * NSEG + s) * C::kKVBytes, &tm_k, gb.kv_full(st), 0, j * BC,
                        ti.problem + s);
            tma_load_3d(sV + (st * NSEG + s) * C::kKVBytes, &tm_v, gb.kv_full(st), 0, j * BC,
                        ti.problem + s);
          }
          if (!checked) ++nkv;
        }
      }
      if (ok) status_ok();  // a short launch that never waited still drains on error
    }
  }

  // Integer constants (host-derived by value, or device-derived).
  IntParams prm = args.prm;
  if (dprm != nullptr) prm = *dprm;
  const bool run = (prm.status == 0);

  if (run) {
    if (warp < 2) {
      // (producer role above)
    } else if (warp < 4) {
      if (warp == 3) {
        // tables of step (11) -> shared memory, off the critical path (the epilogue waits
        // on the tables mbarrier, long complete by then): the reciprocal table, and for
        // the two-launch form's fused dequantization the quantizer's 256 fp32 patterns
#pragma unroll
        for (int k = 0; k < 8; ++k)
          reinterpret_cast<uint4*>(recip)[lane + 32 * k] = reinterpret_cast<const uint4*>(g_recip.v)[lane + 32 * k];
        if (!FQ && VAR < 2 && args.out_f32 != nullptr) {
          const uint4* src = reinterpret_cast<const uint4*>(args.dq_table);
          reinterpret_cast<uint4*>(recip + 1024)[lane] = src[lane];
          reinterpret_cast<uint4*>(recip + 1024)[lane + 32] = src[lane + 32];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(reinterpret_cast<uint64_t*>(smem + C::kTmemSlot + 8));
      }
      // ========================================================= MMA issuer of group `warp - 2`
      // Issue order within a tile (tcgen05.mma of one thread execute in order,
      // which also orders every TMEM WAR hazard between P V and a later Q K^T):
      //   two S buffers:  QK_0 | QK_1 PV_0 | QK_2 PV_1 | ... | PV_last
      //   one S buffer:   QK_0 | PV_0 QK_1 | PV_1 QK_2 | ... | PV_last
      // The next tile's QK_0 follows PV_last, so the TMA loads and QK_0 of tile
      // i+1 overlap the normalization of tile i.
      const int g = warp - 2;
      if (g < QT && lane == 0) {
        const Bars gb{bars + g * C::kBarsPerGroup};
        const uint32_t tG = tmem_base + g * C::kGroupCols;
        const uint32_t tO = tG + C::kOCol;
        const uint32_t ones_addr = smem_u32(sOnes);
        uint8_t* sQ = smem + g * C::kGroupSmem + C::kQ;
        uint8_t* sK = smem + g * C::kGroupSmem + C::kK;
        uint8_t* sV = smem + g * C::kGroupSmem + C::kV;
        TileIter<NSEG> ti;
        ti.init(args, blockIdx.x + g * gridDim.x);
        for (; ti.valid(args); ti.next(args)) {
          const int qb = ti.i & 1;
          const int nseg = ti.nseg;
          const int it0 = ti.i * Tc;
          mbar_wait(gb.q_full(qb), (ti.i >> 1) & 1);
          tc_fence_after();
          if (ti.i == 0 && blockIdx.x == 0 && g == 0) QF_TS(2);
          auto issue_qk = [&](int j) {
            const int it = it0 + j;
            const int st = it % C::kSt;
            const int sb = (C::kNumS == 2) ? (it & 1) : 0;
            mbar_wait(gb.kv_full(st), (it / C::kSt) & 1);
            if constexpr (C::kSepP) {
              if (it > 0) mbar_wait(gb.s_empty(), (it - 1) & 1);  // S_{it-1} read by every softmax warp
            }
            tc_fence_after();
            if (ti.i == 0 && blockIdx.x == 0 && g == 0 && j < 7) QF_TS(3 + 4 * j);
            // (1) S = sum_s Q_s K_{s,j}^T : M=128, N=BC, K=D in steps of 32 bytes.
            for (int s = 0; s < nseg; ++s) {
              const uint32_t q_addr = smem_u32(sQ + (qb * NSEG + s) * C::kQBytes);
              const uint32_t k_addr = smem_u32(sK + (st * NSEG + s) * C::kKVBytes);
#pragma unroll
              for (int kk = 0; kk < D / 32; ++kk) {
                const uint64_t da = make_smem_desc(q_addr + 32 * kk, 16, 8 * D, kSwz);
                const uint64_t db = make_smem_desc(k_addr + 32 * kk, 16, 8 * D, kSwz);
                mma_i8_ss(tG + sb * BC, da, db, kIdescQK, (s > 0 || kk > 0) ? 1u : 0u);
              }
            }
            mma_commit(gb.s_full(sb));
            if (ti.i == 0 && blockIdx.x == 0 && g == 0 && j < 7) QF_TS(6 + 4 * j);
            if (j == Tc - 1) mma_commit(gb.q_empty(qb));  // last read of this Q tile
          };
          auto issue_pv = [&](int j) {
            const int it = it0 + j;
            const int st = it % C::kSt;
            const int sb = (C::kNumS == 2) ? (it & 1) : 0;
            // (8) O (+)= sum_s P_s [V_{s,j} | 1] : M=128, N=D+16, K=BC in steps of 32 keys.
            if constexpr (C::kRC) {
              mbar_wait(gb.p_full(it & 1), (it >> 1) & 1);
              mbar_wait(gb.rel_full(), it & 1);  // O released / consumed
            } else {
              mbar_wait(gb.p_full(), it & 1);
            }
            tc_fence_after();
            if (ti.i == 0 && blockIdx.x == 0 && g == 0 && j < 7) QF_TS(4 + 4 * j);
            for (int s = 0; s < nseg; ++s) {
              const uint32_t v_addr = smem_u32(sV + (st * NSEG + s) * C::kKVBytes);
#pragma unroll
              for (int kk = 0; kk < BC / 32; ++kk) {
                const uint32_t vk = v_addr + 32 * kk * D;
                const uint64_t db = make_smem_desc(vk, ones_addr - v_addr, 8 * D, kSwz);
                mma_i8_ts(tO, C::kSepP ? tG + C::kPCol + 8 * kk : tG + sb * BC + p_col_k<BC, C::kCW>(kk, s),
                          db, kIdescPV,
                          ((VAR == 0 && j > 0) || s > 0 || kk > 0) ? 1u : 0u);  // ablations: P V_j fresh per tile
              }
            }
            mma_commit(gb.kv_empty(st));
            mma_commit(gb.o_full());
          };
          issue_qk(0);
          for (int j = 0; j < Tc; ++j) {
            if ((C::kNumS == 2 || C::kSepP) && j + 1 < Tc) issue_qk(j + 1);
            issue_pv(j);
            if (C::kNumS == 1 && !C::kSepP && j + 1 < Tc) issue_qk(j + 1);
          }
        }
        // every MMA of this group is issued: let the next grid (dequantize) be
        // scheduled while the last tiles' softmax and normalization finish
        griddep_launch();
      }
    } else {
      const int sw = warp - C::kCtl;
      const int wg = sw >> 2;
      if constexpr (C::kRC) {
        const int g = wg >> 1;
        const Bars gb{bars + g * C::kBarsPerGroup};
        const uint32_t abuf = smem_u32(smem + C::kRed) + static_cast<uint32_t>(g * 2 * 128 * 4);
        const uint32_t tG = tmem_base + g * C::kGroupCols;
        const bool fastq = prm.q_shift == 0 &&
                           static_cast<uint64_t>(prm.s_inv) * static_cast<uint64_t>(prm.m_p) < (1ull << 32);
        if ((wg & 1) == 0) {
          if (fastq) softmax_rc_role<D, BC, NSEG, QT, true>(args, prm, tG, gb, abuf, g, warp & 3, lane);
          else softmax_rc_role<D, BC, NSEG, QT, false>(args, prm, tG, gb, abuf, g, warp & 3, lane);
        } else {
          correction_role<D, BC, NSEG, QT, FQ>(args, prm, tG, gb, abuf, recip, g, warp & 3, lane);
        }
      } else {
      const int g = wg / CS;
      const int c = wg - g * CS;
      const Bars gb{bars + g * C::kBarsPerGroup};
      const uint32_t red_group = smem_u32(smem + C::kRed) + static_cast<uint32_t>(g * 2 * CS * 128 * 4);
      const uint32_t tG = tmem_base + g * C::kGroupCols;
      // per-head constants: the fused step derived them into shared memory, else the table
      // qflash_attention_int8_per_head's derive kernel left in the workspace
      const IntParams* head_tab = (FQ && PH) ? reinterpret_cast<const IntParams*>(smem + C::kTotal) : args.head_prm;
      // (PH: the header's q_shift / s_inv / m_p encode "every head takes the fast path")
      if (prm.q_shift == 0 && static_cast<uint64_t>(prm.s_inv) * static_cast<uint64_t>(prm.m_p) < (1ull << 32))
        softmax_role<D, BC, NSEG, CS, QT, DBG, true, PH, VAR, FQ>(args, prm, tG, gb, red_group, recip, g, c,
                                                                  warp & 3, lane, head_tab);
      else
        softmax_role<D, BC, NSEG, CS, QT, DBG, false, PH, VAR, FQ>(args, prm, tG, gb, red_group, recip, g, c,
                                                                   warp & 3, lane, head_tab);
      }
    }
  }

  // ------------------------------------------------------------- teardown
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0 && blockIdx.x == 0) QF_TS(102);
  if constexpr (FQ) QF_FQ_TS(args, 9);
  if constexpr (FQ) QF_FQ_TS_AT(args, 12, gridDim.x - 1, 0);
  if constexpr (DBG) {
    if (threadIdx.x == 0 && args.dbg_t != nullptr) args.dbg_t[129 + 2 * blockIdx.x] = globaltimer_ns();
  }
  if (warp == 2) tmem_dealloc(tmem_base, kTmemCols);
}

// ----------------------------------------------------------------------------
// Host-side launch (called by the instantiation units).  `tiles` = number of
// work tiles; the persistent grid is G = min(ceil(tiles / QT), SMs) CTAs whose
// group g visits tiles b + g G, b + g G + QT G, ...
template <int D, int BC, int NSEG, int CS, int QT, bool DBG, int FQ = 0, bool PH = false, int VAR = 0>
cudaError_t launch_attn_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                          AttnArgs args, int64_t tiles, int sms, cudaStream_t stream) {
  using C = Cfg<D, BC, NSEG, CS, QT>;
  static_assert(C::kAlloc + ((FQ && PH) ? kHeadAreaBytes : 0) <= 227 * 1024, "shared memory budget");
  static_assert(!PH || CS > 1, "per-head constants: column-split configurations only");
  static_assert(VAR == 0 || (CS > 1 && NSEG == 1 && !FQ && !PH), "ablation variants: cfg 0/1 generic tiles");
  auto kern = qflash_attn_kernel<D, BC, NSEG, CS, QT, DBG, FQ, PH, VAR>;
  constexpr int kSmem = C::kAlloc + ((FQ && PH) ? kHeadAreaBytes : 0);
  static int configured[16] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 16 || !configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 16) configured[dev] = 1;
  }
  const int64_t need = (tiles + QT - 1) / QT;
  const int64_t G = need < sms ? need : sms;
  const int64_t stride = QT * G;  // tiles between consecutive visits of one group
  if (NSEG == 1) {
    const int64_t Tr = args.Tr;
    args.tr_magic = Tr > 1 ? static_cast<uint32_t>(((1ull << 32) + Tr - 1) / Tr) : 0u;
    args.g_div = static_cast<int32_t>(stride / Tr);
    args.g_mod = static_cast<int32_t>((stride % Tr) * kBlockR);
  } else {
    const uint64_t n = static_cast<uint64_t>(args.N);  // N >= 2 here
    args.n_magic = ~0ull / n + 1ull;  // ceil(2^64 / N): floor(x / N) = hi64(x * n_magic), x < 2^32
    const int64_t step = stride * kBlockR;
    args.g_div = static_cast<int32_t>(step / args.N);
    args.g_mod = static_cast<int32_t>(step % args.N);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(G));
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = kSmem;

  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  if constexpr (FQ) {
    // small grids (<= 8 CTAs portable; up to 16 where the GPU schedules it): launch
    // the grid as ONE thread-block cluster -- its
    // CTAs are co-scheduled and barrier.cluster (hardware) replaces the two grid
    // barriers of the quantize prologue; falls back to the cooperative launch
    static int cluster_env = -2;
    if (cluster_env == -2) {
      const char* env = getenv("QFLASH_FUSED_CLUSTER");
      cluster_env = (env != nullptr && env[0] == '0') ? 0 : 1;
    }
    if (cluster_env && G <= 16) {
      static int nonportable[16] = {0};
      if (G > 8 && dev >= 0 && dev < 16 && !nonportable[dev]) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess)
          nonportable[dev] = 1;
      }
      cudaLaunchAttribute ca[2];
      ca[0].id = cudaLaunchAttributeClusterDimension;
      ca[0].val.clusterDim.x = static_cast<unsigned>(G);
      ca[0].val.clusterDim.y = 1;
      ca[0].val.clusterDim.z = 1;
      // programmatic serialization as for the cooperative form: the next step's setup
      // overlaps this one's tail (griddep_wait precedes every global access)
      ca[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      ca[1].val.programmaticStreamSerializationAllowed = 1;
      cudaLaunchConfig_t ccfg = cfg;
      ccfg.attrs = ca;
      ccfg.numAttrs = (pdl_mask() & 8) ? 2 : 1;
      AttnArgs cargs = args;
      cargs.cluster_grid = 1;
      const cudaError_t ce = cudaLaunchKernelEx(&ccfg, kern, tq, tk, tv, cargs);
      if (ce == cudaSuccess) return cudaSuccess;
      (void)cudaGetLastError();
      if (getenv("QFLASH_DEBUG_LAUNCH") != nullptr) {
        int nclusters = -1;
        ccfg.numAttrs = 1;
        cudaOccupancyMaxActiveClusters(&nclusters, kern, &ccfg);
        (void)cudaGetLastError();
        fprintf(stderr, "qflash: %d-CTA cluster launch failed (%s); max active clusters %d\n",
                static_cast<int>(G), cudaGetErrorString(ce), nclusters);
        ccfg.numAttrs = (pdl_mask() & 8) ? 2 : 1;
      }
      if (ccfg.numAttrs == 2) {  // without PDL
        ccfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&ccfg, kern, tq, tk, tv, cargs) == cudaSuccess) return cudaSuccess;
        (void)cudaGetLastError();
      }
      // cluster shape not schedulable here: cooperative launch
    }
    // fused step: grid barriers in the quantize prologue need every CTA resident;
    // programmatic serialization lets the next step's grid be launched (and run its
    // setup) while this one drains -- griddep_wait() precedes every global access
    cudaLaunchAttribute a2[2];
    a2[0].id = cudaLaunchAttributeCooperative;
    a2[0].val.cooperative = 1;
    a2[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a2[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = a2;
    cfg.numAttrs = (pdl_mask() & 8) ? 2 : 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, args);
    if (e != cudaSuccess && cfg.numAttrs == 2) {
      (void)cudaGetLastError();
      cfg.numAttrs = 1;
      e = cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, args);
    }
    return e;
  } else {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (griddep_wait)
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (pdl_mask() & 1) ? 1 : 0;
  }
  return cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, args);
}

#undef QF_TS

}  // namespace qf
