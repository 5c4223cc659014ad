// qflash_attention.cu -- the fused integer-only attention kernel (Algorithm 1 of
// arxiv 2604.25306) for B200 / sm_100a.
//
// One CTA owns one 128-row query tile at a time (B_r = 128 = the tcgen05 M;
// TMEM lane r = tile row r) and walks its tiles persistently.  Warp roles:
//   warp 0       TMA producer: Q tile(s), K_j / V_j through a 2-stage ring
//   warp 1       MMA issuer:   S_j = Q K_j^T   (tcgen05.mma kind::i8, SS, s32 in TMEM)
//                              O  += P_j V_j   (kind::i8, TS: P from TMEM, V MN-major)
//   warp 2 / 1   TMEM allocator, reciprocal-table loader
//   softmax      integer softmax in kNWG warpgroups, thread = (query row, a
//                column chunk): rowmax (Eq. 4, combined through shared memory),
//                ShiftExp2 (Alg. 2, division-free exact quotient), requantization
//                (Eq. 10), ScaleRelease of O and l (Eq. 14), normalization (11).
// The row sum l (Eq. 11) is produced by the tensor core: V is extended with a
// block of ones (N = d + 16), so TMEM column d of the O accumulator holds
// floor-released l exactly as the oracle defines it.
//
// Tiling (NSEG template parameter):
//   NSEG = 1  "generic": tile = (problem, 128-row query block); T_r tiles per
//             problem, the last one ragged.
//   NSEG > 1  "row-packed": the query rows of all problems are flattened and cut
//             into 128-row tiles, so a tile spans up to NSEG consecutive problems
//             (segments).  Segment s gets its own Q tile, loaded by TMA with row
//             coordinates shifted by -s N so that rows of other problems fall out
//             of range and are zero-filled; S = sum_s Q_s K_{s,j}^T then holds every
//             row's score against its OWN problem's keys in one accumulator.  P is
//             written once per segment (the thread's own segment gets its P, the
//             others zeros), and O = sum_s P_s [V_{s,j} | 1] again accumulates
//             each row against its own values.  A3 (N = 197) at batch 8 becomes
//             148 tiles (one per SM) instead of 192; Swin windows (N = 49) pack
//             2.6 per tile instead of 2.
//
// No floating-point instruction is executed (integer-only audit in tests).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"
#include "qflash_common.cuh"

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
__device__ const RecipTable g_recip = make_recip_table();


constexpr int kStages = 2;
constexpr int kBlockR = 128;

// Bring-up timeline: clock64() stamps (callers restrict to CTA 0, first tile).
#define QF_TS(slot)                                                               \
  do {                                                                            \
    if (args.dbg_t != nullptr && (slot) < 128)                                    \
      args.dbg_t[(slot)] = clock64();                                             \
  } while (0)

template <int D, int BC, int NSEG>
struct SmemLayout {
  static constexpr int kQBytes = kBlockR * D;
  static constexpr int kKVBytes = BC * D;
  static constexpr int kOnesBytes = BC * D;  // second MN atom of the extended V
  static constexpr int kQ = 0;                                  // [2][NSEG] Q tiles
  static constexpr int kK = kQ + 2 * NSEG * kQBytes;            // [kStages][NSEG]
  static constexpr int kV = kK + kStages * NSEG * kKVBytes;     // [kStages][NSEG]
  static constexpr int kOnes = kV + kStages * NSEG * kKVBytes;
  static constexpr int kBar = kOnes + kOnesBytes;
  static constexpr int kNumBars = 2 * kStages + 8;
  static constexpr int kTmemSlot = kBar + kNumBars * 8;
  static constexpr int kRed = kTmemSlot + 16;           // [2][kNWG<=4][128] int32 row maxima
  static constexpr int kRecip = kRed + 2 * 4 * 128 * 4;  // [1024] u32 reciprocal table
  static constexpr int kTotal = kRecip + 1024 * 4;
  static constexpr int kAlloc = kTotal + 1024;  // slack for 1024-B alignment
};

__host__ __device__ constexpr uint32_t tmem_cols_pow2(int cols) {
  return cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
}

template <int D>
__host__ __device__ constexpr uint32_t swizzle_layout() {
  return D == 32 ? 6u : D == 64 ? 4u : 2u;  // UMMA layout: SW32 / SW64 / SW128
}

// ---------------------------------------------------------------- the math

// ShiftExp2 + requantization of one score (steps 5-6 for one element).
//   d1 = m + s_inv - S  (>= s_inv),  q1 = floor(d1 / s_inv) = q + 1  (exact magic)
//   y  = (q1 s_inv + S + s_inv - m) >> q1  ==  ((r >> 1) + s_inv) >> q   (Alg. 2)
//   P  = floor(y M_P / 2^r_P)                                            (Eq. 10)
// Instruction mix per element: 2 IADD3 + SHF (ALU pipe), 2 IMAD.HI + IMAD (FMA
// pipe); `m` is the row maximum, `nm` = -m.
// ALT = true computes u = S + (s_inv - m) with IMAD (FMA pipe) instead of IADD3
// (ALU pipe); alternating the two forms balances the pipes (ALU 4.5 / FMA 4.5
// issue slots per element).
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
    // y M_P < 2^32 (host-checked: s_inv M_P < 2^32): IMAD.lo + SHF instead of
    // the half-rate IMAD.HI.
    return static_cast<int32_t>((y * static_cast<uint32_t>(p.m_p)) >> p.r_p);
  } else {
    y <<= p.p_pre;
    return static_cast<int32_t>(umulhi(y, p.p_mul));
  }
}

// alpha = ShiftExp2(m_old - m_new) (step 4) -- same formula, x = m_old - m_new.
template <bool FASTQ>
QF_DEV int32_t shift_exp2(int32_t x, const IntParams& p) {
  const uint32_t d1 = static_cast<uint32_t>(p.s_inv - x);  // -x + s_inv
  uint32_t q1 = umulhi(d1, p.q_magic);
  if constexpr (!FASTQ) q1 >>= p.q_shift;
  const uint32_t num = q1 * static_cast<uint32_t>(p.s_inv) + static_cast<uint32_t>(x + p.s_inv);
  return static_cast<int32_t>(shr_clamp(num, q1));
}

// A = min(floor(alpha 2^31 / s_inv), 2^31 - 1): per-row constant of the release.
QF_DEV int32_t release_factor(int32_t alpha, const IntParams& p) {
  const uint64_t n = static_cast<uint64_t>(alpha) << 31;
  const uint64_t mg = (static_cast<uint64_t>(p.rel_magic_hi) << 32) | p.rel_magic_lo;
  uint64_t a = __umul64hi(n, mg) >> p.rel_shift;
  if (a > 0x7FFFFFFFull) a = 0x7FFFFFFFull;
  return static_cast<int32_t>(a);
}

// A_f = floor(alpha 2^32 / s_inv) (mod 2^32; alpha = s_inv rows are passed through).
QF_DEV uint32_t release_factor32(int32_t alpha, const IntParams& p) {
  const uint64_t n = static_cast<uint64_t>(alpha) << 32;  // < 2^56
  const uint64_t mg = (static_cast<uint64_t>(p.rel_magic_hi) << 32) | p.rel_magic_lo;
  return static_cast<uint32_t>(__umul64hi(n, mg) >> p.rel_shift);
}

// Fast exact ScaleRelease (2 instructions per element).  With a per-row bound
// |X| <= bound and (2 bound + s_inv) s_inv < 2^32, pick B = floor(bound/s_inv) + 1
// so X' = X + B s_inv >= 1; since B s_inv alpha / s_inv = B alpha is an integer,
//   floor(X alpha / s_inv) = floor(X' alpha / s_inv) - B alpha
//                          = hi(X' * A_c) - B alpha,   A_c = floor(alpha 2^32 / s_inv) + 1,
// exact because X' s_inv < 2^32 keeps the ceiling error below 1/s_inv (the
// fractional part of X' alpha / s_inv is a multiple of 1/s_inv).  alpha = s_inv rows
// (identity) use A = 2^32 - 1: hi(X' (2^32 - 1)) = X' - 1, corrected by +1.
// Per element: IADD3 (X + B s_inv), IMAD.HI, IADD3 (+ addend): ALU 2, FMA 1.
struct BiasedRelease {
  uint32_t bias;    // B s_inv
  uint32_t mul;     // A_c (or 2^32 - 1 for identity rows)
  uint32_t add;     // -B alpha (+1 for identity rows)
  uint32_t zero;    // runtime 0: keeps the final add a separate ALU IADD3 (ptxas would
                    // otherwise fold it into IMAD.HI's 64-bit addend pair + 2 IMAD.MOV)
  QF_DEV uint32_t apply(uint32_t X) const {
    return iadd3(__umulhi(iadd3(X, bias, zero), mul), add, zero);
  }
};
QF_DEV BiasedRelease make_biased_release(int32_t alpha, uint32_t bound, const IntParams& p) {
  const uint64_t mg = (static_cast<uint64_t>(p.rel_magic_hi) << 32) | p.rel_magic_lo;
  const uint32_t B = static_cast<uint32_t>(__umul64hi(bound, mg) >> p.rel_shift) + 1u;  // floor(bound/s_inv)+1
  const bool ident = alpha == p.s_inv;
  BiasedRelease r;
  r.bias = B * static_cast<uint32_t>(p.s_inv);
  r.mul = ident ? 0xFFFFFFFFu : release_factor32(alpha, p) + 1u;
  r.add = (0u - B * static_cast<uint32_t>(alpha)) + (ident ? 1u : 0u);
  r.zero = static_cast<uint32_t>(p.zero);
  return r;
}

// ScaleRelease of one accumulator element: floor(X alpha / s_inv) exactly
// (Eq. 14 realised per P:L408, reading R10).  q0 = floor(X A / 2^31) is within
// one of the answer; the remainder X alpha - q0 s_inv (exact mod 2^32, true
// value in [-s_inv, 2 s_inv)) corrects it.
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
  const int32_t k = __clz(l);                       // l >= 2  =>  1 <= k <= 30
  const uint32_t ln = static_cast<uint32_t>(l) << k;  // [2^31, 2^32)
  Recip r;
  r.R = static_cast<int32_t>(table[(ln >> 21) & 1023u]);
  r.sh = 30 - k;
  r.l = l;
  return r;
}
// q0 = floor(O R / 2^(62-k)) is within one of floor(O / l) whenever |O / l| < 2^11;
// `bad` flags the (theoretical) rest for an exact slow pass.
QF_DEV int32_t floor_div(int32_t O, const Recip& r, bool& bad) {
  int32_t q0 = __mulhi(O, r.R) >> r.sh;
  const int32_t rem = O - q0 * r.l;
  q0 += (rem >= r.l) ? 1 : 0;
  q0 += rem >> 31;  // -1 if rem < 0
  bad |= (rem >= 2 * r.l) | (rem < -r.l);
  return q0;
}
QF_DEV int32_t floor_div_exact(int32_t O, int32_t l) {
  int32_t q = 0;  // long division by repeated doubling (integer only, rare path)
  int64_t n = O, d = l;
  int64_t qq = 0, acc = 0;
  const bool neg = n < 0;
  uint64_t un = neg ? static_cast<uint64_t>(-(n + 1)) : static_cast<uint64_t>(n);
#pragma unroll 1
  for (int b = 31; b >= 0; --b) {
    acc = (acc << 1) | static_cast<int64_t>((un >> b) & 1u);
    if (acc >= d) { acc -= d; qq |= (1ll << b); }
  }
  q = static_cast<int32_t>(neg ? ~qq : qq);  // floor(O/l) = ~floor(~O/l) for O < 0
  return q;
}

// ---------------------------------------------------------------- configuration
// Warps 0..kCtl-1: control (TMA producer, MMA issuer, TMEM allocator, table
// loader); then kNWG softmax warpgroups.  Softmax warp w handles TMEM lane
// quarter (w & 3), i.e. tile rows 32*(w&3) .. +31 (thread = row); its warpgroup
// g owns key columns [g*CW, (g+1)*CW) of every S tile and O columns
// [g*D/kNWG, (g+1)*D/kNWG) for the release and the normalization.  The row
// maximum is combined across warpgroups through shared memory (one named
// barrier per KV tile).
// MODE 0: one CTA per SM, 4 softmax warpgroups, 4 control warps.
// MODE 1: two CTAs per SM when TMEM allows, 2 softmax warpgroups, 2 control warps.
template <int D, int BC, int NSEG, int MODE>
struct Cfg {
  static constexpr int kNWG = MODE == 1 ? 2 : 4;          // softmax warpgroups
  static constexpr int kCtl = MODE == 0 ? 4 : 2;          // control warps
  static constexpr int kSoftThreads = 128 * kNWG;
  static constexpr int kThreads = 32 * kCtl + kSoftThreads;
  static constexpr int kCW = BC / kNWG;                   // key columns per thread
  static constexpr int kOW = D / kNWG;                    // O columns per thread
  static constexpr int kChunk = kCW < 32 ? kCW : 32;
  static constexpr bool kSInRegs = kCW == kChunk;
  static constexpr int kAllocWarp = kCtl == 4 ? 2 : 1;    // TMEM allocator
  static constexpr int kTableWarp = kCtl == 4 ? 3 : 1;    // reciprocal-table loader
  // TMEM: kNumS S buffers of BC columns (the P_s of tile j alias S buffer j:
  // segment s at columns [s BC/4, (s+1) BC/4)), then O (D columns) + l (column
  // D) + 15 copies of l from the ones block.
  static constexpr int kMinBlocks = (MODE != 0 && BC + D + 16 <= 256) ? 2 : 1;
  static constexpr int kTmemBudget = kMinBlocks == 2 ? 256 : 512;
  static constexpr int kNumS = (2 * BC + D + 16 <= kTmemBudget) ? 2 : 1;
  static constexpr uint32_t kTmemO = kNumS * BC;
  static constexpr uint32_t kTmemCols = tmem_cols_pow2(kNumS * BC + D + 16);
  static_assert(NSEG * (BC / 4) <= BC, "P segments must fit in one S buffer");
};

// Persistent tile iterator (identical in every role); no runtime division
// (integer-only kernel): the host supplies the magics and the grid-stride
// quotient/remainder.
//   generic (NSEG = 1): tile t = problem * T_r + qt, rows [128 qt, 128 qt + 128).
//   row-packed:         tile t = flattened rows [128 t, 128 t + 128) of [P N].
// Either way the tile starts at row `off` of problem `problem` and tile row r is
// flattened row problem * N + off + r.
template <int NSEG>
struct TileIter {
  int problem;  // first problem of the tile
  int off;      // row of tile row 0 inside `problem`
  int rows;     // live tile rows [0, rows)
  int nseg;     // problems the tile spans (1..NSEG)
  int i;        // tiles visited by this CTA
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
  __device__ void init(const AttnArgs& a) {
    i = 0;
    const uint32_t t = blockIdx.x;
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

// ---------------------------------------------------------------- softmax role
template <int D, int BC, int NSEG, int MODE, bool FASTQ>
__device__ __forceinline__ void softmax_role(const AttnArgs& args, const IntParams& prm,
                                             uint32_t tmem_base, uint64_t* bar_s_full,
                                             uint64_t* bar_p_full, uint64_t* bar_o_full,
                                             int32_t* red, const uint32_t* recip, int warp,
                                             int lane) {
  using C = Cfg<D, BC, NSEG, MODE>;
  constexpr int CW = C::kCW;
  constexpr int OW = C::kOW;
  const int N = args.N;
  const int Tc = args.Tc;
  const int g = (warp - C::kCtl) >> 2;  // warpgroup
  const int quarter = warp & 3;
  const int row = quarter * 32 + lane;  // TMEM lane == tile row
  const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
  const uint32_t tS0 = tmem_base + lane_off;  // S buffer b at + b * BC
  const uint32_t tO = tmem_base + lane_off + C::kTmemO;
  const int c0 = g * CW;  // first key column of this thread
  const bool dbg_cta = blockIdx.x == 0;

  TileIter<NSEG> ti;
  ti.init(args);
  for (; ti.valid(args); ti.next(args)) {
    const bool dbg = dbg_cta && ti.i == 0;
    const bool live = row < ti.rows;              // padded rows of the last tile do no work
    const bool warp_live = quarter * 32 < ti.rows;
    int seg = 0;                                  // this row's problem = ti.problem + seg
    if constexpr (NSEG > 1) {
      const int x = ti.off + row;
      seg = (x >= N ? 1 : 0);
      if constexpr (NSEG > 2) seg += (x >= 2 * N ? 1 : 0) + (x >= 3 * N ? 1 : 0);
    }
    const int nseg = ti.nseg;
    int32_t m = -(1 << 21);  // m^(0) = -2^21
    const int it0 = ti.i * Tc;

    for (int j = 0; j < Tc; ++j) {
      const int it = it0 + j;
      const int sb = (C::kNumS == 2) ? (it & 1) : 0;
      const uint32_t tS = tS0 + sb * BC;
      mbar_wait(&bar_s_full[sb], (C::kNumS == 2 ? (it >> 1) : it) & 1);
      tc_fence_after();
      if (dbg && warp == C::kCtl && lane == 0 && j < 7) QF_TS(40 + 8 * j);
      // columns of this thread that exist in KV tile j (ragged last tile, R16)
      const int valid = min(BC, N - j * BC) - c0;
      constexpr int CK = C::kChunk;
      uint32_t s[C::kSInRegs ? CW : CK];
      int32_t tmax = INT32_MIN;
      if (warp_live && valid > 0) {
        if constexpr (C::kSInRegs) {
          tmem_ld<CW>(tS + c0, s);
          tmem_wait_ld();
          if (args.dbg_s != nullptr && dbg && j == 0) {
            for (int e = 0; e < CW; ++e) args.dbg_s[row * BC + c0 + e] = static_cast<int32_t>(s[e]);
          }
          if (valid >= CW) {
#pragma unroll
            for (int e = 0; e < CW; ++e) tmax = max(tmax, static_cast<int32_t>(s[e]));
          } else {
#pragma unroll
            for (int e = 0; e < CW; ++e)
              if (e < valid) tmax = max(tmax, static_cast<int32_t>(s[e]));
          }
        } else {
#pragma unroll
          for (int ch = 0; ch < CW / CK; ++ch) {
            tmem_ld<CK>(tS + c0 + CK * ch, s);
            tmem_wait_ld();
            if (args.dbg_s != nullptr && dbg && j == 0) {
              for (int e = 0; e < CK; ++e) args.dbg_s[row * BC + c0 + CK * ch + e] = static_cast<int32_t>(s[e]);
            }
#pragma unroll
            for (int e = 0; e < CK; ++e)
              if (CK * ch + e < valid) tmax = max(tmax, static_cast<int32_t>(s[e]));
          }
        }
      }
      // (2)(3) combine the partial maxima of the kNWG warpgroups
      {
        int32_t* rb = red + (it & 1) * (C::kNWG * 128);
        rb[g * 128 + row] = tmax;
        named_bar_sync(1, C::kSoftThreads);
        if (dbg && warp == C::kCtl && lane == 0 && j < 7) QF_TS(41 + 8 * j);
#pragma unroll
        for (int h = 0; h < C::kNWG; ++h) tmax = max(tmax, rb[h * 128 + row]);
      }
      const int32_t m_new = max(m, tmax);
      // (4) alpha = ShiftExp2(m_old - m_new)
      const int32_t alpha = shift_exp2<FASTQ>(m - m_new, prm);
      if (dbg && warp == C::kCtl && lane == 0 && j < 7) QF_TS(42 + 8 * j);

      // (5)(6) P = Requant(ShiftExp2(S - m_new)), 4 x int8 per TMEM column.
      const uint32_t mu = static_cast<uint32_t>(m_new);
      const uint32_t nmu = static_cast<uint32_t>(-m_new);
      const uint32_t c3 = static_cast<uint32_t>(prm.s_inv - m_new);
      const uint32_t one = static_cast<uint32_t>(prm.one);
      uint32_t pk[CW / 4];
      if (warp_live && valid > 0) {
        if constexpr (C::kSInRegs) {
          if (valid >= CW) {
#pragma unroll
            for (int e = 0; e < CW; e += 4)
              pk[e / 4] = pack4_sat_s8(
                  shift_exp2_requant<FASTQ, false>(static_cast<int32_t>(s[e]), mu, nmu, c3, one, prm),
                  shift_exp2_requant<FASTQ, true>(static_cast<int32_t>(s[e + 1]), mu, nmu, c3, one, prm),
                  shift_exp2_requant<FASTQ, false>(static_cast<int32_t>(s[e + 2]), mu, nmu, c3, one, prm),
                  shift_exp2_requant<FASTQ, true>(static_cast<int32_t>(s[e + 3]), mu, nmu, c3, one, prm));
          } else {
#pragma unroll
            for (int e = 0; e < CW; e += 4) {
              int32_t pv[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int32_t x = shift_exp2_requant<FASTQ, false>(static_cast<int32_t>(s[e + u]), mu, nmu, c3, one, prm);
                pv[u] = (e + u < valid) ? x : 0;
              }
              pk[e / 4] = pack4_sat_s8(pv[0], pv[1], pv[2], pv[3]);
            }
          }
        } else {
#pragma unroll
          for (int ch = 0; ch < CW / CK; ++ch) {
            tmem_ld<CK>(tS + c0 + CK * ch, s);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < CK; e += 4) {
              int32_t pv[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int32_t x = shift_exp2_requant<FASTQ, false>(static_cast<int32_t>(s[e + u]), mu, nmu, c3, one, prm);
                pv[u] = (CK * ch + e + u < valid) ? x : 0;
              }
              pk[(CK * ch + e) / 4] = pack4_sat_s8(pv[0], pv[1], pv[2], pv[3]);
            }
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < CW / 4; ++e) pk[e] = 0u;
      }
      // P_s columns [s BC/4 + c0/4, +CW/4) alias S columns of this buffer: every
      // S read of this tile must be complete.  With S in registers the
      // max-exchange barrier above already ordered them; otherwise synchronize again.
      if constexpr (!C::kSInRegs) named_bar_sync(1, C::kSoftThreads);
      if (nseg == 1) {
        tmem_st<CW / 4>(tS + (c0 >> 2), pk);
      } else {
        // segment s gets this row's P if the row belongs to it, zeros otherwise
        // (rows of dead lanes have pk = 0 already)
#pragma unroll
        for (int sg = 0; sg < NSEG; ++sg) {
          if (sg < nseg) {
            uint32_t z[CW / 4];
#pragma unroll
            for (int e = 0; e < CW / 4; ++e) z[e] = (seg == sg && live) ? pk[e] : 0u;
            tmem_st<CW / 4>(tS + sg * (BC / 4) + (c0 >> 2), z);
          }
        }
      }
      if (dbg && warp == C::kCtl && lane == 0 && j < 7) QF_TS(44 + 8 * j);

      // (7)(8) ScaleRelease of O (this group's columns) and l (group 0) once
      // PV_{j-1} has landed -- after P_j so that PV_{j-1} completes behind the P
      // computation; skipped for j = 0 (O = l = 0) and for warps whose rows all
      // kept their maximum (alpha = s_inv is the identity, R10).  PV_j is only
      // issued after every warp's p_full arrival below, i.e. after the release.
      if (j > 0) {
        mbar_wait(bar_o_full, (it - 1) & 1);
        tc_fence_after();
        if (dbg && warp == C::kCtl && lane == 0 && j < 7) QF_TS(45 + 8 * j);
        if (warp_live && __any_sync(0xffffffffu, alpha != prm.s_inv)) {
          uint32_t o[OW];
          tmem_ld<OW>(tO + g * OW, o);
          uint32_t lcol;
          tmem_ld1(tO + D, lcol);
          tmem_wait_ld();
          if (dbg && warp == C::kCtl && lane == 0 && j < 7) QF_TS(46 + 8 * j);
          // Fast exact path when every row of the warp satisfies |X| s_inv < 2^32
          // for all its accumulators X (bound |O| <= 128 (l + 2 T_c), DESIGN.md
          // "Kernel arithmetic"): floor(X alpha / s_inv) is then the high word of
          // X * ceil/floor(alpha 2^32 / s_inv) with no correction.
          const uint64_t bound = 128ull * (static_cast<uint64_t>(lcol) + 2ull * Tc);
          const uint64_t D64 = static_cast<uint64_t>(prm.s_inv);
          if (__all_sync(0xffffffffu, (2ull * bound + D64) * D64 < (1ull << 32))) {
            const BiasedRelease br = make_biased_release(alpha, static_cast<uint32_t>(bound), prm);
#pragma unroll
            for (int e = 0; e < OW; ++e) o[e] = br.apply(o[e]);
            tmem_st<OW>(tO + g * OW, o);
            if (g == 0) tmem_st1(tO + D, br.apply(lcol));
          } else {
            const int32_t A = release_factor(alpha, prm);
#pragma unroll
            for (int e = 0; e < OW; ++e)
              o[e] = static_cast<uint32_t>(scale_release(static_cast<int32_t>(o[e]), alpha, A, prm.s_inv));
            tmem_st<OW>(tO + g * OW, o);
            if (g == 0) {
              lcol = static_cast<uint32_t>(scale_release(static_cast<int32_t>(lcol), alpha, A, prm.s_inv));
              tmem_st1(tO + D, lcol);
            }
          }
          if (dbg && warp == C::kCtl && lane == 0 && j < 7) QF_TS(47 + 8 * j);
        }
      }

      tmem_wait_st();
      if (args.dbg_p != nullptr && dbg && j == 0) {
        named_bar_sync(1, C::kSoftThreads);
        if (g == 0) {
          for (int w = 0; w < BC / 4; w += 8) {
            uint32_t pw[8];
            tmem_ld8(tS + w, pw);
            tmem_wait_ld();
            for (int e = 0; e < 8; ++e) args.dbg_p[row * (BC / 4) + w + e] = static_cast<int32_t>(pw[e]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_p_full);
      if (dbg && warp == C::kCtl && lane == 0 && j < 7) QF_TS(43 + 8 * j);
      m = m_new;
    }

    // (11) O_i = floor(O / l), saturated to int8 (R14); this group's O columns.
    mbar_wait(bar_o_full, (it0 + Tc - 1) & 1);
    tc_fence_after();
    if (dbg && warp == C::kCtl && lane == 0) QF_TS(100);
    if (ti.i == 0) named_bar_sync(2, C::kSoftThreads + 32);  // reciprocal table ready
    if (warp_live) {
      uint32_t lraw;
      uint32_t o[OW];
      tmem_ld1(tO + D, lraw);
      tmem_ld<OW>(tO + g * OW, o);
      tmem_wait_ld();
      if (args.dbg_o != nullptr && dbg) {
        for (int e = 0; e < OW; ++e) args.dbg_o[row * (D + 1) + g * OW + e] = static_cast<int32_t>(o[e]);
        if (g == 0) args.dbg_o[row * (D + 1) + D] = static_cast<int32_t>(lraw);
      }
      if (live) {
        const Recip rc = make_recip(static_cast<int32_t>(lraw), recip);
        int32_t qv[OW];
        bool bad = false;
#pragma unroll
        for (int e = 0; e < OW; ++e) qv[e] = floor_div(static_cast<int32_t>(o[e]), rc, bad);
        if (bad) {
#pragma unroll
          for (int e = 0; e < OW; ++e) qv[e] = floor_div_exact(static_cast<int32_t>(o[e]), rc.l);
        }
        uint32_t w[OW / 4];
#pragma unroll
        for (int e = 0; e < OW; e += 4) w[e / 4] = pack4_sat_s8(qv[e], qv[e + 1], qv[e + 2], qv[e + 3]);
        // flattened output row problem * N + off + row (row-packed tiles included)
        int8_t* dst = args.out + (static_cast<int64_t>(ti.problem) * N + ti.off + row) * D + g * OW;
        if constexpr (OW == 8) {
          *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
        } else {
#pragma unroll
          for (int e = 0; e < OW / 16; ++e)
            reinterpret_cast<uint4*>(dst)[e] = make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
        }
      }
    }
    if (dbg && warp == C::kCtl && lane == 0) QF_TS(101);
    // The O/l loads above completed (wait::ld) before this thread's next p_full
    // arrival, so the next tile's first PV (which overwrites O) cannot race them.
  }
}

// ---------------------------------------------------------------- the kernel
template <int D, int BC, int NSEG, int MODE>
__global__ void __launch_bounds__(Cfg<D, BC, NSEG, MODE>::kThreads, Cfg<D, BC, NSEG, MODE>::kMinBlocks)
    qflash_attn_kernel(const __grid_constant__ CUtensorMap tm_q,
                       const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const AttnArgs args) {
  using L = SmemLayout<D, BC, NSEG>;
  using C = Cfg<D, BC, NSEG, MODE>;
  constexpr uint32_t kTmemCols = C::kTmemCols;
  constexpr uint32_t kSwz = swizzle_layout<D>();
  constexpr int kNO = D + 16;  // extended PV width (O columns + ones block)
  constexpr uint32_t kIdescQK = make_idesc_i8(128, BC, 0, 0);
  constexpr uint32_t kIdescPV = make_idesc_i8(128, kNO, 0, 1);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem + L::kQ;  // [2][NSEG]
  uint8_t* sK = smem + L::kK;  // [kStages][NSEG]
  uint8_t* sV = smem + L::kV;  // [kStages][NSEG]
  uint8_t* sOnes = smem + L::kOnes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* bar_kv_full = bars;              // [kStages]
  uint64_t* bar_kv_empty = bars + kStages;   // [kStages]
  uint64_t* bar_q_full = bars + 2 * kStages;  // [2]
  uint64_t* bar_q_empty = bar_q_full + 2;     // [2]
  uint64_t* bar_s_full = bar_q_full + 4;      // [2]
  uint64_t* bar_p_full = bar_q_full + 6;
  uint64_t* bar_o_full = bar_q_full + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlot);
  int32_t* red = reinterpret_cast<int32_t*>(smem + L::kRed);
  uint32_t* recip = reinterpret_cast<uint32_t*>(smem + L::kRecip);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0 && blockIdx.x == 0) QF_TS(0);
  const int Tc = args.Tc;

  // ------------------------------------------------------------- setup
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bar_kv_full[s], 1);
      mbar_init(&bar_kv_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_q_full[b], 1);
      mbar_init(&bar_q_empty[b], 1);
      mbar_init(&bar_s_full[b], 1);
    }
    mbar_init(bar_p_full, C::kSoftThreads / 32);
    mbar_init(bar_o_full, 1);
    fence_barrier_init();
  }
  if (warp == C::kAllocWarp) {
    tmem_alloc(tmem_slot, kTmemCols);
    tmem_relinquish();
  }
  // ones block of the extended V operand (any layout: every byte is 1)
  for (int i = threadIdx.x; i < L::kOnesBytes / 16; i += C::kThreads)
    reinterpret_cast<uint4*>(sOnes)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0 && blockIdx.x == 0) QF_TS(1);
  // Everything above overlaps the tail of the previous kernel (programmatic
  // dependent launch); every global access of this grid comes after the wait.
  griddep_wait();

  // Integer constants (host-derived by value, or device-derived).
  IntParams prm = args.prm;
  if (args.dev_prm != nullptr) prm = *args.dev_prm;
  const bool run = (prm.status == 0);

  if (run) {
    if (warp == C::kTableWarp) {
      // reciprocal table for step (11) -> shared memory, off the critical path:
      // the softmax warps sync on named barrier 2 before their first normalization.
      for (int i = lane; i < 1024; i += 32) recip[i] = g_recip.v[i];
      __threadfence_block();
      named_bar_arrive(2, C::kSoftThreads + 32);
    }
    if (warp == 0) {
      // ========================================================= TMA producer
      if (lane == 0) {
        TileIter<NSEG> ti;
        ti.init(args);
        int it = 0;
        for (; ti.valid(args); ti.next(args)) {
          const int qb = ti.i & 1;
          if (ti.i >= 2) mbar_wait(&bar_q_empty[qb], ((ti.i >> 1) - 1) & 1);
          mbar_arrive_expect_tx(&bar_q_full[qb], ti.nseg * L::kQBytes);
          // segment s: rows of problem + s land at their tile rows, every other
          // tile row is out of range (row < 0 or >= N) and zero-filled
          for (int s = 0; s < ti.nseg; ++s)
            tma_load_3d(sQ + (qb * NSEG + s) * L::kQBytes, &tm_q, &bar_q_full[qb], 0,
                        ti.off - s * args.N, ti.problem + s);
          for (int j = 0; j < Tc; ++j, ++it) {
            const int st = it % kStages;
            if (it >= kStages) mbar_wait(&bar_kv_empty[st], ((it / kStages) - 1) & 1);
            mbar_arrive_expect_tx(&bar_kv_full[st], ti.nseg * 2 * L::kKVBytes);
            for (int s = 0; s < ti.nseg; ++s) {
              tma_load_3d(sK + (st * NSEG + s) * L::kKVBytes, &tm_k, &bar_kv_full[st], 0, j * BC,
                          ti.problem + s);
              tma_load_3d(sV + (st * NSEG + s) * L::kKVBytes, &tm_v, &bar_kv_full[st], 0, j * BC,
                          ti.problem + s);
            }
          }
        }
      }
    } else if (warp == 1) {
      // ========================================================= MMA issuer
      // Issue order within a tile (tcgen05.mma of one thread execute in order,
      // which also orders every TMEM WAR hazard between PV and a later QK):
      //   two S buffers:  QK_0 | QK_1 PV_0 | QK_2 PV_1 | ... | PV_last
      //   one S buffer:   QK_0 | PV_0 QK_1 | PV_1 QK_2 | ... | PV_last
      // The next tile's QK_0 follows PV_last, so the TMA loads and QK_0 of tile
      // i+1 overlap the normalization of tile i.
      if (lane == 0) {
        const uint32_t tO = tmem_base + C::kTmemO;
        const uint32_t ones_addr = smem_u32(sOnes);
        TileIter<NSEG> ti;
        ti.init(args);
        for (; ti.valid(args); ti.next(args)) {
          const int qb = ti.i & 1;
          const int nseg = ti.nseg;
          const int it0 = ti.i * Tc;
          mbar_wait(&bar_q_full[qb], (ti.i >> 1) & 1);
          tc_fence_after();
          if (ti.i == 0 && blockIdx.x == 0) QF_TS(2);
          auto issue_qk = [&](int j) {
            const int it = it0 + j;
            const int st = it % kStages;
            const int sb = (C::kNumS == 2) ? (it & 1) : 0;
            mbar_wait(&bar_kv_full[st], (it / kStages) & 1);
            tc_fence_after();
            if (ti.i == 0 && blockIdx.x == 0 && j < 7) QF_TS(3 + 4 * j);
            // (1) S = sum_s Q_s K_{s,j}^T : M=128, N=BC, K=D in steps of 32 bytes.
            for (int s = 0; s < nseg; ++s) {
              const uint32_t q_addr = smem_u32(sQ + (qb * NSEG + s) * L::kQBytes);
              const uint32_t k_addr = smem_u32(sK + (st * NSEG + s) * L::kKVBytes);
#pragma unroll
              for (int kk = 0; kk < D / 32; ++kk) {
                const uint64_t da = make_smem_desc(q_addr + 32 * kk, 16, 8 * D, kSwz);
                const uint64_t db = make_smem_desc(k_addr + 32 * kk, 16, 8 * D, kSwz);
                mma_i8_ss(tmem_base + sb * BC, da, db, kIdescQK, (s > 0 || kk > 0) ? 1u : 0u);
              }
            }
            mma_commit(&bar_s_full[sb]);
            if (j == Tc - 1) mma_commit(&bar_q_empty[qb]);  // last read of this Q tile
          };
          auto issue_pv = [&](int j) {
            const int it = it0 + j;
            const int st = it % kStages;
            const int sb = (C::kNumS == 2) ? (it & 1) : 0;
            // (8) O (+)= sum_s P_s [V_{s,j} | 1] : M=128, N=D+16, K=BC in steps of 32 keys.
            mbar_wait(bar_p_full, it & 1);
            tc_fence_after();
            if (ti.i == 0 && blockIdx.x == 0 && j < 7) QF_TS(4 + 4 * j);
            for (int s = 0; s < nseg; ++s) {
              const uint32_t v_addr = smem_u32(sV + (st * NSEG + s) * L::kKVBytes);
#pragma unroll
              for (int kk = 0; kk < BC / 32; ++kk) {
                const uint32_t vk = v_addr + 32 * kk * D;
                const uint64_t db = make_smem_desc(vk, ones_addr - v_addr, 8 * D, kSwz);
                mma_i8_ts(tO, tmem_base + sb * BC + s * (BC / 4) + 8 * kk, db, kIdescPV,
                          (j > 0 || s > 0 || kk > 0) ? 1u : 0u);
              }
            }
            mma_commit(&bar_kv_empty[st]);
            mma_commit(bar_o_full);
          };
          issue_qk(0);
          for (int j = 0; j < Tc; ++j) {
            if (C::kNumS == 2 && j + 1 < Tc) issue_qk(j + 1);
            issue_pv(j);
            if (C::kNumS == 1 && j + 1 < Tc) issue_qk(j + 1);
          }
        }
        // every MMA of this CTA is issued: let the next grid (dequantize) be
        // scheduled while the last tile's softmax and normalization finish
        griddep_launch();
      }
    } else if (warp >= C::kCtl) {
      if (prm.q_shift == 0 && static_cast<uint64_t>(prm.s_inv) * static_cast<uint64_t>(prm.m_p) < (1ull << 32))
        softmax_role<D, BC, NSEG, MODE, true>(args, prm, tmem_base, bar_s_full, bar_p_full,
                                              bar_o_full, red, recip, warp, lane);
      else
        softmax_role<D, BC, NSEG, MODE, false>(args, prm, tmem_base, bar_s_full, bar_p_full,
                                               bar_o_full, red, recip, warp, lane);
    }
  }

  // ------------------------------------------------------------- teardown
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0 && blockIdx.x == 0) QF_TS(102);
  if (warp == C::kAllocWarp) tmem_dealloc(tmem_base, kTmemCols);
}

// ----------------------------------------------------------------------------
// Host-side launch helpers (called by qflash_host.cu).  `tiles` = number of work
// tiles; the persistent grid is min(tiles, CTAs-per-SM x SMs).
template <int D, int BC, int NSEG, int MODE>
cudaError_t launch_attn_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                          AttnArgs args, int64_t tiles, int sms, cudaStream_t stream) {
  using L = SmemLayout<D, BC, NSEG>;
  using C = Cfg<D, BC, NSEG, MODE>;
  static_assert(L::kAlloc <= 227 * 1024, "shared memory budget");
  auto kern = qflash_attn_kernel<D, BC, NSEG, MODE>;
  static int configured[16] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 16 || !configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kAlloc);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 16) configured[dev] = 1;
  }
  const int64_t cap = static_cast<int64_t>(C::kMinBlocks) * sms;
  const int64_t G = tiles < cap ? tiles : cap;
  if (NSEG == 1) {
    const int64_t Tr = args.Tr;
    args.tr_magic = Tr > 1 ? static_cast<uint32_t>(((1ull << 32) + Tr - 1) / Tr) : 0u;
    args.g_div = static_cast<int32_t>(G / Tr);
    args.g_mod = static_cast<int32_t>((G % Tr) * kBlockR);
  } else {
    const uint64_t n = static_cast<uint64_t>(args.N);  // N >= 2 here
    args.n_magic = ~0ull / n + 1ull;  // ceil(2^64 / N): floor(x / N) = hi64(x * n_magic), x < 2^32
    const int64_t step = G * kBlockR;
    args.g_div = static_cast<int32_t>(step / args.N);
    args.g_mod = static_cast<int32_t>(step % args.N);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(G));
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = L::kAlloc;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (griddep_wait)
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl_mask() & 1) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, args);
}

// Supported instantiations (qflash_host.cu selects within them):
//   NSEG 1: D in {32, 64, 128} x BC in {64, 128, 256}
//   NSEG 2: D in {32, 64} x BC in {64, 128, 256}, D = 128 x BC in {64, 128}
//   NSEG 4: D in {32, 64} x BC in {64, 128}
bool attention_config_supported(int D, int BC, int nseg) {
  if (D != 32 && D != 64 && D != 128) return false;
  if (BC != 64 && BC != 128 && BC != 256) return false;
  if (nseg == 1) return true;
  if (nseg == 2) return D != 128 || BC != 256;
  if (nseg == 4) return D != 128 && BC != 256;
  return false;
}

template <int MODE>
static cudaError_t launch_attention_mode(int D, int BC, int nseg, const CUtensorMap& tq,
                                        const CUtensorMap& tk, const CUtensorMap& tv,
                                        const AttnArgs& args, int64_t tiles, int sms,
                                        cudaStream_t stream) {
#define QF_CASE(d, bc, ns)                     \
  if (D == d && BC == bc && nseg == ns)        \
    return launch_attn_t<d, bc, ns, MODE>(tq, tk, tv, args, tiles, sms, stream);
  QF_CASE(32, 64, 1) QF_CASE(32, 128, 1) QF_CASE(32, 256, 1)
  QF_CASE(64, 64, 1) QF_CASE(64, 128, 1) QF_CASE(64, 256, 1)
  QF_CASE(128, 64, 1) QF_CASE(128, 128, 1) QF_CASE(128, 256, 1)
  QF_CASE(32, 64, 2) QF_CASE(32, 128, 2) QF_CASE(32, 256, 2)
  QF_CASE(64, 64, 2) QF_CASE(64, 128, 2) QF_CASE(64, 256, 2)
  QF_CASE(128, 64, 2) QF_CASE(128, 128, 2)
  QF_CASE(32, 64, 4) QF_CASE(32, 128, 4)
  QF_CASE(64, 64, 4) QF_CASE(64, 128, 4)
#undef QF_CASE
  return cudaErrorInvalidValue;
}

cudaError_t launch_attention(int D, int BC, int nseg, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, const AttnArgs& args, int64_t tiles, int sms,
                             int mode, cudaStream_t stream) {
  if (mode == 1) return launch_attention_mode<1>(D, BC, nseg, tq, tk, tv, args, tiles, sms, stream);
  return launch_attention_mode<0>(D, BC, nseg, tq, tk, tv, args, tiles, sms, stream);
}

}  // namespace qf
