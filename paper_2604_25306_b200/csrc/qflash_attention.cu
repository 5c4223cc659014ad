// qflash_attention.cu -- the fused integer-only attention kernel (Algorithm 1 of
// arxiv 2604.25306) for B200 / sm_100a.
//
// One CTA owns one 128-row query tile (B_r = 128 = the tcgen05 M; TMEM lane r =
// query row r).  Warp roles (256 threads):
//   warp 0      TMA producer: Q tile once, K_j / V_j through a 2-stage ring
//   warp 1      MMA issuer:   S_j = Q K_j^T   (tcgen05.mma kind::i8, SS, s32 in TMEM)
//                             O  += P_j V_j   (kind::i8, TS: P from TMEM, V MN-major)
//   warp 2      TMEM allocator
//   warps 4..7  integer softmax, thread = query row: rowmax (Eq. 4), ShiftExp2
//               (Alg. 2, division-free exact quotient), requantization (Eq. 10),
//               ScaleRelease of O and l (Eq. 14), normalization (step 11).
// The row sum l (Eq. 11) is produced by the tensor core: V is extended with a
// block of ones (N = d + 16), so TMEM column d of the O accumulator holds
// floor-released l exactly as the oracle defines it.
//
// PACKED (the Swin-window variant, N <= 64): a 128-row tile holds two problems
// (windows) at rows 0-63 / 64-127 and the KV tile holds their 2 x 64 keys;
// each thread only evaluates its own window's diagonal block and writes P = 0
// elsewhere, so P V never mixes windows.  T_c = 1.
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

constexpr int kThreads = 256;
constexpr int kSoftmaxWarp0 = 4;
constexpr int kStages = 2;
constexpr int kBlockR = 128;

template <int D, int BC>
struct SmemLayout {
  static constexpr int kQBytes = kBlockR * D;
  static constexpr int kKVBytes = BC * D;
  static constexpr int kOnesBytes = BC * D;  // second MN atom of the extended V
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kQBytes;
  static constexpr int kV = kK + kStages * kKVBytes;
  static constexpr int kOnes = kV + kStages * kKVBytes;
  static constexpr int kBar = kOnes + kOnesBytes;
  static constexpr int kNumBars = 2 * kStages + 4;
  static constexpr int kTmemSlot = kBar + kNumBars * 8;
  static constexpr int kTotal = kTmemSlot + 16;
  static constexpr int kAlloc = kTotal + 1024;  // slack for 1024-B alignment
};

__host__ __device__ constexpr uint32_t tmem_cols_for(int BC, int D) {
  return (BC + D + 16) <= 32    ? 32
         : (BC + D + 16) <= 64  ? 64
         : (BC + D + 16) <= 128 ? 128
         : (BC + D + 16) <= 256 ? 256
                                : 512;
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
template <bool FASTQ>
QF_DEV int32_t shift_exp2_requant(int32_t S, uint32_t c2, int32_t c3, const IntParams& p) {
  const uint32_t d1 = c2 - static_cast<uint32_t>(S);
  uint32_t q1 = umulhi(d1, p.q_magic);
  if constexpr (!FASTQ) q1 >>= p.q_shift;
  const uint32_t num = q1 * static_cast<uint32_t>(p.s_inv) + static_cast<uint32_t>(S + c3);
  uint32_t y = shr_clamp(num, q1);
  if constexpr (!FASTQ) y <<= p.p_pre;
  return static_cast<int32_t>(umulhi(y, p.p_mul));
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

// ScaleRelease of one accumulator element: floor(X alpha / s_inv) exactly
// (Eq. 14 realised per P:L408, reading R10).  q0 = floor(X A / 2^31) is within
// one of the answer; the remainder X alpha - q0 s_inv (exact mod 2^32, true
// value in [-s_inv, 2 s_inv)) corrects it.
QF_DEV int32_t scale_release(int32_t X, int32_t alpha, int32_t A, int32_t s_inv) {
  const int64_t t = static_cast<int64_t>(X) * static_cast<int64_t>(A);
  int32_t q0 = static_cast<int32_t>(t >> 31);
  const int32_t rem = X * alpha - q0 * s_inv;
  q0 += (rem >= s_inv) ? 1 : 0;
  q0 -= (rem < 0) ? 1 : 0;
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
QF_DEV Recip make_recip(int32_t l) {
  const int32_t k = __clz(l);                       // l >= 2  =>  1 <= k <= 30
  const uint32_t ln = static_cast<uint32_t>(l) << k;  // [2^31, 2^32)
  Recip r;
  r.R = static_cast<int32_t>(g_recip.v[(ln >> 21) & 1023u]);
  r.sh = 30 - k;
  r.l = l;
  return r;
}
QF_DEV int32_t floor_div(int32_t O, const Recip& r) {
  int32_t q0 = __mulhi(O, r.R) >> r.sh;
  const int32_t rem = O - q0 * r.l;
  q0 += (rem >= r.l) ? 1 : 0;
  q0 -= (rem < 0) ? 1 : 0;
  return q0;
}

// Softmax/epilogue role (warps 4..7): thread = query row = TMEM lane.
template <int D, int BC, bool PACKED, bool FASTQ>
__device__ __forceinline__ void softmax_rows(const AttnArgs& args, const IntParams& prm,
                                             uint32_t tmem_base, uint64_t* bar_s_full,
                                             uint64_t* bar_p_full, uint64_t* bar_o_full,
                                             int problem, int q0, int warp, int lane) {
  constexpr uint32_t kTmemS = 0;
  constexpr uint32_t kTmemO = BC;
  const int N = args.N;
  const int Tc = PACKED ? 1 : args.Tc;

  // ========================================================= softmax rows
  const int quarter = warp & 3;
  const int row = quarter * 32 + lane;  // TMEM lane == tile row
  const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
  const uint32_t tS = tmem_base + lane_off + kTmemS;
  const uint32_t tO = tmem_base + lane_off + kTmemO;
  // packed: this row's window occupies key columns [col0, col0 + 64)
  const int col0 = PACKED ? (row >> 6) * 64 : 0;
  constexpr int kCols = PACKED ? 64 : BC;  // columns this thread evaluates
  int32_t m = -(1 << 21);                  // m^(0) = -2^21

  for (int j = 0; j < Tc; ++j) {
    mbar_wait(bar_s_full, j & 1);
    tc_fence_after();
    const int valid = PACKED ? N : min(BC, N - j * BC);  // ragged last tile (R16)

    // (2)(3) row max over the valid columns
    int32_t tmax = INT32_MIN;
#pragma unroll
    for (int ch = 0; ch < kCols / 32; ++ch) {
      uint32_t s[32];
      tmem_ld32(tS + col0 + ch * 32, s);
      tmem_wait_ld();
      if (args.dbg_s != nullptr && j == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
#pragma unroll
        for (int e = 0; e < 32; ++e) args.dbg_s[row * BC + col0 + ch * 32 + e] = static_cast<int32_t>(s[e]);
      }
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const int c = ch * 32 + e;
        if (c < valid) tmax = max(tmax, static_cast<int32_t>(s[e]));
      }
    }
    const int32_t m_new = max(m, tmax);
    // (4) alpha = ShiftExp2(m_old - m_new)
    const int32_t alpha = shift_exp2<FASTQ>(m - m_new, prm);

    // (7)(8) ScaleRelease of O and l once PV_{j-1} has landed (skip j = 0:
    // O = l = 0; skip warps whose rows all keep their max: alpha = s_inv).
    if (j > 0) {
      mbar_wait(bar_o_full, (j - 1) & 1);
      tc_fence_after();
      if (__any_sync(0xffffffffu, alpha != prm.s_inv)) {
        const int32_t A = release_factor(alpha, prm);
#pragma unroll
        for (int ch = 0; ch < D / 32; ++ch) {
          uint32_t o[32];
          tmem_ld32(tO + ch * 32, o);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e)
            o[e] = static_cast<uint32_t>(
                scale_release(static_cast<int32_t>(o[e]), alpha, A, prm.s_inv));
          tmem_st32(tO + ch * 32, o);
        }
        uint32_t lcol;
        tmem_ld1(tO + D, lcol);
        tmem_wait_ld();
        lcol = static_cast<uint32_t>(scale_release(static_cast<int32_t>(lcol), alpha, A, prm.s_inv));
        tmem_st1(tO + D, lcol);
      }
    }

    // (5)(6) P = Requant(ShiftExp2(S - m_new)), packed 4 x int8 per column.
    const uint32_t c2 = static_cast<uint32_t>(m_new + prm.s_inv);
    const int32_t c3 = prm.s_inv - m_new;
    if constexpr (PACKED) {
      // own window: 64 columns -> 16 packed words at P column (col0 / 4)
      uint32_t pk[16];
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        uint32_t s[32];
        tmem_ld32(tS + col0 + ch * 32, s);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          int32_t pv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = ch * 32 + e + u;
            const int32_t pval = shift_exp2_requant<FASTQ>(static_cast<int32_t>(s[e + u]), c2, c3, prm);
            pv[u] = (c < valid) ? pval : 0;
          }
          pk[ch * 8 + e / 4] = pack4_sat_s8(pv[0], pv[1], pv[2], pv[3]);
        }
      }
      uint32_t zero[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) zero[i] = 0u;
      // P occupies columns [0, 32): own half from pk, the other window's half zero
      tmem_st16(tS + (col0 >> 2), pk);
      tmem_st16(tS + ((64 - col0) >> 2), zero);
    } else {
#pragma unroll
      for (int ch = 0; ch < BC / 32; ++ch) {
        uint32_t s[32];
        tmem_ld32(tS + ch * 32, s);
        tmem_wait_ld();
        uint32_t pk[8];
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          int32_t pv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = ch * 32 + e + u;
            const int32_t pval = shift_exp2_requant<FASTQ>(static_cast<int32_t>(s[e + u]), c2, c3, prm);
            pv[u] = (c < valid) ? pval : 0;
          }
          pk[e / 4] = pack4_sat_s8(pv[0], pv[1], pv[2], pv[3]);
        }
        // P chunk ch -> P columns [8 ch, 8 ch + 8) (aliases S columns already read)
        tmem_st8(tS + ch * 8, pk);
      }
    }
    tmem_wait_st();
    if (args.dbg_p != nullptr && j == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
      for (int w = 0; w < BC / 4; w += 8) {
        uint32_t pw[8];
        tmem_ld8(tS + w, pw);
        tmem_wait_ld();
        for (int e = 0; e < 8; ++e) args.dbg_p[row * (BC / 4) + w + e] = static_cast<int32_t>(pw[e]);
      }
    }
    tc_fence_before();
    mbar_arrive(bar_p_full);
    m = m_new;
  }

  // (11) O_i = floor(O / l), saturated to int8; write the row.
  mbar_wait(bar_o_full, (Tc - 1) & 1);
  tc_fence_after();
  uint32_t lraw;
  tmem_ld1(tO + D, lraw);
  tmem_wait_ld();
  const Recip rc = make_recip(static_cast<int32_t>(lraw));
  if (args.dbg_o != nullptr && blockIdx.x == 0 && blockIdx.y == 0) {
    for (int c = 0; c < D; c += 8) {
      uint32_t ow[8];
      tmem_ld8(tO + c, ow);
      tmem_wait_ld();
      for (int e = 0; e < 8; ++e) args.dbg_o[row * (D + 1) + c + e] = static_cast<int32_t>(ow[e]);
    }
    args.dbg_o[row * (D + 1) + D] = static_cast<int32_t>(lraw);
  }
  int out_row;
  bool row_ok;
  int out_problem;
  if constexpr (PACKED) {
    out_problem = problem + (row >> 6);
    out_row = row & 63;
    row_ok = (out_row < N) && (out_problem < args.P);
  } else {
    out_problem = problem;
    out_row = q0 + row;
    row_ok = out_row < N;
  }
  int8_t* dst = args.out + (static_cast<int64_t>(out_problem) * N + out_row) * D;
#pragma unroll
  for (int ch = 0; ch < D / 32; ++ch) {
    uint32_t o[32];
    tmem_ld32(tO + ch * 32, o);
    tmem_wait_ld();
    uint32_t w[8];
#pragma unroll
    for (int e = 0; e < 32; e += 4)
      w[e / 4] = pack4_sat_s8(floor_div(static_cast<int32_t>(o[e]), rc),
                              floor_div(static_cast<int32_t>(o[e + 1]), rc),
                              floor_div(static_cast<int32_t>(o[e + 2]), rc),
                              floor_div(static_cast<int32_t>(o[e + 3]), rc));
    if (row_ok) {
      uint4* d4 = reinterpret_cast<uint4*>(dst + ch * 32);
      d4[0] = make_uint4(w[0], w[1], w[2], w[3]);
      d4[1] = make_uint4(w[4], w[5], w[6], w[7]);
    }
  }
}

// ---------------------------------------------------------------- the kernel
template <int D, int BC, bool PACKED>
__global__ void __launch_bounds__(kThreads, 1)
    qflash_attn_kernel(const __grid_constant__ CUtensorMap tm_q,
                       const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const AttnArgs args) {
  using L = SmemLayout<D, BC>;
  constexpr uint32_t kTmemCols = tmem_cols_for(BC, D);
  static_assert(kTmemCols >= BC + D + 16, "TMEM budget");
  constexpr uint32_t kSwz = swizzle_layout<D>();
  constexpr int kNO = D + 16;  // extended PV width (O columns + ones block)
  constexpr uint32_t kIdescQK = make_idesc_i8(128, BC, 0, 0);
  constexpr uint32_t kIdescPV = make_idesc_i8(128, kNO, 0, 1);
  constexpr uint32_t kTmemS = 0;    // S_j (BC cols, s32); P_j (BC/4 cols, int8 x4) aliases it
  constexpr uint32_t kTmemO = BC;   // O accumulator (D cols) + l (col D) + 15 copies of l

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem + L::kQ;
  uint8_t* sK = smem + L::kK;
  uint8_t* sV = smem + L::kV;
  uint8_t* sOnes = smem + L::kOnes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* bar_kv_full = bars;              // [kStages]
  uint64_t* bar_kv_empty = bars + kStages;   // [kStages]
  uint64_t* bar_q_full = bars + 2 * kStages;
  uint64_t* bar_s_full = bar_q_full + 1;
  uint64_t* bar_p_full = bar_q_full + 2;
  uint64_t* bar_o_full = bar_q_full + 3;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlot);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // Work item: generic -> (problem, query tile) = (blockIdx.x, blockIdx.y);
  // packed -> problems 2*blockIdx.x and 2*blockIdx.x + 1.
  const int Tc = PACKED ? 1 : args.Tc;
  const int problem = PACKED ? 2 * blockIdx.x : blockIdx.x;
  const int q0 = PACKED ? 0 : blockIdx.y * kBlockR;

  // ------------------------------------------------------------- setup
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bar_kv_full[s], 1);
      mbar_init(&bar_kv_empty[s], 1);
    }
    mbar_init(bar_q_full, 1);
    mbar_init(bar_s_full, 1);
    mbar_init(bar_p_full, 128);
    mbar_init(bar_o_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, kTmemCols);
    tmem_relinquish();
  }
  // ones block of the extended V operand (any layout: every byte is 1)
  for (int i = threadIdx.x; i < L::kOnesBytes / 16; i += kThreads)
    reinterpret_cast<uint4*>(sOnes)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // Integer constants (host-derived by value, or device-derived).
  IntParams prm = args.prm;
  if (args.dev_prm != nullptr) prm = *args.dev_prm;
  const bool run = (prm.status == 0);

  if (run) {
    if (warp == 0) {
      // ========================================================= TMA producer
      if (lane == 0) {
        mbar_arrive_expect_tx(bar_q_full, L::kQBytes);
        if constexpr (PACKED)
          tma_load_3d(sQ, &tm_q, bar_q_full, 0, 0, problem);  // box {D, 64, 2}
        else
          tma_load_3d(sQ, &tm_q, bar_q_full, 0, q0, problem);  // box {D, 128, 1}
        for (int j = 0; j < Tc; ++j) {
          const int st = j % kStages;
          if (j >= kStages) mbar_wait(&bar_kv_empty[st], ((j / kStages) - 1) & 1);
          mbar_arrive_expect_tx(&bar_kv_full[st], 2 * L::kKVBytes);
          const int kv_row = PACKED ? 0 : j * BC;
          tma_load_3d(sK + st * L::kKVBytes, &tm_k, &bar_kv_full[st], 0, kv_row, problem);
          tma_load_3d(sV + st * L::kKVBytes, &tm_v, &bar_kv_full[st], 0, kv_row, problem);
        }
      }
    } else if (warp == 1) {
      // ========================================================= MMA issuer
      if (lane == 0) {
        const uint32_t tS = tmem_base + kTmemS;
        const uint32_t tO = tmem_base + kTmemO;
        const uint32_t q_addr = smem_u32(sQ);
        const uint32_t ones_addr = smem_u32(sOnes);
        mbar_wait(bar_q_full, 0);
        tc_fence_after();
        for (int j = 0; j < Tc; ++j) {
          const int st = j % kStages;
          mbar_wait(&bar_kv_full[st], (j / kStages) & 1);
          if (j > 0) mbar_wait(bar_o_full, (j - 1) & 1);  // P_{j-1} consumed: S free
          tc_fence_after();
          const uint32_t k_addr = smem_u32(sK + st * L::kKVBytes);
          const uint32_t v_addr = smem_u32(sV + st * L::kKVBytes);
          // (1) S = Q K_j^T : M=128, N=BC, K=D in steps of 32 bytes.
#pragma unroll
          for (int kk = 0; kk < D / 32; ++kk) {
            const uint64_t da = make_smem_desc(q_addr + 32 * kk, 16, 8 * D, kSwz);
            const uint64_t db = make_smem_desc(k_addr + 32 * kk, 16, 8 * D, kSwz);
            mma_i8_ss(tS, da, db, kIdescQK, kk > 0 ? 1u : 0u);
          }
          mma_commit(bar_s_full);
          // (8) O (+)= P_j [V_j | 1] : M=128, N=D+16, K=BC in steps of 32 keys.
          mbar_wait(bar_p_full, j & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BC / 32; ++kk) {
            const uint32_t vk = v_addr + 32 * kk * D;
            const uint64_t db = make_smem_desc(vk, ones_addr - v_addr, 8 * D, kSwz);
            mma_i8_ts(tO, tS + 8 * kk, db, kIdescPV, (j > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&bar_kv_empty[st]);
          mma_commit(bar_o_full);
        }
      }
    } else if (warp >= kSoftmaxWarp0) {
      if (prm.q_shift == 0 && prm.p_pre == 0)
        softmax_rows<D, BC, PACKED, true>(args, prm, tmem_base, bar_s_full, bar_p_full, bar_o_full,
                                          problem, q0, warp, lane);
      else
        softmax_rows<D, BC, PACKED, false>(args, prm, tmem_base, bar_s_full, bar_p_full, bar_o_full,
                                           problem, q0, warp, lane);
    }
  }

  // ------------------------------------------------------------- teardown
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, kTmemCols);
}

// ----------------------------------------------------------------------------
// Host-side launch helpers (called by qflash_host.cu).
template <int D, int BC, bool PACKED>
cudaError_t launch_attn_t(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                          const AttnArgs& args, dim3 grid, cudaStream_t stream) {
  using L = SmemLayout<D, BC>;
  auto kern = qflash_attn_kernel<D, BC, PACKED>;
  static int configured[16] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 16 || !configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kAlloc);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 16) configured[dev] = 1;
  }
  kern<<<grid, kThreads, L::kAlloc, stream>>>(tq, tk, tv, args);
  return cudaGetLastError();
}

cudaError_t launch_attention(int D, int BC, bool packed, const CUtensorMap& tq,
                             const CUtensorMap& tk, const CUtensorMap& tv, const AttnArgs& args,
                             dim3 grid, cudaStream_t stream) {
  if (packed) {
    // T_c = 1 and the KV tile is 2 x 64 keys regardless of block_kv.
    switch (D) {
      case 32: return launch_attn_t<32, 128, true>(tq, tk, tv, args, grid, stream);
      case 64: return launch_attn_t<64, 128, true>(tq, tk, tv, args, grid, stream);
      case 128: return launch_attn_t<128, 128, true>(tq, tk, tv, args, grid, stream);
    }
    return cudaErrorInvalidValue;
  }
#define QF_CASE(d, bc) \
  if (D == d && BC == bc) return launch_attn_t<d, bc, false>(tq, tk, tv, args, grid, stream);
  QF_CASE(32, 64) QF_CASE(32, 128) QF_CASE(32, 256)
  QF_CASE(64, 64) QF_CASE(64, 128) QF_CASE(64, 256)
  QF_CASE(128, 64) QF_CASE(128, 128) QF_CASE(128, 256)
#undef QF_CASE
  return cudaErrorInvalidValue;
}

}  // namespace qf
