// qflash_common.cuh -- structures shared by the host library and the kernels of
// libqflash.so (NOT shared with the oracle).
#pragma once
#include <cstdint>
#include <cstdlib>

namespace qf {

// Per-launch integer constants of Algorithm 1 as the kernel consumes them.
struct IntParams {
  int32_t status;     // 0 = OK (device-derived path may report a range error)
  int32_t s_inv;      // round(1/s)                               (Alg. 2)
  uint32_t q_magic;   // q1 = umulhi(t, q_magic) >> q_shift == floor(t / s_inv)
  int32_t q_shift;
  uint32_t p_mul;     // P = umulhi(y << p_pre, p_mul) == floor(y M_P / 2^r_P)
  int32_t p_pre;
  uint32_t rel_magic_lo;  // floor(n / s_inv) == umul64hi(n, rel_magic) >> rel_shift
  uint32_t rel_magic_hi;
  int32_t rel_shift;
  int32_t p_max;
  int32_t r_p, m_p, n;
  int32_t one;        // always 1 (a runtime multiplier that keeps an add on the FMA pipe)
  int32_t zero;       // always 0 (a runtime addend that keeps an add on the ALU pipe)
  int32_t pad[1];
  double s;
};
static_assert(sizeof(IntParams) == 72, "IntParams layout");

constexpr int kPdlDefault = 15;
// Workspace layout of the device-scale paths (QFLASH_DSCALE_WORKSPACE_BYTES = 8192):
// [0, 128) IntParams, [256, 4096) per-CTA amax partials (3 floats per CTA),
// [4096, 5120) the 256-entry dequant table.
constexpr int kWsPartialOffset = 256;
constexpr int kWsDqTableOffset = 4096;
constexpr int kWsMaxPartialCtas = (kWsDqTableOffset - kWsPartialOffset) / 12;  // = 320
static_assert(kWsMaxPartialCtas == 320, "partials must end before the dequant table");
constexpr int kHeadPrmStride = 80;   // bytes per head in the per-head constant table
constexpr int kHeadPrmOffset = 128;  // table offset in the per-head workspace
constexpr int kMaxHeads = 96;        // 128 + 96 * 80 <= QFLASH_DSCALE_WORKSPACE_BYTES
// Fused per-head step workspace (QFLASH_PH_FUSED_WORKSPACE_BYTES = 16384): header at 0,
// per-head table at kHeadPrmOffset, per-(tensor, head) amax accumulators at 8192.
constexpr int kWsPhAmaxOffset = 8192;
// shared-memory head area of the fused per-head kernels: table [96] x 80 B, s[3][96],
// 1/s[3][96], amax bits[3][96]
constexpr int kHeadAreaBytes = kMaxHeads * kHeadPrmStride + 3 * 3 * kMaxHeads * 4;

struct AttnArgs {
  int32_t N;        // sequence length
  int32_t P;        // number of problems
  int32_t Tc;       // ceil(N / B_c) KV tiles
  int32_t Tr;       // ceil(N / 128) query tiles per problem (generic tiling)
  uint32_t tr_magic;  // ceil(2^32 / Tr): t / Tr == umulhi(t, tr_magic) for t < 2^32 / Tr
  int32_t g_div;    // grid stride in whole problems (generic: G / Tr; packed: 128 G / N)
  int32_t g_mod;    // ... and the leftover rows (generic: 128 (G % Tr); packed: 128 G % N)
  int32_t pad0;
  uint64_t n_magic;  // ceil(2^64 / N) (row-packed tiling)
  IntParams prm;    // used when dev_prm == nullptr
  const IntParams* dev_prm;  // device-derived constants (dscale path) or nullptr
  int8_t* out;          // int8 output (may be nullptr when out_f32 is set)
  float* out_f32;       // fused dequantized fp32 output, or nullptr
  const uint32_t* dq_table;  // [256] fp32 bits of s_V * (i - 128) (device), with out_f32
  // fused step (FQ instantiations): the kernel's prologue quantizes fp32 inputs
  const float* xin[3];  // Q, K, V fp32 [P, N, d] (device)
  int8_t* xq[3];        // their int8 codes (the TMA maps point here)
  float* scales_out;    // device float[3]: s_q, s_k, s_v
  float* partial;       // device float[3 * gridDim.x]: per-CTA amax partials
  IntParams* prm_out;   // device copy of the derived constants (workspace)
  uint32_t* table_out;  // device copy of the dequant table (workspace + 4096)
  int64_t numel;        // elements per tensor (a multiple of 4: d in {32, 64, 128})
  // per-head granularity (PH instantiations): head h = problem mod H
  const IntParams* head_prm;  // device table, kHeadPrmStride bytes per head
  int32_t H;
  uint32_t h_magic;           // ceil(2^32 / H): problem / H = umulhi(problem, h_magic)
  const float* amax_in;       // fused step: device float[3] amax of Q, K, V supplied by the
                              // caller (sharded quantization), or nullptr (computed here)
  int32_t* acc_flags;         // scale-accumulation ablation (Eq. 13): overflow flags, or nullptr
  int32_t variant;            // ablation variant (0 = the method; 1 Eq. 13; 2 V3; 3 V2)
  float s_v;                  // V2 / V3 ablations: s_V for the fp32 output y = s_V O / l
  // fused step, packed QKV projection output: xin[0..2] all point at one
  // [P / H, N, 3, H, d] fp32 tensor; qkv_H = H (0: three separate [P, N, d] tensors)
  // fused per-head step (FQ + PH): per-(tensor, head) amax accumulators
  // (device uint32 [3][H], zero at launch start; the kernel re-zeroes them at its end)
  uint32_t* ph_amax;
  uint64_t vp_magic;          // ceil(2^64 / (N d / 4)): problem of a float4 index
  int32_t qkv_H;
  int32_t pad3;
  uint64_t qkv_n_magic;       // ceil(2^64 / N): floor(x / N) = umul64hi(x, magic), x < 2^32
  uint64_t qkv_h_magic;       // ceil(2^64 / H)
  int32_t cluster_grid;       // fused step: 1 = the grid is one thread-block cluster
                              // (barrier.cluster replaces the grid barriers)
  int32_t pad2;
  // bring-up dumps for CTA 0's first tile only; nullptr in production:
  int32_t* dbg_s;  // [128][BC] raw S of KV tile 0
  int32_t* dbg_p;  // [128][BC/4] packed P words of KV tile 0
  int32_t* dbg_o;  // [128][D+1] final O and l before normalization
  long long* dbg_t;  // [128] clock64 timeline of CTA 0 (see QF_TS slots), then
                     // globaltimer (entry, exit) of every CTA b at [128 + 2b]
};

// Up to three tensors quantized by one launch pair (Q/K/V fusion).
struct QuantTensors {
  const void* x[3];
  int8_t* xq[3];
  float* scale[3];
};

// Programmatic dependent launch per kernel (bit 0 attention, bit 1 dequantize,
// bit 2 second quantize pass, bit 3 fused step); QFLASH_PDL=<mask> overrides the
// default (A/B).
inline int pdl_mask() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("QFLASH_PDL");
    m = (e != nullptr) ? static_cast<int>(strtol(e, nullptr, 10)) : kPdlDefault;
  }
  return m;
}

}  // namespace qf
