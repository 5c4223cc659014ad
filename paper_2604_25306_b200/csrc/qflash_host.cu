// qflash_host.cu -- the C ABI of libqflash.so (include/qflash.h): argument
// validation, derivation of the integer constants (host fp64, or on the device
// for the dscale path), TMA descriptor encoding and kernel launches.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include "../../include/qflash.h"
#include "../../include/qflash_debug.h"
#include "qflash_common.cuh"
#include "qflash_params.cuh"

namespace qf {
#define QF_DECL_D(D)                                                                      \
  cudaError_t launch_attention_d##D(int BC, int nseg, int cfg, const CUtensorMap& tq,      \
                                    const CUtensorMap& tk, const CUtensorMap& tv,          \
                                    const AttnArgs& args, int64_t tiles, int sms,          \
                                    cudaStream_t stream);                                  \
  bool attention_supported_d##D(int BC, int nseg, int cfg);
QF_DECL_D(32)
QF_DECL_D(64)
QF_DECL_D(128)
#undef QF_DECL_D
cudaError_t launch_fused_d32(int BC, int nseg, int cfg, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, const AttnArgs& args, int64_t tiles, int sms,
                             cudaStream_t stream);
cudaError_t launch_fused_d64(int BC, int nseg, int cfg, const CUtensorMap& tq, const CUtensorMap& tk,
                             const CUtensorMap& tv, const AttnArgs& args, int64_t tiles, int sms,
                             cudaStream_t stream);
cudaError_t launch_fused_d128(int BC, int nseg, int cfg, const CUtensorMap& tq, const CUtensorMap& tk,
                              const CUtensorMap& tv, const AttnArgs& args, int64_t tiles, int sms,
                              cudaStream_t stream);
cudaError_t launch_attention_var(int var, int D, int BC, const CUtensorMap& tq, const CUtensorMap& tk,
                                 const CUtensorMap& tv, const AttnArgs& args, int64_t tiles, int sms,
                                 cudaStream_t stream);
cudaError_t launch_fused_ph(int D, int BC, int nseg, int cfg, const CUtensorMap& tq, const CUtensorMap& tk,
                            const CUtensorMap& tv, const AttnArgs& args, int64_t tiles, int sms,
                            cudaStream_t stream);
cudaError_t launch_attention_ph(int D, int BC, int nseg, int cfg, const CUtensorMap& tq,
                                const CUtensorMap& tk, const CUtensorMap& tv,
                                const AttnArgs& args, int64_t tiles, int sms,
                                cudaStream_t stream);
cudaError_t launch_quantize_per_head(const QuantTensors& t, int ntensors, int64_t P,
                                     int64_t vec_per_problem, int H, cudaStream_t stream);
cudaError_t launch_derive_per_head(const float* scales, int H, int32_t d, void* ws, cudaStream_t stream);
cudaError_t launch_dequantize_per_head(const int8_t* xq, const float* scales, int64_t P,
                                       int64_t vec_per_problem, int H, float* y, cudaStream_t stream);
cudaError_t launch_attention_dbg(int D, int BC, int nseg, int cfg, const CUtensorMap& tq,
                                 const CUtensorMap& tk, const CUtensorMap& tv,
                                 const AttnArgs& args, int64_t tiles, int sms,
                                 cudaStream_t stream);
inline bool attention_supported(int D, int BC, int nseg, int cfg) {
  return D == 32 ? attention_supported_d32(BC, nseg, cfg)
       : D == 64 ? attention_supported_d64(BC, nseg, cfg)
       : D == 128 ? attention_supported_d128(BC, nseg, cfg) : false;
}
inline cudaError_t launch_attention(int D, int BC, int nseg, int cfg, const CUtensorMap& tq,
                                    const CUtensorMap& tk, const CUtensorMap& tv,
                                    const AttnArgs& args, int64_t tiles, int sms, bool dbg,
                                    bool fused, cudaStream_t stream) {
  if (fused) {
    if (D == 32) return launch_fused_d32(BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
    if (D == 64) return launch_fused_d64(BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
    if (D == 128) return launch_fused_d128(BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
    return cudaErrorNotSupported;
  }
  if (dbg) return launch_attention_dbg(D, BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
  if (D == 32) return launch_attention_d32(BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
  if (D == 64) return launch_attention_d64(BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
  if (D == 128) return launch_attention_d128(BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
  return cudaErrorNotSupported;
}
cudaError_t launch_quantize(const QuantTensors& t, int ntensors, int dtype, int64_t numel,
                            IntParams* prm_out, int32_t head_dim, cudaStream_t stream,
                            float* partial);
cudaError_t launch_amax3(const float* q, const float* k, const float* v, int64_t numel, float* amax,
                         cudaStream_t stream);
cudaError_t launch_dequantize(const int8_t* xq, float scale, const float* scale_dev,
                              int64_t numel, float* y, cudaStream_t stream);
}  // namespace qf

namespace {

constexpr int32_t kVersion = (1 << 16) | 0;
thread_local char g_err[512] = "";

void set_err(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

qflash_status fail(qflash_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

qflash_status cuda_fail(cudaError_t e, const char* where) {
  set_err("%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
  return QFLASH_ERR_CUDA;
}

__global__ void derive_params_kernel(const float* __restrict__ scales, int32_t d,
                                     qf::IntParams* __restrict__ out) {
  qf::IntParams p;
  const int st = qf::derive_core(scales[0], scales[1], d, &p, nullptr);
  if (st != QFLASH_OK) {
    memset(&p, 0, sizeof(p));
    p.status = st;
  }
  *out = p;
}

// ------------------------------------------------------------------------
// Device capability check (sm_100 only), cached per device ordinal.
qflash_status check_device(int* dev_out) {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  static int cached[64];  // 0 unknown, 1 ok, 2 bad
  if (dev >= 0 && dev < 64 && cached[dev] == 1) {
    *dev_out = dev;
    return QFLASH_OK;
  }
  int major = 0, minor = 0;
  e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  e = cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  if (!(major == 10 && minor == 0))
    return fail(QFLASH_ERR_UNSUPPORTED_DEVICE, "device %d is sm_%d%d; libqflash is built for sm_100a",
                dev, major, minor);
  if (dev >= 0 && dev < 64) cached[dev] = 1;
  *dev_out = dev;
  return QFLASH_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D int8 tensor map over [P][N][d] with box {d, rows, probs}.  Rows outside
// [0, N) of a box are zero-filled by the TMA unit (ragged tiles, row-packed Q).
// A tensor map is a pure function of (base, P, N, d, rows, probs): the last few encodings
// are cached per thread so repeated eager calls on the same buffers (serving loops,
// single-call latency) skip cuTensorMapEncodeTiled.
struct TmapKey {
  const int8_t* base;
  int P, N, d, rows, probs, dev;
  bool operator==(const TmapKey& o) const {
    return base == o.base && P == o.P && N == o.N && d == o.d && rows == o.rows && probs == o.probs &&
           dev == o.dev;
  }
};
constexpr int kTmapCache = 16;
thread_local TmapKey g_tmap_key[kTmapCache];
thread_local CUtensorMap g_tmap_val[kTmapCache];
thread_local int g_tmap_n = 0, g_tmap_next = 0;

qflash_status make_tmap_uncached(CUtensorMap* m, const int8_t* base, int P, int N, int d, int rows,
                                 int probs);
qflash_status make_tmap(CUtensorMap* m, const int8_t* base, int P, int N, int d, int rows, int probs) {
  int dev = -1;
  cudaGetDevice(&dev);
  const TmapKey key{base, P, N, d, rows, probs, dev};
  for (int i = 0; i < g_tmap_n; ++i)
    if (g_tmap_key[i] == key) {
      *m = g_tmap_val[i];
      return QFLASH_OK;
    }
  qflash_status st = make_tmap_uncached(m, base, P, N, d, rows, probs);
  if (st != QFLASH_OK) return st;
  g_tmap_key[g_tmap_next] = key;
  g_tmap_val[g_tmap_next] = *m;
  g_tmap_next = (g_tmap_next + 1) % kTmapCache;
  if (g_tmap_n < kTmapCache) ++g_tmap_n;
  return QFLASH_OK;
}

qflash_status make_tmap_uncached(CUtensorMap* m, const int8_t* base, int P, int N, int d, int rows,
                                 int probs) {
  auto enc = get_encode_fn();
  if (!enc) return fail(QFLASH_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(N),
                        static_cast<cuuint64_t>(P)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(N) * d};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(d), static_cast<cuuint32_t>(rows),
                       static_cast<cuuint32_t>(probs)};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapSwizzle sw = d == 32   ? CU_TENSOR_MAP_SWIZZLE_32B
                                : d == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                          : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(QFLASH_ERR_CUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", static_cast<int>(r));
  return QFLASH_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Attention kernel configuration override (qflash_debug_force_config, or the
// QFLASH_ATTN_CFG environment variable read once): -1 = the host heuristic.
std::atomic<int> g_force_config{-2};
thread_local int g_last_config = -1;  // cfg | nseg << 4 of this thread's last launch
int forced_config() {
  int c = g_force_config.load(std::memory_order_relaxed);
  if (c == -2) {
    const char* env = getenv("QFLASH_ATTN_CFG");
    c = (env != nullptr && env[0] >= '0' && env[0] <= '3') ? env[0] - '0' : -1;
    int expected = -2;
    g_force_config.compare_exchange_strong(expected, c);
    c = g_force_config.load(std::memory_order_relaxed);
  }
  return c;
}

bool overlaps(const void* a, int64_t na, const void* b, int64_t nb) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
  return a0 < b0 + static_cast<uintptr_t>(nb) && b0 < a0 + static_cast<uintptr_t>(na);
}

qflash_status validate_shape(const qflash_attn_shape* shape, int* bc_out) {
  if (!shape) return fail(QFLASH_ERR_INVALID_ARGUMENT, "shape is NULL");
  const int P = shape->num_problems, N = shape->seq_len, d = shape->head_dim;
  const int bc = shape->block_kv == 0 ? 128 : shape->block_kv;
  if (P < 1) return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "num_problems %d < 1", P);
  if (N < 1 || N > 65536) return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "seq_len %d not in [1, 65536]", N);
  if (d != 32 && d != 64 && d != 128)
    return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "head_dim %d not in {32, 64, 128}", d);
  if (bc != 64 && bc != 128 && bc != 256)
    return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "block_kv %d not in {64, 128, 256}", shape->block_kv);
  *bc_out = bc;
  return QFLASH_OK;
}

qflash_status validate_qkvo(const int8_t* q, const int8_t* k, const int8_t* v, const int8_t* o,
                            int64_t bytes) {
  if (!q || !k || !v || !o) return fail(QFLASH_ERR_INVALID_ARGUMENT, "NULL tensor pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "tensor pointers must be 16-byte aligned");
  if (overlaps(o, bytes, q, bytes) || overlaps(o, bytes, k, bytes) || overlaps(o, bytes, v, bytes))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "output o aliases q/k/v");
  return QFLASH_OK;
}

struct FusedIn {
  const float* x[3];
  int8_t* xq[3];
  float* scales;
  void* workspace;
  const float* amax_in;  // nullptr: the kernel computes the amax itself
  int qkv_heads;         // > 0: x[0] is one packed [P / H, N, 3, H, d] projection output
};

qflash_status launch_common(const int8_t* q, const int8_t* k, const int8_t* v,
                            const qflash_attn_shape* shape, int bc, qflash_variant variant,
                            int8_t* o, const qf::IntParams* host_prm,
                            const qf::IntParams* dev_prm, cudaStream_t stream, float* y,
                            const FusedIn* fin, int heads,
                            int32_t* dbg_s = nullptr, int32_t* dbg_p = nullptr,
                            int32_t* dbg_o = nullptr, long long* dbg_t = nullptr,
                            int32_t* acc_flags = nullptr, int abl_var = 0, float abl_sv = 0.f) {
  const int P = shape->num_problems, N = shape->seq_len, d = shape->head_dim;
  // KV block: with T_c = 1 every B_c >= N gives the same result (one block), so
  // take the smallest supported one; otherwise B_c = block_kv as requested.
  const int bc_eff = N <= bc ? (N <= 64 ? 64 : N <= 128 ? 128 : 256) : bc;
  // Row-packed tiling: 128 consecutive flattened rows span at most
  // floor((N + 126) / N) + 1 problems; supported up to 4 segments.
  const int seg_need = N >= 2 ? (N + 126) / N + 1 : 129;
  const int nseg_tpl = seg_need <= 2 ? 2 : 4;
  const bool packable = seg_need <= 4 && (qf::attention_supported(d, bc_eff, nseg_tpl, 0) ||
                                          qf::attention_supported(d, bc_eff, nseg_tpl, 1));
  const int64_t Tr = (N + 127) / 128;
  const int64_t tiles_generic = static_cast<int64_t>(P) * Tr;
  const int64_t tiles_packed = (static_cast<int64_t>(P) * N + 127) / 128;
  int sms = 0;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    static int sm_cache[64];
    if (dev >= 0 && dev < 64 && sm_cache[dev] > 0) {
      sms = sm_cache[dev];
    } else {
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (sms <= 0) sms = 148;
      if (dev >= 0 && dev < 64) sm_cache[dev] = sms;
    }
  }
  // the fused step's per-CTA amax partials must fit the workspace (one CTA per SM)
  if (fin != nullptr && sms > qf::kWsMaxPartialCtas) sms = qf::kWsMaxPartialCtas;
  // AUTO packs rows only when that saves a wave of one-tile-per-SM work: a
  // row-packed tile costs a little more (one TMA load and MMA per segment).
  const int64_t waves_generic = (tiles_generic + sms - 1) / sms;
  const int64_t waves_packed = (tiles_packed + sms - 1) / sms;
  bool packed;
  if (abl_var != 0) variant = QFLASH_VARIANT_GENERIC;  // ablation variants: generic tiles
  switch (variant) {
    case QFLASH_VARIANT_AUTO:
      // one wave: pack when it saves a wave (A3 b8: 192 -> 148 tiles); several waves:
      // generic tiles get configuration 1's separate P region (measured L14 b64: 802 us
      // generic vs 844 us packed), so pack only for a large tile saving (Swin windows)
      packed = packable && (tiles_generic > sms ? tiles_packed * 100 < tiles_generic * 85
                                                : waves_packed < waves_generic);
      break;
    case QFLASH_VARIANT_GENERIC: packed = false; break;
    case QFLASH_VARIANT_PACKED:
      if (!packable)
        return fail(QFLASH_ERR_UNSUPPORTED_SHAPE,
                    "row-packed variant needs seq_len >= 43 (<= 4 problems per 128-row tile) "
                    "and a supported (head_dim, block) pair");
      packed = true;
      break;
    default: return fail(QFLASH_ERR_INVALID_ARGUMENT, "unknown variant %d", static_cast<int>(variant));
  }
  const int nseg = packed ? nseg_tpl : 1;
  const int64_t tiles = packed ? tiles_packed : tiles_generic;
  // Kernel configuration (qflash_attn_inst.cuh): with more than one wave of
  // tiles, cfg 2 (two ping-ponging query tiles, row-owner softmax + correction
  // warpgroups) or cfg 1 (two tiles, 2 column splits) where it fits TMEM /
  // shared memory; else cfg 0 (one tile, 4 column splits: lowest latency per
  // tile).  QFLASH_ATTN_CFG=0..3 overrides.
  const int cfg_env = forced_config();
  // Measured: multi-wave with several KV tiles -> cfg 1 (profiles/r1_cfg_ab.txt, L14 b64:
  // 848 vs 938 us for cfg 2); multi-wave with one KV tile (Swin windows) -> cfg 1 as well
  // since round 2 (profiles/r2b_cfg_ab.txt, chained graphs: A4 b8 25.7 vs 26.6 us for cfg 2,
  // Swin-B s1 b8 32.3 vs 33.2 us); cfg 2 where cfg 1 does not fit.
  const int Tc_host = (N + bc_eff - 1) / bc_eff;
  int cfg = 0;
  if (tiles > sms && heads == 0) {
    const int pref[2] = {1, 2};
    for (int c : pref)
      if (cfg == 0 && qf::attention_supported(d, bc_eff, nseg, c)) cfg = c;
  }
  // per-head constants: cfg 1 for multi-wave generic tiles with several KV tiles (the
  // row-owner configurations have no per-head instantiation), else cfg 0
  if (heads > 0 && tiles > sms && nseg == 1 && Tc_host > 1 && bc_eff <= 128 &&
      qf::attention_supported(d, bc_eff, 1, 1))
    cfg = 1;
  if (heads > 0 && cfg_env >= 0) cfg = (cfg_env == 1 && nseg == 1 && bc_eff <= 128) ? 1 : 0;
  if (cfg_env >= 0 && heads == 0 && qf::attention_supported(d, bc_eff, nseg, cfg_env)) cfg = cfg_env;
  if (abl_var != 0) cfg = 0;
  if (!qf::attention_supported(d, bc_eff, nseg, cfg))
    return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "no kernel configuration for d=%d block=%d", d, bc_eff);
  g_last_config = cfg | (nseg << 4);
  CUtensorMap tq, tk, tv;
  qflash_status st;
  if ((st = make_tmap(&tq, q, P, N, d, 128, 1)) != QFLASH_OK) return st;
  if ((st = make_tmap(&tk, k, P, N, d, bc_eff, 1)) != QFLASH_OK) return st;
  if ((st = make_tmap(&tv, v, P, N, d, bc_eff, 1)) != QFLASH_OK) return st;
  qf::AttnArgs args;
  memset(&args, 0, sizeof(args));
  args.N = N;
  args.P = P;
  args.Tc = (N + bc_eff - 1) / bc_eff;
  if (host_prm) args.prm = *host_prm;
  args.dev_prm = dev_prm;
  args.out = o;
  if (y != nullptr && fin == nullptr && abl_var == 0) {
    args.out_f32 = y;
    args.dq_table = reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(dev_prm) + 4096);
  }
  if (abl_var >= 2) {  // V3 / V2 ablations: fp32 y = s_V O / l written by the epilogue
    args.out_f32 = y;
    args.s_v = abl_sv;
  }
  if (fin != nullptr) {  // fused step: the kernel quantizes fin->x into q/k/v itself
    args.out_f32 = y;
    args.dev_prm = nullptr;
    for (int t = 0; t < 3; ++t) {
      args.xin[t] = fin->x[t];
      args.xq[t] = fin->xq[t];
    }
    args.scales_out = fin->scales;
    args.amax_in = fin->amax_in;
    if (fin->qkv_heads > 0) {
      args.qkv_H = fin->qkv_heads;
      args.qkv_n_magic = ~0ull / static_cast<uint64_t>(N) + 1ull;  // ceil(2^64 / N) (N = 1, H = 1: identity)
      args.qkv_h_magic = ~0ull / static_cast<uint64_t>(fin->qkv_heads) + 1ull;
    }
    args.prm_out = reinterpret_cast<qf::IntParams*>(fin->workspace);
    args.partial = reinterpret_cast<float*>(static_cast<char*>(fin->workspace) + qf::kWsPartialOffset);
    args.table_out = reinterpret_cast<uint32_t*>(static_cast<char*>(fin->workspace) + qf::kWsDqTableOffset);
    args.numel = static_cast<int64_t>(P) * N * d;
  }
  args.acc_flags = acc_flags;
  args.variant = abl_var;
  args.dbg_s = dbg_s;
  args.dbg_p = dbg_p;
  args.dbg_o = dbg_o;
  args.dbg_t = dbg_t;
  // Persistent grid: one CTA per SM, its groups walking tiles b + g G, + QT G, ...
  args.Tr = static_cast<int32_t>(Tr);
  const bool dbg = dbg_s != nullptr || dbg_p != nullptr || dbg_o != nullptr || dbg_t != nullptr;
  cudaError_t e;
  if (abl_var != 0) {
    e = qf::launch_attention_var(abl_var, d, bc_eff, tq, tk, tv, args, tiles, sms, stream);
  } else if (heads > 0 && fin != nullptr) {  // fused per-head step (one cooperative launch)
    args.H = heads;
    args.h_magic = static_cast<uint32_t>(((1ull << 32) + heads - 1) / heads);
    const uint64_t vpp = static_cast<uint64_t>(N) * d / 4;
    args.vp_magic = vpp == 1 ? 0ull : ~0ull / vpp + 1ull;  // ceil(2^64 / vpp)
    args.ph_amax = reinterpret_cast<uint32_t*>(static_cast<char*>(fin->workspace) + qf::kWsPhAmaxOffset);
    if (bc_eff > 128) return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "fused per-head step: block_kv <= 128");
    e = qf::launch_fused_ph(d, bc_eff, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
  } else if (heads > 0) {  // per-head constants (configuration 0 or 1)
    args.head_prm = reinterpret_cast<const qf::IntParams*>(reinterpret_cast<const char*>(dev_prm) +
                                                          qf::kHeadPrmOffset);
    args.H = heads;
    args.h_magic = static_cast<uint32_t>(((1ull << 32) + heads - 1) / heads);
    e = qf::launch_attention_ph(d, bc_eff, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
  } else {
    e = qf::launch_attention(d, bc_eff, nseg, cfg, tq, tk, tv, args, tiles, sms, dbg,
                             fin != nullptr, stream);
  }
  if (e == cudaErrorNotSupported)
    return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "no kernel instantiation for d=%d block=%d nseg=%d cfg=%d", d,
                bc_eff, nseg, cfg);
  if (e != cudaSuccess) return cuda_fail(e, "attention launch");
  return QFLASH_OK;
}

qflash_status attention_host_scales(const int8_t* q, const int8_t* k, const int8_t* v, float s_q,
                                    float s_k, float s_v, const qflash_attn_shape* shape,
                                    qflash_variant variant, int8_t* o, float* s_o,
                                    cudaStream_t stream) {
  int bc = 0;
  qflash_status st = validate_shape(shape, &bc);
  if (st != QFLASH_OK) return st;
  const int64_t bytes = static_cast<int64_t>(shape->num_problems) * shape->seq_len * shape->head_dim;
  if ((st = validate_qkvo(q, k, v, o, bytes)) != QFLASH_OK) return st;
  if (!(s_v > 0.0f) || !std::isfinite(s_v))
    return fail(QFLASH_ERR_SCALE_RANGE, "s_v must be positive and finite");
  qf::IntParams prm;
  const int rc = qf::derive_core(s_q, s_k, shape->head_dim, &prm, nullptr);
  if (rc != QFLASH_OK)
    return fail(static_cast<qflash_status>(rc),
                "s = s_q s_k log2(e)/sqrt(d) outside [2^-24, 0.5] (s_q=%g, s_k=%g, d=%d)",
                static_cast<double>(s_q), static_cast<double>(s_k), shape->head_dim);
  int dev = 0;
  if ((st = check_device(&dev)) != QFLASH_OK) return st;
  if ((st = launch_common(q, k, v, shape, bc, variant, o, &prm, nullptr, stream, nullptr, nullptr, 0)) != QFLASH_OK)
    return st;
  if (s_o) *s_o = s_v;  // s_O = s_V
  return QFLASH_OK;
}

}  // namespace

// ============================================================================ C ABI
extern "C" {

int32_t qflash_version(void) { return kVersion; }

const char* qflash_status_string(qflash_status s) {
  switch (s) {
    case QFLASH_OK: return "QFLASH_OK";
    case QFLASH_ERR_INVALID_ARGUMENT: return "QFLASH_ERR_INVALID_ARGUMENT";
    case QFLASH_ERR_UNSUPPORTED_SHAPE: return "QFLASH_ERR_UNSUPPORTED_SHAPE";
    case QFLASH_ERR_SCALE_RANGE: return "QFLASH_ERR_SCALE_RANGE";
    case QFLASH_ERR_CUDA: return "QFLASH_ERR_CUDA";
    case QFLASH_ERR_UNSUPPORTED_DEVICE: return "QFLASH_ERR_UNSUPPORTED_DEVICE";
  }
  return "QFLASH_ERR_UNKNOWN";
}

const char* qflash_last_error(void) { return g_err; }

qflash_status qflash_derive_params(float s_q, float s_k, int32_t head_dim, qflash_int_params* out) {
  if (!out) return fail(QFLASH_ERR_INVALID_ARGUMENT, "out is NULL");
  if (head_dim != 32 && head_dim != 64 && head_dim != 128)
    return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "head_dim %d not in {32, 64, 128}", head_dim);
  const int rc = qf::derive_core(s_q, s_k, head_dim, nullptr, out);
  if (rc != QFLASH_OK) return fail(static_cast<qflash_status>(rc), "scale out of range");
  return QFLASH_OK;
}

void qflash_partition(int32_t num_problems, int32_t world, int32_t rank, int32_t* begin,
                      int32_t* count) {
  int32_t b = 0, c = 0;
  if (num_problems >= 0 && world >= 1 && rank >= 0 && rank < world) {
    const int64_t lo = static_cast<int64_t>(rank) * num_problems / world;
    const int64_t hi = static_cast<int64_t>(rank + 1) * num_problems / world;
    b = static_cast<int32_t>(lo);
    c = static_cast<int32_t>(hi - lo);
  }
  if (begin) *begin = b;
  if (count) *count = c;
}

qflash_status qflash_attention_int8(const int8_t* q, const int8_t* k, const int8_t* v, float s_q,
                                    float s_k, float s_v, const qflash_attn_shape* shape,
                                    int8_t* o, float* s_o, qflash_stream_t stream) {
  return attention_host_scales(q, k, v, s_q, s_k, s_v, shape, QFLASH_VARIANT_AUTO, o, s_o,
                               reinterpret_cast<cudaStream_t>(stream));
}

qflash_status qflash_attention_int8_ex(const int8_t* q, const int8_t* k, const int8_t* v,
                                       float s_q, float s_k, float s_v,
                                       const qflash_attn_shape* shape, qflash_variant variant,
                                       int8_t* o, float* s_o, qflash_stream_t stream) {
  return attention_host_scales(q, k, v, s_q, s_k, s_v, shape, variant, o, s_o,
                               reinterpret_cast<cudaStream_t>(stream));
}

qflash_status qflash_attention_int8_dscale(const int8_t* q, const int8_t* k, const int8_t* v,
                                           const float* scales_dev,
                                           const qflash_attn_shape* shape, qflash_variant variant,
                                           int8_t* o, void* workspace_dev,
                                           qflash_stream_t stream) {
  int bc = 0;
  qflash_status st = validate_shape(shape, &bc);
  if (st != QFLASH_OK) return st;
  const int64_t bytes = static_cast<int64_t>(shape->num_problems) * shape->seq_len * shape->head_dim;
  if ((st = validate_qkvo(q, k, v, o, bytes)) != QFLASH_OK) return st;
  if (!scales_dev || !workspace_dev || !aligned16(workspace_dev))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "scales_dev / workspace_dev NULL or misaligned");
  int dev = 0;
  if ((st = check_device(&dev)) != QFLASH_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  auto* prm = reinterpret_cast<qf::IntParams*>(workspace_dev);
  derive_params_kernel<<<1, 1, 0, s>>>(scales_dev, shape->head_dim, prm);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "derive_params_kernel launch");
  return launch_common(q, k, v, shape, bc, variant, o, nullptr, prm, s, nullptr, nullptr, 0);
}

static qflash_status quantize_impl(const void* const* xs, int8_t* const* xqs, float* const* scales,
                                   int nt, qflash_dtype dtype, int64_t numel, cudaStream_t stream,
                                   qf::IntParams* prm_out = nullptr, int32_t head_dim = 0,
                                   float* partial = nullptr) {
  if (numel < 0) return fail(QFLASH_ERR_INVALID_ARGUMENT, "numel < 0");
  if (dtype != QFLASH_F32 && dtype != QFLASH_BF16 && dtype != QFLASH_F16)
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "unknown dtype %d", static_cast<int>(dtype));
  for (int i = 0; i < nt; ++i) {
    // an empty tensor (numel == 0) may pass NULL data pointers: no codes are
    // written and its scale is 1/127 (amax of the empty set is 0, reading R3)
    if ((numel > 0 && (!xs[i] || !xqs[i])) || !scales[i])
      return fail(QFLASH_ERR_INVALID_ARGUMENT, "NULL pointer");
    if (!aligned16(xs[i]) || !aligned16(xqs[i]))
      return fail(QFLASH_ERR_INVALID_ARGUMENT, "x and x_q must be 16-byte aligned");
  }
  int dev = 0;
  qflash_status st = check_device(&dev);
  if (st != QFLASH_OK) return st;
  qf::QuantTensors t;
  memset(&t, 0, sizeof(t));
  for (int i = 0; i < nt; ++i) {
    t.x[i] = xs[i];
    t.xq[i] = xqs[i];
    t.scale[i] = scales[i];
  }
  cudaError_t e = qf::launch_quantize(t, nt, static_cast<int>(dtype), numel, prm_out, head_dim, stream,
                                      partial);
  if (e != cudaSuccess) return cuda_fail(e, "quantize launch");
  return QFLASH_OK;
}

qflash_status qflash_quantize_per_tensor(const void* x, qflash_dtype dtype, int64_t numel,
                                         int8_t* x_q, float* scale_dev, float* scale_host,
                                         qflash_stream_t stream) {
  if (!scale_dev && !scale_host)
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "need scale_dev or scale_host");
  if (numel > 0 && (!x || !x_q)) return fail(QFLASH_ERR_INVALID_ARGUMENT, "NULL pointer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  float* sd = scale_dev;
  bool temp = false;
  if (!sd) {
    int dev = 0;
    qflash_status st = check_device(&dev);
    if (st != QFLASH_OK) return st;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&sd), sizeof(float), s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(scale)");
    temp = true;
  }
  const void* xs[1] = {x};
  int8_t* xqs[1] = {x_q};
  float* scs[1] = {sd};
  qflash_status st = quantize_impl(xs, xqs, scs, 1, dtype, numel, s);
  if (st == QFLASH_OK && scale_host) {
    cudaError_t e = cudaMemcpyAsync(scale_host, sd, sizeof(float), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = cuda_fail(e, "scale D2H");
  }
  if (temp) cudaFreeAsync(sd, s);
  return st;
}

qflash_status qflash_quantize_qkv(const void* q, const void* k, const void* v, qflash_dtype dtype,
                                  int64_t numel, int8_t* q_q, int8_t* k_q, int8_t* v_q,
                                  float* scales_dev, qflash_stream_t stream) {
  if (!scales_dev) return fail(QFLASH_ERR_INVALID_ARGUMENT, "scales_dev is NULL");
  const void* xs[3] = {q, k, v};
  int8_t* xqs[3] = {q_q, k_q, v_q};
  float* scs[3] = {scales_dev, scales_dev + 1, scales_dev + 2};
  return quantize_impl(xs, xqs, scs, 3, dtype, numel, reinterpret_cast<cudaStream_t>(stream));
}

qflash_status qflash_quantize_qkv_prepare(const void* q, const void* k, const void* v,
                                          qflash_dtype dtype, int64_t numel, int8_t* q_q,
                                          int8_t* k_q, int8_t* v_q, float* scales_dev,
                                          int32_t head_dim, void* workspace_dev,
                                          qflash_stream_t stream) {
  if (!scales_dev) return fail(QFLASH_ERR_INVALID_ARGUMENT, "scales_dev is NULL");
  if (!workspace_dev || !aligned16(workspace_dev))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "workspace_dev NULL or misaligned");
  if (head_dim != 32 && head_dim != 64 && head_dim != 128)
    return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "head_dim %d not in {32, 64, 128}", head_dim);
  const void* xs[3] = {q, k, v};
  int8_t* xqs[3] = {q_q, k_q, v_q};
  float* scs[3] = {scales_dev, scales_dev + 1, scales_dev + 2};
  // workspace layout: [0, 128) integer constants, [256, ...) per-CTA amax partials
  return quantize_impl(xs, xqs, scs, 3, dtype, numel, reinterpret_cast<cudaStream_t>(stream),
                       reinterpret_cast<qf::IntParams*>(workspace_dev), head_dim,
                       reinterpret_cast<float*>(static_cast<char*>(workspace_dev) + 256));
}

qflash_status qflash_attention_int8_prepared(const int8_t* q, const int8_t* k, const int8_t* v,
                                             const qflash_attn_shape* shape,
                                             qflash_variant variant, int8_t* o,
                                             const void* workspace_dev, qflash_stream_t stream) {
  int bc = 0;
  qflash_status st = validate_shape(shape, &bc);
  if (st != QFLASH_OK) return st;
  const int64_t bytes = static_cast<int64_t>(shape->num_problems) * shape->seq_len * shape->head_dim;
  if ((st = validate_qkvo(q, k, v, o, bytes)) != QFLASH_OK) return st;
  if (!workspace_dev || !aligned16(workspace_dev))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "workspace_dev NULL or misaligned");
  int dev = 0;
  if ((st = check_device(&dev)) != QFLASH_OK) return st;
  return launch_common(q, k, v, shape, bc, variant, o, nullptr,
                       reinterpret_cast<const qf::IntParams*>(workspace_dev),
                       reinterpret_cast<cudaStream_t>(stream), nullptr, nullptr, 0);
}

qflash_status qflash_attention_dequant_prepared(const int8_t* q, const int8_t* k, const int8_t* v,
                                                const qflash_attn_shape* shape,
                                                qflash_variant variant, int8_t* o, float* y,
                                                const void* workspace_dev, qflash_stream_t stream) {
  int bc = 0;
  qflash_status st = validate_shape(shape, &bc);
  if (st != QFLASH_OK) return st;
  const int64_t n = static_cast<int64_t>(shape->num_problems) * shape->seq_len * shape->head_dim;
  if (!y || !aligned16(y)) return fail(QFLASH_ERR_INVALID_ARGUMENT, "y NULL or not 16-byte aligned");
  if (o != nullptr) {
    if ((st = validate_qkvo(q, k, v, o, n)) != QFLASH_OK) return st;
    if (overlaps(reinterpret_cast<const int8_t*>(y), 4 * n, o, n))
      return fail(QFLASH_ERR_INVALID_ARGUMENT, "y aliases o");
  } else {
    if (!q || !k || !v) return fail(QFLASH_ERR_INVALID_ARGUMENT, "NULL tensor pointer");
    if (!aligned16(q) || !aligned16(k) || !aligned16(v))
      return fail(QFLASH_ERR_INVALID_ARGUMENT, "tensor pointers must be 16-byte aligned");
  }
  const int8_t* yb = reinterpret_cast<const int8_t*>(y);
  if (overlaps(yb, 4 * n, q, n) || overlaps(yb, 4 * n, k, n) || overlaps(yb, 4 * n, v, n))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "y aliases q/k/v");
  if (!workspace_dev || !aligned16(workspace_dev))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "workspace_dev NULL or misaligned");
  int dev = 0;
  if ((st = check_device(&dev)) != QFLASH_OK) return st;
  return launch_common(q, k, v, shape, bc, variant, o, nullptr,
                       reinterpret_cast<const qf::IntParams*>(workspace_dev),
                       reinterpret_cast<cudaStream_t>(stream), y, nullptr, 0);
}

qflash_status qflash_forward_fused(const float* q, const float* k, const float* v,
                                   const qflash_attn_shape* shape, qflash_variant variant,
                                   int8_t* q_q, int8_t* k_q, int8_t* v_q, int8_t* o, float* y,
                                   float* scales_dev, void* workspace_dev,
                                   qflash_stream_t stream) {
  return qflash_forward_fused_amax(q, k, v, shape, variant, q_q, k_q, v_q, o, y, scales_dev,
                                   workspace_dev, nullptr, stream);
}

qflash_status qflash_forward_fused_per_head(const float* q, const float* k, const float* v, int32_t heads,
                                           const qflash_attn_shape* shape, qflash_variant variant,
                                           int8_t* q_q, int8_t* k_q, int8_t* v_q, float* y,
                                           float* scales_dev, void* workspace_dev, qflash_stream_t stream) {
  int bc = 0;
  qflash_status st = validate_shape(shape, &bc);
  if (st != QFLASH_OK) return st;
  if (heads < 1 || heads > qf::kMaxHeads || shape->num_problems % heads != 0)
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "heads must be in [1, %d] and divide num_problems",
                qf::kMaxHeads);
  const int64_t n = static_cast<int64_t>(shape->num_problems) * shape->seq_len * shape->head_dim;
  if (!q || !k || !v || !y || !scales_dev || !workspace_dev || !q_q || !k_q || !v_q)
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(y) || !aligned16(workspace_dev) ||
      !aligned16(q_q) || !aligned16(k_q) || !aligned16(v_q))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "all buffers must be 16-byte aligned");
  const void* ins[3] = {q, k, v};
  const int8_t* codes[3] = {q_q, k_q, v_q};
  const int8_t* yb = reinterpret_cast<const int8_t*>(y);
  const int8_t* ws = static_cast<const int8_t*>(workspace_dev);
  const int8_t* sc = reinterpret_cast<const int8_t*>(scales_dev);
  for (int i = 0; i < 3; ++i) {
    if (overlaps(yb, 4 * n, ins[i], 4 * n) || overlaps(yb, 4 * n, codes[i], n))
      return fail(QFLASH_ERR_INVALID_ARGUMENT, "y aliases a tensor");
    if (overlaps(ws, QFLASH_PH_FUSED_WORKSPACE_BYTES, ins[i], 4 * n) ||
        overlaps(ws, QFLASH_PH_FUSED_WORKSPACE_BYTES, codes[i], n) ||
        overlaps(sc, 12 * heads, ins[i], 4 * n) || overlaps(sc, 12 * heads, codes[i], n))
      return fail(QFLASH_ERR_INVALID_ARGUMENT, "workspace / scales alias a tensor");
    for (int j = 0; j < 3; ++j) {
      if (overlaps(codes[i], n, ins[j], 4 * n))
        return fail(QFLASH_ERR_INVALID_ARGUMENT, "int8 code buffer %d aliases input %d", i, j);
      if (j != i && overlaps(codes[i], n, codes[j], n))
        return fail(QFLASH_ERR_INVALID_ARGUMENT, "int8 code buffers %d and %d alias", i, j);
    }
  }
  if (overlaps(ws, QFLASH_PH_FUSED_WORKSPACE_BYTES, sc, 12 * heads) ||
      overlaps(ws, QFLASH_PH_FUSED_WORKSPACE_BYTES, yb, 4 * n) || overlaps(sc, 12 * heads, yb, 4 * n))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "workspace, scales and y must be disjoint");
  int dev = 0;
  if ((st = check_device(&dev)) != QFLASH_OK) return st;
  FusedIn fin;
  fin.x[0] = q;
  fin.x[1] = k;
  fin.x[2] = v;
  fin.xq[0] = q_q;
  fin.xq[1] = k_q;
  fin.xq[2] = v_q;
  fin.scales = scales_dev;
  fin.workspace = workspace_dev;
  fin.amax_in = nullptr;
  fin.qkv_heads = 0;
  return launch_common(q_q, k_q, v_q, shape, bc, variant, nullptr, nullptr, nullptr,
                       reinterpret_cast<cudaStream_t>(stream), y, &fin, heads);
}

qflash_status qflash_attention_int8_accum(const int8_t* q, const int8_t* k, const int8_t* v, float s_q,
                                         float s_k, const qflash_attn_shape* shape, int8_t* o,
                                         int32_t* flags_dev, qflash_stream_t stream) {
  int bc = 0;
  qflash_status st = validate_shape(shape, &bc);
  if (st != QFLASH_OK) return st;
  if (shape->head_dim == 128) return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "scale accumulation: head_dim 32 or 64");
  const int N = shape->seq_len;
  const int bc_eff = N <= bc ? (N <= 64 ? 64 : N <= 128 ? 128 : 256) : bc;
  if (bc_eff > 128) return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "scale accumulation: block_kv 64 or 128");
  const int64_t bytes = static_cast<int64_t>(shape->num_problems) * N * shape->head_dim;
  if ((st = validate_qkvo(q, k, v, o, bytes)) != QFLASH_OK) return st;
  if (!flags_dev || (reinterpret_cast<uintptr_t>(flags_dev) & 3u))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "flags_dev must be a 4-byte aligned device int32");
  if (overlaps(flags_dev, 4, o, bytes)) return fail(QFLASH_ERR_INVALID_ARGUMENT, "flags_dev aliases o");
  qf::IntParams prm;
  const int rc = qf::derive_core(s_q, s_k, shape->head_dim, &prm, nullptr);
  if (rc != QFLASH_OK) return fail(static_cast<qflash_status>(rc), "scale out of range");
  int dev = 0;
  if ((st = check_device(&dev)) != QFLASH_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(flags_dev, 0, 4, s);
  if (e != cudaSuccess) return cuda_fail(e, "flags reset");
  return launch_common(q, k, v, shape, bc, QFLASH_VARIANT_GENERIC, o, &prm, nullptr, s, nullptr, nullptr, 0,
                       nullptr, nullptr, nullptr, nullptr, flags_dev, 1);
}

qflash_status qflash_attention_ablation(const int8_t* q, const int8_t* k, const int8_t* v, float s_q,
                                       float s_k, float s_v, const qflash_attn_shape* shape,
                                       int32_t variant, float* y, qflash_stream_t stream) {
  int bc = 0;
  qflash_status st = validate_shape(shape, &bc);
  if (st != QFLASH_OK) return st;
  if (variant != QFLASH_ABLATION_V2 && variant != QFLASH_ABLATION_V3)
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "ablation variant %d not in {2 (V2), 3 (V3)}", variant);
  if (shape->head_dim == 128) return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "ablations: head_dim 32 or 64");
  const int N = shape->seq_len;
  const int bc_eff = N <= bc ? (N <= 64 ? 64 : N <= 128 ? 128 : 256) : bc;
  if (bc_eff > 128) return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "ablations: block_kv 64 or 128");
  const int64_t n = static_cast<int64_t>(shape->num_problems) * N * shape->head_dim;
  if (!q || !k || !v || !y) return fail(QFLASH_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(y))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "q, k, v, y must be 16-byte aligned");
  const int8_t* yb = reinterpret_cast<const int8_t*>(y);
  if (overlaps(yb, 4 * n, q, n) || overlaps(yb, 4 * n, k, n) || overlaps(yb, 4 * n, v, n))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "y aliases an input");
  if (!(s_v > 0.0f) || !std::isfinite(s_v)) return fail(QFLASH_ERR_SCALE_RANGE, "s_v must be positive");
  qf::IntParams prm;
  const int rc = qf::derive_core(s_q, s_k, shape->head_dim, &prm, nullptr);
  if (rc != QFLASH_OK) return fail(static_cast<qflash_status>(rc), "scale out of range");
  int dev = 0;
  if ((st = check_device(&dev)) != QFLASH_OK) return st;
  // internal variant numbering: 2 = V3 (integer exp, FP accumulation), 3 = V2 (FP exp)
  const int var = variant == QFLASH_ABLATION_V3 ? 2 : 3;
  return launch_common(q, k, v, shape, bc, QFLASH_VARIANT_GENERIC, nullptr, &prm, nullptr,
                       reinterpret_cast<cudaStream_t>(stream), y, nullptr, 0, nullptr, nullptr, nullptr,
                       nullptr, nullptr, var, s_v);
}

qflash_status qflash_amax_qkv(const float* q, const float* k, const float* v, int64_t numel,
                              float* amax_dev, qflash_stream_t stream) {
  if (numel < 0) return fail(QFLASH_ERR_INVALID_ARGUMENT, "numel < 0");
  if (!amax_dev || (numel > 0 && (!q || !k || !v)))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || (reinterpret_cast<uintptr_t>(amax_dev) & 3u))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "q, k, v must be 16-byte aligned, amax_dev 4-byte aligned");
  for (int i = 0; i < 3; ++i) {
    const float* x = i == 0 ? q : i == 1 ? k : v;
    if (numel > 0 && overlaps(reinterpret_cast<const int8_t*>(amax_dev), 12, x, 4 * numel))
      return fail(QFLASH_ERR_INVALID_ARGUMENT, "amax_dev aliases an input");
  }
  int dev = 0;
  qflash_status st;
  if ((st = check_device(&dev)) != QFLASH_OK) return st;
  cudaError_t e = qf::launch_amax3(q, k, v, numel, amax_dev, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "amax launch");
  return QFLASH_OK;
}

static qflash_status forward_fused_impl(const float* q, const float* k, const float* v, int qkv_heads,
                                        const qflash_attn_shape* shape, qflash_variant variant,
                                        int8_t* q_q, int8_t* k_q, int8_t* v_q, int8_t* o, float* y,
                                        float* scales_dev, void* workspace_dev, const float* amax_dev,
                                        qflash_stream_t stream);

qflash_status qflash_forward_fused_amax(const float* q, const float* k, const float* v,
                                        const qflash_attn_shape* shape, qflash_variant variant,
                                        int8_t* q_q, int8_t* k_q, int8_t* v_q, int8_t* o, float* y,
                                        float* scales_dev, void* workspace_dev, const float* amax_dev,
                                        qflash_stream_t stream) {
  return forward_fused_impl(q, k, v, 0, shape, variant, q_q, k_q, v_q, o, y, scales_dev, workspace_dev,
                            amax_dev, stream);
}

qflash_status qflash_forward_fused_qkv(const float* qkv, int32_t heads, const qflash_attn_shape* shape,
                                       qflash_variant variant, int8_t* q_q, int8_t* k_q, int8_t* v_q,
                                       int8_t* o, float* y, float* scales_dev, void* workspace_dev,
                                       qflash_stream_t stream) {
  if (!shape) return fail(QFLASH_ERR_INVALID_ARGUMENT, "shape is NULL");
  if (heads < 1 || shape->num_problems % heads != 0)
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "heads must be >= 1 and divide num_problems (%d, %d)",
                heads, shape->num_problems);
  return forward_fused_impl(qkv, qkv, qkv, heads, shape, variant, q_q, k_q, v_q, o, y, scales_dev,
                            workspace_dev, nullptr, stream);
}

static qflash_status forward_fused_impl(const float* q, const float* k, const float* v, int qkv_heads,
                                        const qflash_attn_shape* shape, qflash_variant variant,
                                        int8_t* q_q, int8_t* k_q, int8_t* v_q, int8_t* o, float* y,
                                        float* scales_dev, void* workspace_dev, const float* amax_dev,
                                        qflash_stream_t stream) {
  if (amax_dev != nullptr && (reinterpret_cast<uintptr_t>(amax_dev) & 3u))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "amax_dev must be 4-byte aligned");
  int bc = 0;
  qflash_status st = validate_shape(shape, &bc);
  if (st != QFLASH_OK) return st;
  const int64_t n = static_cast<int64_t>(shape->num_problems) * shape->seq_len * shape->head_dim;
  if (!q || !k || !v || !y || !scales_dev || !workspace_dev)
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(y) || !aligned16(workspace_dev))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "q, k, v, y and workspace_dev must be 16-byte aligned");
  const int8_t* outs[2] = {o, reinterpret_cast<const int8_t*>(y)};
  const int64_t out_n[2] = {n, 4 * n};
  if (o != nullptr) {
    if ((st = validate_qkvo(q_q, k_q, v_q, o, n)) != QFLASH_OK) return st;
  } else {
    if (!q_q || !k_q || !v_q) return fail(QFLASH_ERR_INVALID_ARGUMENT, "NULL int8 buffer");
    if (!aligned16(q_q) || !aligned16(k_q) || !aligned16(v_q))
      return fail(QFLASH_ERR_INVALID_ARGUMENT, "int8 buffers must be 16-byte aligned");
  }
  const void* ins[3] = {q, k, v};
  const int64_t in_bytes = qkv_heads > 0 ? 12 * n : 4 * n;  // packed QKV: one [P/H, N, 3, H, d] tensor
  const int8_t* codes[3] = {q_q, k_q, v_q};
  // every written buffer (codes, o, y) must be disjoint from every input and from
  // every other written buffer: the prologue re-reads inputs after other CTAs have
  // started writing codes, and the TMA loads read codes while y / o are written
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 2; ++j)
      if (outs[j] && overlaps(outs[j], out_n[j], ins[i], in_bytes))
        return fail(QFLASH_ERR_INVALID_ARGUMENT, "outputs alias the inputs");
    for (int j = 0; j < 3; ++j) {
      if (overlaps(codes[i], n, ins[j], in_bytes))
        return fail(QFLASH_ERR_INVALID_ARGUMENT, "int8 code buffer %d aliases input %d", i, j);
      if (j != i && overlaps(codes[i], n, codes[j], n))
        return fail(QFLASH_ERR_INVALID_ARGUMENT, "int8 code buffers %d and %d alias", i, j);
    }
    if (overlaps(reinterpret_cast<const int8_t*>(y), 4 * n, codes[i], n))
      return fail(QFLASH_ERR_INVALID_ARGUMENT, "int8 buffers alias y");
  }
  const int8_t* ws = static_cast<const int8_t*>(workspace_dev);
  for (int i = 0; i < 3; ++i)
    if (overlaps(ws, QFLASH_DSCALE_WORKSPACE_BYTES, ins[i], in_bytes) ||
        overlaps(ws, QFLASH_DSCALE_WORKSPACE_BYTES, codes[i], n))
      return fail(QFLASH_ERR_INVALID_ARGUMENT, "workspace aliases a tensor");
  int dev = 0;
  if ((st = check_device(&dev)) != QFLASH_OK) return st;
  FusedIn fin;
  fin.x[0] = q;
  fin.x[1] = k;
  fin.x[2] = v;
  fin.xq[0] = q_q;
  fin.xq[1] = k_q;
  fin.xq[2] = v_q;
  fin.scales = scales_dev;
  fin.workspace = workspace_dev;
  fin.amax_in = amax_dev;
  fin.qkv_heads = qkv_heads;
  if (amax_dev != nullptr) {
    const int8_t* am = reinterpret_cast<const int8_t*>(amax_dev);
    if (overlaps(am, 12, ws, QFLASH_DSCALE_WORKSPACE_BYTES) ||
        overlaps(am, 12, reinterpret_cast<const int8_t*>(scales_dev), 12) ||
        overlaps(am, 12, reinterpret_cast<const int8_t*>(y), 4 * n))
      return fail(QFLASH_ERR_INVALID_ARGUMENT, "amax_dev aliases a written buffer");
  }
  return launch_common(q_q, k_q, v_q, shape, bc, variant, o, nullptr, nullptr,
                       reinterpret_cast<cudaStream_t>(stream), y, &fin, 0);
}

static qflash_status dequant_impl(const int8_t* x_q, float scale, const float* scale_dev,
                                  int64_t numel, float* y, cudaStream_t stream) {
  if (!x_q || !y) return fail(QFLASH_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (numel < 0) return fail(QFLASH_ERR_INVALID_ARGUMENT, "numel < 0");
  if (!aligned16(x_q) || !aligned16(y))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "x_q and y must be 16-byte aligned");
  if (!scale_dev && (!std::isfinite(scale)))
    return fail(QFLASH_ERR_SCALE_RANGE, "scale must be finite");
  int dev = 0;
  qflash_status st = check_device(&dev);
  if (st != QFLASH_OK) return st;
  if (numel == 0) return QFLASH_OK;
  cudaError_t e = qf::launch_dequantize(x_q, scale, scale_dev, numel, y, stream);
  if (e != cudaSuccess) return cuda_fail(e, "dequantize launch");
  return QFLASH_OK;
}

qflash_status qflash_dequantize(const int8_t* x_q, float scale, int64_t numel, float* y,
                                qflash_stream_t stream) {
  return dequant_impl(x_q, scale, nullptr, numel, y, reinterpret_cast<cudaStream_t>(stream));
}

qflash_status qflash_dequantize_dscale(const int8_t* x_q, const float* scale_dev, int64_t numel,
                                       float* y, qflash_stream_t stream) {
  if (!scale_dev) return fail(QFLASH_ERR_INVALID_ARGUMENT, "scale_dev is NULL");
  return dequant_impl(x_q, 0.0f, scale_dev, numel, y, reinterpret_cast<cudaStream_t>(stream));
}

// ------------------------------------------------ per-head granularity
static qflash_status check_heads(int32_t P, int32_t H) {
  if (H < 1 || H > qf::kMaxHeads)
    return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "heads %d not in [1, %d]", H, qf::kMaxHeads);
  if (P % H != 0) return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "num_problems %d not a multiple of heads %d", P, H);
  // problem / H by umulhi(problem, ceil(2^32 / H)) is exact for problem < 2^32 / H^2
  if (static_cast<uint64_t>(P) * H * H >= (1ull << 32))
    return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "num_problems * heads^2 must be < 2^32");
  return QFLASH_OK;
}

qflash_status qflash_quantize_per_head(const float* q, const float* k, const float* v,
                                       int32_t num_problems, int32_t seq_len, int32_t head_dim,
                                       int32_t heads, int8_t* q_q, int8_t* k_q, int8_t* v_q,
                                       float* scales_dev, qflash_stream_t stream) {
  if (!q || !k || !v || !q_q || !k_q || !v_q || !scales_dev)
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (num_problems < 1 || seq_len < 1 || (head_dim != 32 && head_dim != 64 && head_dim != 128))
    return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "shape (%d, %d, %d)", num_problems, seq_len, head_dim);
  qflash_status st = check_heads(num_problems, heads);
  if (st != QFLASH_OK) return st;
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(q_q) || !aligned16(k_q) || !aligned16(v_q))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "pointers must be 16-byte aligned");
  int dev = 0;
  if ((st = check_device(&dev)) != QFLASH_OK) return st;
  qf::QuantTensors t;
  memset(&t, 0, sizeof(t));
  const void* xs[3] = {q, k, v};
  int8_t* xqs[3] = {q_q, k_q, v_q};
  for (int i = 0; i < 3; ++i) {
    t.x[i] = xs[i];
    t.xq[i] = xqs[i];
    t.scale[i] = scales_dev + i * heads;
  }
  const int64_t vpp = static_cast<int64_t>(seq_len) * head_dim / 4;
  cudaError_t e = qf::launch_quantize_per_head(t, 3, num_problems, vpp, heads,
                                               reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "per-head quantize launch");
  return QFLASH_OK;
}

qflash_status qflash_attention_int8_per_head(const int8_t* q, const int8_t* k, const int8_t* v,
                                             const float* scales_dev, int32_t heads,
                                             const qflash_attn_shape* shape, qflash_variant variant,
                                             int8_t* o, void* workspace_dev, qflash_stream_t stream) {
  int bc = 0;
  qflash_status st = validate_shape(shape, &bc);
  if (st != QFLASH_OK) return st;
  if ((st = check_heads(shape->num_problems, heads)) != QFLASH_OK) return st;
  const int64_t bytes = static_cast<int64_t>(shape->num_problems) * shape->seq_len * shape->head_dim;
  if ((st = validate_qkvo(q, k, v, o, bytes)) != QFLASH_OK) return st;
  if (!scales_dev || !workspace_dev || !aligned16(workspace_dev))
    return fail(QFLASH_ERR_INVALID_ARGUMENT, "scales_dev / workspace_dev NULL or misaligned");
  int dev = 0;
  if ((st = check_device(&dev)) != QFLASH_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = qf::launch_derive_per_head(scales_dev, heads, shape->head_dim, workspace_dev, s);
  if (e != cudaSuccess) return cuda_fail(e, "derive_per_head launch");
  return launch_common(q, k, v, shape, bc, variant, o, nullptr,
                       reinterpret_cast<const qf::IntParams*>(workspace_dev), s, nullptr, nullptr, heads);
}

qflash_status qflash_dequantize_per_head(const int8_t* x_q, const float* scales_dev,
                                         int32_t num_problems, int32_t seq_len, int32_t head_dim,
                                         int32_t heads, float* y, qflash_stream_t stream) {
  if (!x_q || !scales_dev || !y) return fail(QFLASH_ERR_INVALID_ARGUMENT, "NULL pointer");
  if (num_problems < 1 || seq_len < 1 || (head_dim != 32 && head_dim != 64 && head_dim != 128))
    return fail(QFLASH_ERR_UNSUPPORTED_SHAPE, "shape (%d, %d, %d)", num_problems, seq_len, head_dim);
  qflash_status st = check_heads(num_problems, heads);
  if (st != QFLASH_OK) return st;
  if (!aligned16(x_q) || !aligned16(y)) return fail(QFLASH_ERR_INVALID_ARGUMENT, "pointers must be 16-byte aligned");
  int dev = 0;
  if ((st = check_device(&dev)) != QFLASH_OK) return st;
  cudaError_t e = qf::launch_dequantize_per_head(x_q, scales_dev, num_problems,
                                                 static_cast<int64_t>(seq_len) * head_dim / 4, heads, y,
                                                 reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "per-head dequantize launch");
  return QFLASH_OK;
}

qflash_status qflash_debug_force_config(int32_t cfg) {
  if (cfg < -1 || cfg > 3) return fail(QFLASH_ERR_INVALID_ARGUMENT, "config %d not in [-1, 3]", cfg);
  g_force_config.store(cfg, std::memory_order_relaxed);
  return QFLASH_OK;
}

int32_t qflash_debug_last_config(void) { return g_last_config; }

// Bring-up entry (include/qflash_debug.h): qflash_attention_int8_ex plus raw
// dumps of S, P and the final (O, l) of CTA (problem 0, query tile 0).
qflash_status qflash_debug_attention(const int8_t* q, const int8_t* k, const int8_t* v, float s_q,
                                     float s_k, const qflash_attn_shape* shape,
                                     qflash_variant variant, int8_t* o, int32_t* dbg_s,
                                     int32_t* dbg_p, int32_t* dbg_o, long long* dbg_t,
                                     qflash_stream_t stream) {
  int bc = 0;
  qflash_status st = validate_shape(shape, &bc);
  if (st != QFLASH_OK) return st;
  qf::IntParams prm;
  const int rc = qf::derive_core(s_q, s_k, shape->head_dim, &prm, nullptr);
  if (rc != QFLASH_OK) return fail(static_cast<qflash_status>(rc), "scale out of range");
  int dev = 0;
  if ((st = check_device(&dev)) != QFLASH_OK) return st;
  return launch_common(q, k, v, shape, bc, variant, o, &prm, nullptr,
                       reinterpret_cast<cudaStream_t>(stream), nullptr, nullptr, 0, dbg_s, dbg_p, dbg_o, dbg_t);
}

}  // extern "C"
