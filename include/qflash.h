/*
 * qflash.h -- C ABI of libqflash.so: the B200 (sm_100a) hot path of QFlash,
 * integer-only fused attention (arxiv 2604.25306).
 *
 * Citations: "P:Lnnn" = line of the paper source; Eq./Alg. numbers are the
 * paper's; R# = a reading of an ambiguous passage.
 *
 * Conventions for every entry point
 *  - Memory: all tensors are DEVICE pointers on the current CUDA device unless a
 *    parameter says "host".  The caller owns every buffer; the library never
 *    allocates persistent device memory and keeps no mutable global state except
 *    a thread-local error string and per-device one-time setup (kernel
 *    attributes).  Layout: [P, N, d] int8 row-major, contiguous, 16-byte aligned.
 *  - Streams: work is enqueued on `stream` (cudaStream_t; NULL = legacy default
 *    stream) and is asynchronous unless a host output pointer is given.
 *  - Errors: arguments are validated before anything is enqueued; on error
 *    nothing is written.  CUDA failures return QFLASH_ERR_CUDA with details in
 *    qflash_last_error().  The functions never throw and never call exit().
 *  - Determinism: integer outputs are bit-identical across runs and equal to
 *    the CPU oracle (oracle/qflash_oracle.c) for the same inputs.
 */
#ifndef QFLASH_H_
#define QFLASH_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define QFLASH_API __attribute__((visibility("default")))
#else
#define QFLASH_API
#endif

typedef struct CUstream_st* qflash_stream_t; /* == cudaStream_t */

typedef enum {
  QFLASH_OK = 0,
  QFLASH_ERR_INVALID_ARGUMENT = 1,  /* null pointer, negative size, bad dtype, aliasing   */
  QFLASH_ERR_UNSUPPORTED_SHAPE = 2, /* d not in {32,64,128}; N<1 or N>65536; P<1;
                                       block_kv not in {0,64,128,256}                       */
  QFLASH_ERR_SCALE_RANGE = 3,       /* scale <= 0 or non-finite, or
                                       s = s_q*s_k*log2(e)/sqrt(d) outside [2^-24, 0.5]     */
  QFLASH_ERR_CUDA = 4,              /* CUDA runtime/driver error (see qflash_last_error)    */
  QFLASH_ERR_UNSUPPORTED_DEVICE = 5 /* current device is not compute capability 10.0       */
} qflash_status;

typedef enum { QFLASH_F32 = 0, QFLASH_BF16 = 1, QFLASH_F16 = 2 } qflash_dtype;

/* --------------------------------------------------------------------------
 * Eq. 2: per-tensor symmetric int8 quantization, dynamic scale
 * (computed on the fly).
 *   s   = fl32(max|x| / 127)   (all-zero tensor: s = 1/127, R3)
 *   x^  = sat8(roundf(fl32(x / s)))   round half away from zero (R1), IEEE fp32
 *         division (R2); bf16/f16 inputs are widened exactly to fp32.
 * x: device, numel elements of `dtype`, contiguous.  x_q: device int8[numel].
 * scale_dev: device float* receiving s (may be NULL).  scale_host: host float*
 * receiving s (may be NULL; if set the call synchronizes `stream`).  At least
 * one scale pointer is required.  numel == 0 gives s = 1/127 (x and x_q may then
 * be NULL).  A non-finite
 * input yields a non-finite s (rejected later by qflash_attention_int8).
 * ------------------------------------------------------------------------ */
QFLASH_API qflash_status qflash_quantize_per_tensor(const void* x, qflash_dtype dtype, int64_t numel,
                                         int8_t* x_q, float* scale_dev, float* scale_host,
                                         qflash_stream_t stream);

/* Fused Q/K/V variant: three tensors of identical dtype and numel quantized in
 * one amax launch and one quantize launch.  scales_dev: device float[3]
 * receiving (s_q, s_k, s_v), required.  Same semantics per tensor as above. */
QFLASH_API qflash_status qflash_quantize_qkv(const void* q, const void* k, const void* v, qflash_dtype dtype,
                                  int64_t numel, int8_t* q_q, int8_t* k_q, int8_t* v_q,
                                  float* scales_dev, qflash_stream_t stream);

typedef struct {
  int32_t num_problems; /* P = batch * windows * heads (windows folded into batch)   */
  int32_t seq_len;      /* N, 1..65536                                               */
  int32_t head_dim;     /* d in {32, 64, 128}                                        */
  int32_t block_kv;     /* B_c in {64, 128, 256}; 0 -> 128.  PART OF THE NUMERICAL
                           CONTRACT: the tiled result depends on B_c (R15).          */
} qflash_attn_shape;

/* Kernel tiling (tests / ablation); every variant gives identical bytes.
 *   GENERIC: one 128-row query tile of one problem per work item (ceil(N/128)
 *            tiles per problem, the last one ragged).
 *   PACKED:  the query rows of all problems are flattened and cut into 128-row
 *            tiles that may span up to 4 consecutive problems (Swin windows
 *            N = 49 pack 2.6 per tile; ViT N = 197 at batch 8 needs 148 tiles
 *            instead of 192).  Requires seq_len >= 43 and, for head_dim = 128,
 *            seq_len >= 127 with B_c <= 128; QFLASH_ERR_UNSUPPORTED_SHAPE otherwise.
 *   AUTO:    PACKED when supported and it needs fewer tiles, else GENERIC. */
typedef enum {
  QFLASH_VARIANT_AUTO = 0,
  QFLASH_VARIANT_GENERIC = 1,
  QFLASH_VARIANT_PACKED = 2
} qflash_variant;

/* --------------------------------------------------------------------------
 * Algorithm 1: QFlash integer-only fused attention forward.
 * q, k, v: device int8 [P, N, d] (Q^, K^, V^ of Eq. 2, per-tensor scales s_q,
 * s_k, s_v given on the host).  o: device int8 [P, N, d], must not alias
 * q/k/v.  s_o: host float* receiving s_O = s_V, may be NULL.
 * Per problem and query row (all integer):
 *   S = Q K_j^T (int32, Eq. 3); m' = max(m, rowmax S) (Eq. 4);
 *   alpha = ShiftExp2(m - m') and P~ = ShiftExp2(S - m') (Alg. 2, Eq. 5-8,
 *   exact quotient R6); P = min(127, (P~ M_P) >> r_P) (Eq. 9-10, s_P = 1/127);
 *   l = floor(l alpha / s_inv) + rowsum P; O = floor(O alpha / s_inv) + P V_j
 *   (ScaleRelease, Eq. 14 / P:L408); out = sat8(floor(O / l)) (step 11).
 * Asynchronous on `stream`; no allocation, no host synchronization.
 * ------------------------------------------------------------------------ */
QFLASH_API qflash_status qflash_attention_int8(const int8_t* q, const int8_t* k, const int8_t* v, float s_q,
                                    float s_k, float s_v, const qflash_attn_shape* shape,
                                    int8_t* o, float* s_o, qflash_stream_t stream);

/* Same as qflash_attention_int8 with an explicit kernel variant. */
QFLASH_API qflash_status qflash_attention_int8_ex(const int8_t* q, const int8_t* k, const int8_t* v,
                                       float s_q, float s_k, float s_v,
                                       const qflash_attn_shape* shape, qflash_variant variant,
                                       int8_t* o, float* s_o, qflash_stream_t stream);

/* Device-scale variant for fully asynchronous pipelines (dynamic quantization,
 * P:L703): scales_dev = device float[3] holding (s_q, s_k, s_v), e.g. as written
 * by qflash_quantize_qkv.  A one-thread kernel derives the integer constants on
 * the device with the same fp64 expression (no FMA contraction) as
 * qflash_derive_params and stores them in workspace_dev (caller-owned device
 * memory of QFLASH_DSCALE_WORKSPACE_BYTES bytes, 16-byte aligned); the
 * attention kernel reads them there.  No host synchronization.  If the scales
 * are out of range nothing is written to o and the int32 at workspace_dev[0]
 * holds QFLASH_ERR_SCALE_RANGE (QFLASH_OK otherwise).  s_O = s_V stays in
 * scales_dev[2]. */
#define QFLASH_DSCALE_WORKSPACE_BYTES 8192
QFLASH_API qflash_status qflash_attention_int8_dscale(const int8_t* q, const int8_t* k, const int8_t* v,
                                           const float* scales_dev,
                                           const qflash_attn_shape* shape, qflash_variant variant,
                                           int8_t* o, void* workspace_dev,
                                           qflash_stream_t stream);

/* The fused step for dynamic quantization without an extra launch:
 * qflash_quantize_qkv_prepare = qflash_quantize_qkv that also derives the
 * attention's integer constants from the final (s_q, s_k) on the device (block 0
 * of the quantize kernel, same fp64 expression as qflash_derive_params) into
 * workspace_dev (QFLASH_DSCALE_WORKSPACE_BYTES, 16-byte aligned; int32 status at
 * offset 0; bytes 256..4095 hold per-CTA amax partials, bytes 4096..5119 the
 * 256-entry dequantization table fl32(s_V * i), i = -128..127).  When Q, K and V fit in the
 * GPU's aggregate shared memory the quantization is a single cooperative pass
 * (HBM read once); otherwise amax and quantize are two streaming launches.  qflash_attention_int8_prepared then runs Algorithm 1 with the
 * constants found in workspace_dev (nothing is written to o if the status is
 * not QFLASH_OK).  head_dim must be the d of the following attention call. */
QFLASH_API qflash_status qflash_quantize_qkv_prepare(const void* q, const void* k, const void* v,
                                                     qflash_dtype dtype, int64_t numel,
                                                     int8_t* q_q, int8_t* k_q, int8_t* v_q,
                                                     float* scales_dev, int32_t head_dim,
                                                     void* workspace_dev, qflash_stream_t stream);
QFLASH_API qflash_status qflash_attention_int8_prepared(const int8_t* q, const int8_t* k,
                                                        const int8_t* v,
                                                        const qflash_attn_shape* shape,
                                                        qflash_variant variant, int8_t* o,
                                                        const void* workspace_dev,
                                                        qflash_stream_t stream);

/* Algorithm 1 fused with the dequantization of its output (the DQ step): after
 * qflash_quantize_qkv_prepare, writes y = fl32(s_V * (float)O^) (fp32 [P, N, d],
 * s_O = s_V) straight from the attention epilogue -- bit-identical to
 * qflash_attention_int8_prepared followed by qflash_dequantize_dscale, one launch
 * and one HBM pass fewer.  The epilogue stays integer-only: the fp32 bit pattern
 * of every int8 value comes from a 256-entry table that the quantize kernel
 * computed with the same IEEE multiply (workspace_dev bytes 4096..5119).  o (int8
 * [P, N, d]) may be NULL; if given it receives O^ as well.  Nothing is written if
 * the device-derived status is not QFLASH_OK. */
QFLASH_API qflash_status qflash_attention_dequant_prepared(const int8_t* q, const int8_t* k,
                                                           const int8_t* v,
                                                           const qflash_attn_shape* shape,
                                                           qflash_variant variant, int8_t* o,
                                                           float* y, const void* workspace_dev,
                                                           qflash_stream_t stream);

/* The whole hot path in ONE launch (fp32 inputs): per-tensor quantization of Q,
 * K, V (Eq. 2, dynamic scales P:L703) in a cooperative prologue of the attention
 * kernel (amax over a grid-stride share, grid barrier, scales + integer
 * constants + dequant table derived identically in every CTA, int8 codes written
 * to q_q / k_q / v_q, grid barrier), then Algorithm 1 on those codes and the
 * fused dequantization y = fl32(s_V * O^).  Bit-identical to
 * qflash_quantize_qkv_prepare + qflash_attention_dequant_prepared.  q, k, v:
 * device fp32 [P, N, d]; q_q, k_q, v_q: device int8 [P, N, d] (written); o:
 * optional int8 O^; y: device fp32 [P, N, d]; scales_dev: device float[3]
 * (written: s_q, s_k, s_v); workspace_dev: QFLASH_DSCALE_WORKSPACE_BYTES (same
 * layout as the prepare path).  All pointers 16-byte aligned, outputs must not
 * alias inputs.  Launched cooperatively (every CTA resident, one per SM). */
QFLASH_API qflash_status qflash_forward_fused(const float* q, const float* k, const float* v,
                                              const qflash_attn_shape* shape,
                                              qflash_variant variant, int8_t* q_q, int8_t* k_q,
                                              int8_t* v_q, int8_t* o, float* y,
                                              float* scales_dev, void* workspace_dev,
                                              qflash_stream_t stream);

/* Sharded per-tensor quantization (Eq. 2 P:L241-246 with dynamic
 * scales P:L703).  When several GPUs each hold a slab of ONE logical [P, N, d]
 * tensor (contiguous problem ranges, qflash_partition), the per-tensor scale
 * s = fl32(amax / 127) must be the amax over every slab:
 *   qflash_amax_qkv        amax_dev[t] = max |x_t| over this device's slab of Q, K,
 *                          V (fp32, numel elements each; device float[3], written;
 *                          0 for numel = 0).  Inputs 16-byte aligned.
 *   (caller)               MAX all-reduce of the 3 floats across the ranks
 *   qflash_forward_fused_amax  qflash_forward_fused with the amax taken from
 *                          amax_dev (device float[3], read) instead of computed: no
 *                          amax pass and no first grid barrier.  amax_dev = NULL is
 *                          qflash_forward_fused.  The output of each slab is then
 *                          byte-identical to the same rows of a 1-GPU run on the
 *                          whole tensor.  amax_dev must not alias a written buffer.
 * Errors as qflash_forward_fused; asynchronous on `stream`. */
QFLASH_API qflash_status qflash_amax_qkv(const float* q, const float* k, const float* v,
                                         int64_t numel, float* amax_dev, qflash_stream_t stream);
QFLASH_API qflash_status qflash_forward_fused_amax(const float* q, const float* k, const float* v,
                                                   const qflash_attn_shape* shape,
                                                   qflash_variant variant, int8_t* q_q,
                                                   int8_t* k_q, int8_t* v_q, int8_t* o, float* y,
                                                   float* scales_dev, void* workspace_dev,
                                                   const float* amax_dev, qflash_stream_t stream);

/* qflash_forward_fused on the packed output of a QKV projection (
 * dynamic quantization of the projection output P:L703, Eq. 2): qkv is
 * ONE device fp32 tensor [P / heads, N, 3, heads, d] (batch x windows, tokens, {Q, K, V},
 * heads, channels -- a Linear(d_model, 3 d_model) output viewed per head), problem p =
 * b heads + h.  The prologue reads it with the (token, head) transpose and writes the
 * [P, N, d] codes q_q / k_q / v_q itself: no permute pass.  heads must divide P.  The
 * result equals qflash_forward_fused on the three permuted tensors byte for byte.
 * Other arguments and errors as qflash_forward_fused (qkv 16-byte aligned). */
QFLASH_API qflash_status qflash_forward_fused_qkv(const float* qkv, int32_t heads,
                                                  const qflash_attn_shape* shape, qflash_variant variant,
                                                  int8_t* q_q, int8_t* k_q, int8_t* v_q, int8_t* o,
                                                  float* y, float* scales_dev, void* workspace_dev,
                                                  qflash_stream_t stream);

/* Scale Accumulation ablation (Eq. 13, App. B.1
 * P:L762-805) -- the alternative the paper REJECTS, for the fig:tile_sqnr
 * experiment only.  Algorithm 1 with step (8)(10) replaced by
 *   O <- O alpha + (P V_j) s_inv,   l <- l alpha + rowsum(P_j) s_inv
 * (floor(PV / s_alpha) with the integer inverse scale, reading R24) in int64, then
 * O^ = sat8(floor(O / l)) (0 when l <= 0).  Values that leave int64 wrap modulo 2^64
 * exactly like the CPU oracle's mode 1.  *flags_dev (device int32, written): bit 0 =
 * some accumulator left int64, bit 1 = some accumulator left int32 (where an
 * int32-accumulator kernel overflows).  Generic tiles, head_dim 32/64, block_kv
 * 64/128; other arguments and errors as qflash_attention_int8 (s_O = s_V). */
QFLASH_API qflash_status qflash_attention_int8_accum(const int8_t* q, const int8_t* k, const int8_t* v,
                                                     float s_q, float s_k, const qflash_attn_shape* shape,
                                                     int8_t* o, int32_t* flags_dev, qflash_stream_t stream);

/* The whole per-head step in ONE cooperative launch (per-head scales
 * P:L221): fp32 q, k, v [P, N, d] (head = problem mod heads, heads <= 96,
 * dividing P) -> per-(tensor, head) quantization in the kernel's prologue -> Algorithm 1
 * with head h's constants -> y = fl32(s_V[h] O^).  scales_dev: device float[3 heads]
 * (written: s_q[h], s_k[h], s_v[h]); q_q / k_q / v_q: int8 codes (written); workspace_dev:
 * QFLASH_PH_FUSED_WORKSPACE_BYTES, ZERO-FILLED before its first use (the kernel keeps its
 * per-(tensor, head) amax accumulators there and re-zeroes them at the end of every call;
 * the status of the constant derivation is its first int32, the head table follows at 128).
 * Bit-identical to qflash_quantize_per_head + qflash_attention_int8_per_head +
 * qflash_dequantize_per_head.  block_kv <= 128. */
#define QFLASH_PH_FUSED_WORKSPACE_BYTES 16384
QFLASH_API qflash_status qflash_forward_fused_per_head(const float* q, const float* k, const float* v,
                                                       int32_t heads, const qflash_attn_shape* shape,
                                                       qflash_variant variant, int8_t* q_q, int8_t* k_q,
                                                       int8_t* v_q, float* y, float* scales_dev,
                                                       void* workspace_dev, qflash_stream_t stream);

/* Ablation steps of the paper's Table on the same kernel
 * skeleton (int8 Q K^T and int8 P V on tcgen05, generic tiles, configuration 0):
 *   QFLASH_ABLATION_V3: integer ShiftExp2 + requant (the method's P bytes), but O and l
 *       accumulated in fp32: O <- O (alpha / s_inv) + P V_j (no integer ScaleRelease);
 *   QFLASH_ABLATION_V2: floating-point softmax: P = rint(127 exp2(s (S - m))) with
 *       ex2.approx, alpha = exp2(s (m_old - m_new)), int8 P V, fp32 accumulation.
 * y: device fp32 [P, N, d] = s_v O / l.  Not integer-only and not bit-exact to anything:
 * for the speed / accuracy comparison with the method (qflash_attention_int8 = V4).
 * head_dim 32/64, block_kv 64/128; errors as qflash_attention_int8. */
#define QFLASH_ABLATION_V2 2
#define QFLASH_ABLATION_V3 3
QFLASH_API qflash_status qflash_attention_ablation(const int8_t* q, const int8_t* k, const int8_t* v,
                                                   float s_q, float s_k, float s_v,
                                                   const qflash_attn_shape* shape, int32_t variant,
                                                   float* y, qflash_stream_t stream);

/* --------------------------------------------------------------------------
 * Per-head granularity (the paper's per-tensor scales are the
 * H = 1 case).  Problems are the flattened (batch,
 * window, head) with the head fastest, so head = problem mod H; every head gets
 * its own (s_q, s_k, s_v) and hence its own integer constants.  Bit-identical to
 * running the per-tensor path on each head's problems separately.
 *   H in [1, 96], num_problems a multiple of H, num_problems * H^2 < 2^32.
 * qflash_quantize_per_head: fp32 q, k, v [P, N, d] -> int8 codes; scales_dev =
 *   device float[3 H] written as (s_q[0..H), s_k[0..H), s_v[0..H)).
 * qflash_attention_int8_per_head: Algorithm 1 with head h's constants derived on
 *   the device from scales_dev (same layout) into workspace_dev
 *   (QFLASH_DSCALE_WORKSPACE_BYTES; int32 status at offset 0, nothing written to o
 *   if a head's scales are out of range); s_O[h] = s_V[h].
 * qflash_dequantize_per_head: y = fl32(s[head] * x^), scales_dev = device float[H]
 *   (e.g. scales_dev + 2 H of the calls above). */
QFLASH_API qflash_status qflash_quantize_per_head(const float* q, const float* k, const float* v,
                                                  int32_t num_problems, int32_t seq_len,
                                                  int32_t head_dim, int32_t heads, int8_t* q_q,
                                                  int8_t* k_q, int8_t* v_q, float* scales_dev,
                                                  qflash_stream_t stream);
QFLASH_API qflash_status qflash_attention_int8_per_head(const int8_t* q, const int8_t* k,
                                                        const int8_t* v, const float* scales_dev,
                                                        int32_t heads,
                                                        const qflash_attn_shape* shape,
                                                        qflash_variant variant, int8_t* o,
                                                        void* workspace_dev,
                                                        qflash_stream_t stream);
QFLASH_API qflash_status qflash_dequantize_per_head(const int8_t* x_q, const float* scales_dev,
                                                    int32_t num_problems, int32_t seq_len,
                                                    int32_t head_dim, int32_t heads, float* y,
                                                    qflash_stream_t stream);

/* Inverse of Eq. 2: y = fl32(scale * (float)x^).  x_q device int8[numel],
 * y device float[numel]. */
QFLASH_API qflash_status qflash_dequantize(const int8_t* x_q, float scale, int64_t numel, float* y,
                                qflash_stream_t stream);
/* Same with the scale read from device memory (scale_dev: device float*). */
QFLASH_API qflash_status qflash_dequantize_dscale(const int8_t* x_q, const float* scale_dev, int64_t numel,
                                       float* y, qflash_stream_t stream);

/* --------------------------------------------------------------------------
 * Pure host helpers (no CUDA calls; usable without a GPU).
 * ------------------------------------------------------------------------ */
typedef struct {
  double s;           /* s = s_q s_k d^(-1/2) log2(e)  */
  int32_t s_inv;      /* round(1/s)  */
  int32_t n;          /* floor(log2(127 s))                              (Eq. 9)   */
  int32_t r_p;        /* 8 - n                                           (Eq. 9)   */
  int32_t m_p;        /* round(127 s 2^r_p)                              (Eq. 10)  */
  /* realisation constants of the kernel (division-free, exact):            */
  uint32_t q_magic;   /* floor(t / s_inv) == umulhi(t, q_magic) >> q_shift          */
  int32_t q_shift;    /*   for every t the kernel can produce (t < 2^25)            */
  uint32_t p_mul;     /* floor(y M_P / 2^r_P) == umulhi(y << p_pre, p_mul)          */
  int32_t p_pre;
  int32_t p_max;      /* floor(s_inv M_P / 2^r_P): largest P before the 127 clamp  */
  uint64_t rel_magic; /* floor(n / s_inv) == umul64hi(n, rel_magic) >> rel_shift    */
  int32_t rel_shift;  /*   for n < 2^56 (ScaleRelease per-row constant)            */
} qflash_int_params;

/* Derive every constant of one attention call from the host scales.
 * Returns QFLASH_ERR_SCALE_RANGE / UNSUPPORTED_SHAPE / INVALID_ARGUMENT. */
QFLASH_API qflash_status qflash_derive_params(float s_q, float s_k, int32_t head_dim,
                                   qflash_int_params* out);

/* Contiguous split of P independent problems over `world` ranks:
 * rank r gets [floor(r P / world), floor((r+1) P / world)).  Invalid input
 * (P < 0, world < 1, rank outside [0, world)) yields begin = count = 0. */
QFLASH_API void qflash_partition(int32_t num_problems, int32_t world, int32_t rank, int32_t* begin,
                      int32_t* count);

QFLASH_API const char* qflash_status_string(qflash_status status);
QFLASH_API const char* qflash_last_error(void); /* thread-local detail of the last failure */

/* Library/ABI version: (major << 16) | minor. */
QFLASH_API int32_t qflash_version(void);

#ifdef __cplusplus
}
#endif

#endif /* QFLASH_H_ */
