// qflash_attn_inst.cuh -- instantiation helper: one translation unit per head
// dimension (qflash_attn_d32.cu, ...) defines launch_attention_d<D>() over every
// supported (B_c, NSEG, CS, QT) so the heavy kernel instantiations compile in
// parallel.  Configurations that do not fit TMEM / shared memory report
// cudaErrorNotSupported without instantiating anything.
#pragma once
#include "qflash_attn_kernel.cuh"

namespace qf {

template <int D, int BC, int NSEG, int CS, int QT, bool DBG, int FQ, bool PH = false, int VAR = 0>
cudaError_t try_launch(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                       const AttnArgs& args, int64_t tiles, int sms, cudaStream_t stream) {
  if constexpr (config_fits<D, BC, NSEG, CS, QT>()) {
    // the fused per-head step also keeps its head area in shared memory
    if constexpr (FQ && PH && Cfg<D, BC, NSEG, CS, QT>::kAlloc + kHeadAreaBytes > 227 * 1024)
      return cudaErrorNotSupported;
    else
      return launch_attn_t<D, BC, NSEG, CS, QT, DBG, FQ, PH, VAR>(tq, tk, tv, args, tiles, sms, stream);
  } else {
    return cudaErrorNotSupported;
  }
}

// cfg 0: CS = 4 column splits x QT = 1 (one query tile in flight, 16 softmax warps)
// cfg 1: CS = 2 x QT = 2 (two ping-ponging query tiles, 8 softmax warps each)
// cfg 2: CS = 1 x QT = 2 (two ping-ponging query tiles, each a row-owner softmax
//        warpgroup + a correction warpgroup)
// cfg 3: CS = 1 x QT = 1
template <int D, bool DBG, int FQ = 0>
cudaError_t launch_attention_d(int BC, int nseg, int cfg, const CUtensorMap& tq,
                               const CUtensorMap& tk, const CUtensorMap& tv, const AttnArgs& args,
                               int64_t tiles, int sms, cudaStream_t stream) {
#define QF_BC_SEG(bc, ns)                                                                      \
  if (BC == bc && nseg == ns)                                                                  \
    return cfg == 1   ? try_launch<D, bc, ns, 2, 2, DBG, FQ>(tq, tk, tv, args, tiles, sms, stream) \
           : cfg == 2 ? try_launch<D, bc, ns, 1, 2, DBG, FQ>(tq, tk, tv, args, tiles, sms, stream) \
           : cfg == 3 ? try_launch<D, bc, ns, 1, 1, DBG, FQ>(tq, tk, tv, args, tiles, sms, stream) \
                      : try_launch<D, bc, ns, 4, 1, DBG, FQ>(tq, tk, tv, args, tiles, sms, stream);
  QF_BC_SEG(64, 1) QF_BC_SEG(128, 1) QF_BC_SEG(256, 1)
  QF_BC_SEG(64, 2) QF_BC_SEG(128, 2) QF_BC_SEG(256, 2)
  QF_BC_SEG(64, 4) QF_BC_SEG(128, 4)
#undef QF_BC_SEG
  return cudaErrorNotSupported;
}

// Per-head constants: cfg 0 (CS = 4 x QT = 1) for every (B_c, NSEG), and cfg 1 (CS = 2 x
// QT = 2: multi-wave with several KV tiles, e.g. L14) for generic tiles.
template <int D>
cudaError_t launch_attention_ph_d(int BC, int nseg, int cfg, const CUtensorMap& tq, const CUtensorMap& tk,
                                  const CUtensorMap& tv, const AttnArgs& args, int64_t tiles,
                                  int sms, cudaStream_t stream) {
  if (cfg == 1 && nseg == 1) {
    if (BC == 64) return try_launch<D, 64, 1, 2, 2, false, 0, true>(tq, tk, tv, args, tiles, sms, stream);
    if (BC == 128) return try_launch<D, 128, 1, 2, 2, false, 0, true>(tq, tk, tv, args, tiles, sms, stream);
  }
#define QF_PH(bc, ns)           \
  if (BC == bc && nseg == ns)   \
    return try_launch<D, bc, ns, 4, 1, false, 0, true>(tq, tk, tv, args, tiles, sms, stream);
  QF_PH(64, 1) QF_PH(128, 1) QF_PH(256, 1)
  QF_PH(64, 2) QF_PH(128, 2) QF_PH(256, 2)
  QF_PH(64, 4) QF_PH(128, 4)
#undef QF_PH
  return cudaErrorNotSupported;
}

// Ablation variants (generic tiles, configuration 0): VAR 1 = Scale Accumulation (Eq. 13,
// App. B.1), VAR 2 = V3 (integer exp, FP accumulation), VAR 3 = V2 (FP exp2, int8 P V).
template <int D, int VAR>
cudaError_t launch_attention_var_d(int BC, const CUtensorMap& tq, const CUtensorMap& tk,
                                   const CUtensorMap& tv, const AttnArgs& args, int64_t tiles, int sms,
                                   cudaStream_t stream) {
  if (BC == 64) return try_launch<D, 64, 1, 4, 1, false, 0, false, VAR>(tq, tk, tv, args, tiles, sms, stream);
  if (BC == 128) return try_launch<D, 128, 1, 4, 1, false, 0, false, VAR>(tq, tk, tv, args, tiles, sms, stream);
  return cudaErrorNotSupported;
}

// Fused per-head step (FQ + PH): cfg 0 for every (B_c, NSEG) with B_c <= 128, cfg 1 for
// generic tiles.
template <int D>
cudaError_t launch_fused_ph_d(int BC, int nseg, int cfg, const CUtensorMap& tq, const CUtensorMap& tk,
                              const CUtensorMap& tv, const AttnArgs& args, int64_t tiles, int sms,
                              cudaStream_t stream) {
  if (cfg == 1 && nseg == 1) {
    if (BC == 64) return try_launch<D, 64, 1, 2, 2, false, 1, true>(tq, tk, tv, args, tiles, sms, stream);
    if (BC == 128) return try_launch<D, 128, 1, 2, 2, false, 1, true>(tq, tk, tv, args, tiles, sms, stream);
  }
#define QF_FPH(bc, ns)          \
  if (BC == bc && nseg == ns)   \
    return try_launch<D, bc, ns, 4, 1, false, 1, true>(tq, tk, tv, args, tiles, sms, stream);
  QF_FPH(64, 1) QF_FPH(128, 1)
  QF_FPH(64, 2) QF_FPH(128, 2)
  QF_FPH(64, 4) QF_FPH(128, 4)
#undef QF_FPH
  return cudaErrorNotSupported;
}

template <int D>
constexpr bool supported_d(int BC, int nseg, int cfg) {
#define QF_FITS(bc, ns)                                                                 \
  if (BC == bc && nseg == ns)                                                           \
    return cfg == 1   ? config_fits<D, bc, ns, 2, 2>()                  \
           : cfg == 2 ? config_fits<D, bc, ns, 1, 2>()                  \
           : cfg == 3 ? config_fits<D, bc, ns, 1, 1>()                  \
                      : config_fits<D, bc, ns, 4, 1>();
  QF_FITS(64, 1) QF_FITS(128, 1) QF_FITS(256, 1)
  QF_FITS(64, 2) QF_FITS(128, 2) QF_FITS(256, 2)
  QF_FITS(64, 4) QF_FITS(128, 4)
#undef QF_FITS
  return false;
}

}  // namespace qf
