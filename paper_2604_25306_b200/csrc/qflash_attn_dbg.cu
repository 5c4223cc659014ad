// qflash_attn_dbg.cu -- bring-up instantiations (DBG = true: clock64 timeline and
// S / P / O dumps of CTA 0, group 0, first tile) for d in {32, 64}.  Used only by
// qflash_debug_attention (include/qflash_debug.h).
#include "qflash_attn_inst.cuh"

namespace qf {
cudaError_t launch_attention_dbg(int D, int BC, int nseg, int cfg, const CUtensorMap& tq,
                                 const CUtensorMap& tk, const CUtensorMap& tv,
                                 const AttnArgs& args, int64_t tiles, int sms,
                                 cudaStream_t stream) {
  if (D == 32) return launch_attention_d<32, true>(BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
  if (D == 64) return launch_attention_d<64, true>(BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
  return cudaErrorNotSupported;
}
}  // namespace qf
