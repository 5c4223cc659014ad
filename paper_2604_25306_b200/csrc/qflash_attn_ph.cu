// qflash_attn_ph.cu -- per-head-constant instantiations of the attention kernel
// (configuration 0, every head dimension).
#include "qflash_attn_inst.cuh"

namespace qf {
cudaError_t launch_attention_ph(int D, int BC, int nseg, int cfg, const CUtensorMap& tq,
                                const CUtensorMap& tk, const CUtensorMap& tv,
                                const AttnArgs& args, int64_t tiles, int sms,
                                cudaStream_t stream) {
  if (D == 32) return launch_attention_ph_d<32>(BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
  if (D == 64) return launch_attention_ph_d<64>(BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
  if (D == 128) return launch_attention_ph_d<128>(BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
  return cudaErrorNotSupported;
}
cudaError_t launch_fused_ph(int D, int BC, int nseg, int cfg, const CUtensorMap& tq, const CUtensorMap& tk,
                            const CUtensorMap& tv, const AttnArgs& args, int64_t tiles, int sms,
                            cudaStream_t stream) {
  if (D == 32) return launch_fused_ph_d<32>(BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
  if (D == 64) return launch_fused_ph_d<64>(BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
  if (D == 128) return launch_fused_ph_d<128>(BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
  return cudaErrorNotSupported;
}
}  // namespace qf
