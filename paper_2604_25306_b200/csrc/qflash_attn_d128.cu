// qflash_attn_d128.cu -- production instantiations of the attention kernel, d = 128.
#include "qflash_attn_inst.cuh"

namespace qf {
cudaError_t launch_attention_d128(int BC, int nseg, int cfg, const CUtensorMap& tq,
                                 const CUtensorMap& tk, const CUtensorMap& tv,
                                 const AttnArgs& args, int64_t tiles, int sms,
                                 cudaStream_t stream) {
  return launch_attention_d<128, false>(BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
}
bool attention_supported_d128(int BC, int nseg, int cfg) { return supported_d<128>(BC, nseg, cfg); }
}  // namespace qf
