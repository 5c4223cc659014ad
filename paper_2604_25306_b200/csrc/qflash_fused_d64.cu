// qflash_fused_d64.cu -- fused-step instantiations (FQ: fp32 Q/K/V quantized in the
// kernel's cooperative prologue, attention, dequantized fp32 output), d = 64.
#include "qflash_attn_inst.cuh"

namespace qf {
cudaError_t launch_fused_d64(int BC, int nseg, int cfg, const CUtensorMap& tq,
                             const CUtensorMap& tk, const CUtensorMap& tv, const AttnArgs& args,
                             int64_t tiles, int sms, cudaStream_t stream) {
  return launch_attention_d<64, false, 1>(BC, nseg, cfg, tq, tk, tv, args, tiles, sms, stream);
}
}  // namespace qf
