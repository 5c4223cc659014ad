// qflash_attn_acc.cu -- instantiations of the Scale Accumulation ablation (Eq. 13,
// App. B.1): int64 accumulation of O and l in registers with overflow flags.
#include "qflash_attn_inst.cuh"

namespace qf {
cudaError_t launch_attention_acc(int D, int BC, const CUtensorMap& tq, const CUtensorMap& tk,
                                 const CUtensorMap& tv, const AttnArgs& args, int64_t tiles, int sms,
                                 cudaStream_t stream) {
  if (D == 32) return launch_attention_acc_d<32>(BC, tq, tk, tv, args, tiles, sms, stream);
  if (D == 64) return launch_attention_acc_d<64>(BC, tq, tk, tv, args, tiles, sms, stream);
  return cudaErrorNotSupported;
}
}  // namespace qf
