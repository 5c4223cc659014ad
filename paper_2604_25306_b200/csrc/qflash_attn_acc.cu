// qflash_attn_acc.cu -- instantiations of the ablation variants of the attention kernel:
// Scale Accumulation (Eq. 13, App. B.1) and the V3 / V2 steps of
// the paper's ablation (N4): integer exp with FP accumulation, FP exp with int8 P V.
#include "qflash_attn_inst.cuh"

namespace qf {
cudaError_t launch_attention_var(int var, int D, int BC, const CUtensorMap& tq, const CUtensorMap& tk,
                                 const CUtensorMap& tv, const AttnArgs& args, int64_t tiles, int sms,
                                 cudaStream_t stream) {
#define QF_VAR(v)                                                                            \
  if (var == v) {                                                                            \
    if (D == 32) return launch_attention_var_d<32, v>(BC, tq, tk, tv, args, tiles, sms, stream); \
    if (D == 64) return launch_attention_var_d<64, v>(BC, tq, tk, tv, args, tiles, sms, stream); \
  }
  QF_VAR(1) QF_VAR(2) QF_VAR(3)
#undef QF_VAR
  return cudaErrorNotSupported;
}
}  // namespace qf
