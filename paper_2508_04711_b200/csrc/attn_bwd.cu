// Fused jagged HSTU attention backward (placeholder until the tcgen05 kernel lands).
#include "abi_internal.h"
#include "attn_common.cuh"

namespace jh {
template <int D>
int launch_bwd(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const AttnParams&,
               const jh_attn_args&, int, cudaStream_t) {
  set_error(JH_ERR_UNSUPPORTED, "backward not built");
  return -1;
}
template int launch_bwd<64>(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                            const AttnParams&, const jh_attn_args&, int, cudaStream_t);
template int launch_bwd<128>(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                             const AttnParams&, const jh_attn_args&, int, cudaStream_t);
}  // namespace jh
