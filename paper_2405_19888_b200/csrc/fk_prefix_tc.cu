// tcgen05 shared-prefix kernel (placeholder until the TMEM path lands).
#include "fk_common.cuh"
namespace fk {
cudaError_t launch_prefix_tc(const ArenaDev&, const PlanDev&, int, const void*, void*, float*, float,
                             const CUtensorMap*, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace fk
