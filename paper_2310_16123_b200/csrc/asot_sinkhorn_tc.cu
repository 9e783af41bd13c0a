// asot_sinkhorn_tc.cu -- placeholder until the tcgen05 kernel lands.
#include "asot_internal.cuh"
namespace asot {
bool sinkhorn_tc_supported(int K) { (void)K; return false; }
cudaError_t launch_sinkhorn_tc(int64_t, int64_t, int64_t, const PairSink&, const float*, int,
                               const uint32_t*, const uint32_t*, int, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace asot
