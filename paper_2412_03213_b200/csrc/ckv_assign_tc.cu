// ckv_assign_tc.cu — K1: tensor-core (tcgen05) assignment filter.  (stub)
#include "ckv_internal.cuh"
namespace ckvb {
bool assign_tc_supported(uint32_t, uint32_t) { return false; }
size_t assign_tc_scratch_bytes(uint32_t, uint32_t, uint32_t) { return 0; }
int assign_tc(cudaStream_t, const uint16_t*, uint64_t, uint32_t, uint32_t, uint32_t, uint32_t,
              const uint16_t*, const float*, int32_t*, uint32_t, const int32_t*, void*, size_t,
              uint64_t*) {
  set_error("assign_tc: not built");
  return CKV_EINVAL;
}
}  // namespace ckvb
