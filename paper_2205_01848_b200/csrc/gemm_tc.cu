// gemm_tc.cu -- tcgen05 grouped GEMMs (placeholder until the tcgen05 kernels land).
#include "gemm_tc.h"

namespace moe {
void tc_plan_free(TcPlan* p) { (void)p; }
moe_status_t tc_ffn_forward(TcPlan*, void*, const void*, const void*, const void*, const void*,
                            void*, void*, int64_t, int, int, int, const int32_t*, const int32_t*,
                            int, const CapTable&, int, cudaStream_t, int64_t*) {
  return MOE_ERR_CONFIG;
}
moe_status_t tc_ffn_backward(TcPlan*, void*, void*, void*, void*, const void*, const void*,
                             void*, void*, void*, void*, int, int64_t, int, int, int,
                             const int32_t*, const int32_t*, int, const CapTable&, int,
                             cudaStream_t, int64_t*) {
  return MOE_ERR_CONFIG;
}
}  // namespace moe
