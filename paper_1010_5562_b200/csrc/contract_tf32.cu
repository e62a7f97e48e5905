// contract_tf32.cu — a3 (split-TF32 tcgen05 path).  Placeholder until the tensor-core
// kernel lands: reports FCFS_E_UNSUPPORTED rather than silently computing elsewhere.
#include "common.cuh"

namespace fcfs {

fcfs_status tf32_supported(const GemmPlan &, int32_t) {
    set_error("FCFS_TF32X3 is not built yet");
    return FCFS_E_UNSUPPORTED;
}

fcfs_status launch_gemm_tf32(const CornerSrc &, const GemmPlan &, int32_t, double *, cudaStream_t) {
    set_error("FCFS_TF32X3 is not built yet");
    return FCFS_E_UNSUPPORTED;
}

}  // namespace fcfs
