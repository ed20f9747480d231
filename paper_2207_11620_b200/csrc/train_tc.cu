// tcgen05 fused training / inference tile pipeline (sm_100a).  Placeholder
// until the tensor-core path lands: reports "unsupported" so callers fall
// back to mode 0 explicitly (no silent substitution).
#include "common.cuh"

namespace nvol {

int train_tc_launch(const float *, const float *, int64_t, int64_t, const float *, float *, const GridTables &, int,
                    int, int, int, double *, void *, int64_t, cudaStream_t) {
    set_error("tcgen05 training path not built");
    return NVOL_EINVAL;
}
int64_t train_tc_workspace(int64_t, int, int, int, int) { return 0; }

int nvol_decode_tc(const float *, const GridTables &, const float *, const int32_t *, int32_t, int32_t, int64_t,
                   int64_t, int64_t, int64_t, int64_t, double, double, float *, cudaStream_t) {
    set_error("tcgen05 decode path not built");
    return NVOL_EINVAL;
}

}  // namespace nvol

extern "C" int nvol_has_tcgen05(int) { return 0; }
