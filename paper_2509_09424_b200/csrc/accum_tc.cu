// accum_tc.cu -- row a3 on the 5th-generation tensor cores (byte-sliced INT8 tcgen05.mma).  Placeholder
// until the kernel lands: tc_supported() reports false so the CUDA-core path (accum.cu) runs.
#include "ensi_internal.h"

namespace ensi {

bool tc_supported(const ensi_ctx*, uint32_t) { return false; }

int accum_ternary_tc(ensi_ctx* ctx, const uint64_t*, uint32_t, ensi_weights*, uint64_t*, uint32_t, cudaStream_t, uint64_t,
                     uint32_t) {
    return set_err(ctx, ENSI_EINVAL, "tensor-core accumulate not built");
}

}  // namespace ensi
