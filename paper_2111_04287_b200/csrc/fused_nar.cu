// fused_nar.cu -- instantiations of the local-agent fused exchange kernel for
// neighbor_allreduce (Eq. 5): every dtype combination x K = 1, 2, 4, 8 local agents.
#include "exchange_fused.cuh"

namespace bf {

cudaError_t launch_fused_nar(const ExchParams &p, int x_kind, int grid, cudaStream_t s) {
    if (x_kind == 0) return launch_fused_t<float, float, float, float, 0>(p, grid, s);
    return launch_fused_t<bf16, bf16, bf16, bf16, 0>(p, grid, s);
}

}  // namespace bf
