// fused_gt.cu -- instantiations of the fused exchange kernels for push-sum
// gradient tracking (appendix): MODE 4 (y-step,
// y <- W(y + g - g_prev)) and MODE 5 (u/v-step, u <- W(u - lr y), v <- W v,
// x = u / v), fp32 tensors, fp32 or bf16 wire, K = 1, 2, 4, 8 local agents.
#include "exchange_fused.cuh"

namespace bf {

cudaError_t launch_fused_gt(const ExchParams &p, int wire_kind, int grid, cudaStream_t s) {
    if (p.gt == 4)
        return wire_kind == 0 ? launch_fused_t<float, float, float, float, 4>(p, grid, s)
                              : launch_fused_t<float, float, bf16, float, 4>(p, grid, s);
    return wire_kind == 0 ? launch_fused_t<float, float, float, float, 5>(p, grid, s)
                          : launch_fused_t<float, float, bf16, float, 5>(p, grid, s);
}

}  // namespace bf
