// fused_ed.cu -- instantiations of the local-agent fused exchange kernel for
// Exact-Diffusion (appendix ed-1..ed-3, MODE 3): fp32 x / psi, fp32 or bf16 g
// and wire, K = 1, 2, 4, 8 local agents.
#include "exchange_fused.cuh"

namespace bf {

cudaError_t launch_fused_ed(const ExchParams &p, int g_kind, int wire_kind, int grid, cudaStream_t s) {
    if (g_kind == 0 && wire_kind == 0) return launch_fused_t<float, float, float, float, 3>(p, grid, s);
    if (g_kind == 0 && wire_kind == 1) return launch_fused_t<float, float, bf16, float, 3>(p, grid, s);
    if (g_kind == 1 && wire_kind == 0) return launch_fused_t<float, bf16, float, float, 3>(p, grid, s);
    return launch_fused_t<float, bf16, bf16, float, 3>(p, grid, s);
}

}  // namespace bf
