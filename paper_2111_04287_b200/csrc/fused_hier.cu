// fused_hier.cu -- instantiations of the cross-GPU push kernel for the
// hierarchical modes (exchange_push.cuh MODE 6 / 7 / 8: hierarchical
// neighbor_allreduce, H-ATC, H-AWC, caption P:869) when every machine
// lies inside one process: K = machines per process = 1, 2 or 4.
#include "exchange_fused.cuh"

namespace bf {

template <typename XT, typename GT, int MODE>
static cudaError_t hier_push_t(const ExchParams &p, cudaStream_t s) {
    switch (p.geo.k) {
        case 1: return launch_push_k<XT, GT, XT, XT, MODE, 1>(p, p.max_ctas, s);
        case 2: return launch_push_k<XT, GT, XT, XT, MODE, 2>(p, p.max_ctas, s);
        case 4: return launch_push_k<XT, GT, XT, XT, MODE, 4>(p, p.max_ctas, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_hier_push(const ExchParams &p, int x_kind, int g_kind, cudaStream_t s) {
    if (p.hier_mode == 6) return x_kind == 0 ? hier_push_t<float, float, 6>(p, s) : hier_push_t<bf16, bf16, 6>(p, s);
    if (x_kind != 0) return cudaErrorInvalidValue;   // H-ATC / H-AWC: fp32 master x
    if (p.hier_mode == 7) return g_kind == 0 ? hier_push_t<float, float, 7>(p, s) : hier_push_t<float, bf16, 7>(p, s);
    return g_kind == 0 ? hier_push_t<float, float, 8>(p, s) : hier_push_t<float, bf16, 8>(p, s);
}

}  // namespace bf
