// hier_nvls.cu -- the intra-machine average of the hierarchical neighbour
// allreduce (P:660 step 1, "intra-machine allreduce"; reading R12) through
// the NVSwitch's in-fabric reduction (NVLS), for machines that span processes.
//
// Every process of a machine writes the sum of its K rows (H-ATC: of x - lr g)
// into its copy of a multicast-backed buffer (unicast address), tells the other
// processes of the machine -- per CTA, the same element ranges on every process --
// and then reads the machine sum of its elements with ONE multimem.ld_reduce per
// 16 bytes through the multicast address: the switch adds the P copies, so the
// partials never travel to every peer.  The machine average lands in a local row;
// the machine-level neighbour averaging and the broadcast back to the K rows are
// the push kernel's hierarchical mode over it (exchange_push.cuh, hier_in = 1).
// The multicast object itself is plumbing: torch symmetric memory allocates it
// (api.py Context.enable_nvls) and hands the two addresses to bf_hier_set_multicast.
#include <cuda_bf16.h>

#include "exchange_common.cuh"

namespace bf {

__device__ __forceinline__ float4 multimem_ld_reduce_add_v4(unsigned long long mc_addr) {
    float4 r;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(mc_addr)
                 : "memory");
    return r;
}

template <typename GT>
__global__ void __launch_bounds__(256) hier_nvls_kernel(const __grid_constant__ NvlsParams p) {
    const Geometry &g = p.geo;
    Pad *pad = pad_of(g, g.me);
    if (aborted(g)) return;
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long *>(&pad->epoch) + 1;
    const int parity = static_cast<int>(e & 1);
    if (!war_wait(g, e)) return;   // the parity half of the multicast buffer is free everywhere
    const long long count = g.count, nvec = (count + 3) / 4;
    const bool vec = g.vec_ok != 0;
    float *mine = p.uc + static_cast<long long>(parity) * p.cap;
    // ---- partial sum of the local rows (H-ATC: of fp32(x - lr g), Eq. 4) ----
    for (long long v = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; v < nvec;
         v += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long e0 = v * 4;
        const int valid = clamp_valid_v<4>(count - e0, 0);
        float s[4] = {0.f, 0.f, 0.f, 0.f};
        for (int r = 0; r < g.k; ++r) {
            float xv[4];
            Vec4<float>::load(p.x + r * count + e0, xv, valid, vec);
            if (p.hmode == 1) {
                float gv[4];
                Vec4<GT>::load(static_cast<const GT *>(p.g) + r * count + e0, gv, valid, vec);
#pragma unroll
                for (int i = 0; i < 4; ++i) xv[i] = fmaf(-p.lr, gv[i], xv[i]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) s[i] += xv[i];
        }
        *reinterpret_cast<float4 *>(mine + e0) = make_float4(s[0], s[1], s[2], s[3]);   // padded: tail lanes 0
    }
    // ---- this CTA's partials, visible system-wide, then flagged to the machine ----
    __syncthreads();
    if (threadIdx.x == 0) {
        fence_acq_rel(true);
        for (int i = 0; i < p.P; ++i) {
            const int q = p.proc0 + i;
            if (q != g.me)
                st_relaxed(at<unsigned long long>(g.peer_base[q], p.nflag_off) +
                               static_cast<long long>(g.me) * kMaxGrid + blockIdx.x,
                           e, true);
        }
    }
    bool ok = true;
    if (threadIdx.x < p.P) {
        const int q = p.proc0 + threadIdx.x;
        if (q != g.me)
            ok = spin_ge(g, at<unsigned long long>(g.peer_base[g.me], p.nflag_off) + static_cast<long long>(q) * kMaxGrid +
                                blockIdx.x,
                         e);
    }
    if (!__syncthreads_and(ok)) return;
    // ---- machine sum of the same elements through the switch, / L ----
    const unsigned long long mbase = p.mc + static_cast<unsigned long long>(parity) * p.cap * 4;
    for (long long v = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; v < nvec;
         v += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long e0 = v * 4;
        const int valid = clamp_valid_v<4>(count - e0, 0);
        const float4 s = multimem_ld_reduce_add_v4(mbase + static_cast<unsigned long long>(e0) * 4);
        const float avg[4] = {s.x * p.invL, s.y * p.invL, s.z * p.invL, s.w * p.invL};
        Vec4<float>::store(p.avg + e0, avg, valid, true);
    }
    last_cta(pad, [&] {
        pad->epoch = e;
        publish_done(g, e);
    });
}

cudaError_t launch_hier_nvls(const NvlsParams &p, int g_kind, cudaStream_t s) {
    const long long nvec = (p.geo.count + 3) / 4;
    long long grid = (nvec + 255) / 256;
    static int maxg[2] = {0, 0};   // co-resident CTAs (the same on every process: same count, same device)
    const void *fn0 = g_kind == 1 ? reinterpret_cast<const void *>(hier_nvls_kernel<__nv_bfloat16>)
                                  : reinterpret_cast<const void *>(hier_nvls_kernel<float>);
    if (maxg[g_kind == 1] == 0) maxg[g_kind == 1] = max_coresident(fn0, 256, 0);
    if (grid > maxg[g_kind == 1]) grid = maxg[g_kind == 1];
    if (grid > kMaxGrid) grid = kMaxGrid;
    if (grid < 1) grid = 1;
    void *args[] = {const_cast<NvlsParams *>(&p)};
    // cooperative: CTA b waits for CTA b of the machine's other processes
    const void *fn = g_kind == 1 ? reinterpret_cast<const void *>(hier_nvls_kernel<__nv_bfloat16>)
                                 : reinterpret_cast<const void *>(hier_nvls_kernel<float>);
    return cudaLaunchCooperativeKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(256), args, 0, s);
}

}  // namespace bf
