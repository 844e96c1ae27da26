// hier_nvls.cu -- the intra-machine average of the hierarchical neighbour
// allreduce (P:660 step 1, "intra-machine allreduce"; reading R12) through
// the NVSwitch's in-fabric reduction (NVLS), for machines that span processes.
//
// Every process of a machine writes the sum of its K rows (H-ATC: of x - lr g)
// into its copy of a multicast-backed buffer (unicast address) and tells the other
// processes of the machine -- per CTA, the same element ranges on every process.
// Then reduce-scatter + broadcast through the switch: process l of the machine
// reads the machine sum of every P-th vector of the range with one
// multimem.ld_reduce per 16 bytes (the switch adds the P partials) and writes the
// average into every process's copy with one multimem.st -- per process M/P bytes
// out to the reductions and M/P of broadcasts, instead of (P - 1) M partials in
// and out when every process reads every partial.  After a second per-CTA flag
// the machine average sits in the local copy; the machine-level neighbour
// averaging and the broadcast back to the K rows are the push kernel's
// hierarchical mode over it (exchange_push.cuh, hier_in = 1).
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

__device__ __forceinline__ void multimem_st_v4(unsigned long long mc_addr, float4 v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc_addr), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

// Flags between the P processes of the machine, per CTA (every process runs the same
// grid over the same elements): value 2e after the partials, 2e + 1 after the slices.
__device__ __forceinline__ bool nvls_sync(const NvlsParams &p, unsigned long long v) {
    const Geometry &g = p.geo;
    __syncthreads();
    if (threadIdx.x == 0) {
        fence_acq_rel(true);
        for (int i = 0; i < p.P; ++i) {
            const int q = p.proc0 + i;
            if (q != g.me)
                st_relaxed(at<unsigned long long>(g.peer_base[q], p.nflag_off) +
                               static_cast<long long>(g.me) * kMaxGrid + blockIdx.x,
                           v, true);
        }
    }
    bool ok = true;
    if (threadIdx.x < p.P) {
        const int q = p.proc0 + threadIdx.x;
        if (q != g.me)
            ok = spin_ge(g, at<unsigned long long>(g.peer_base[g.me], p.nflag_off) +
                                static_cast<long long>(q) * kMaxGrid + blockIdx.x,
                         v);
    }
    return __syncthreads_and(ok);
}

template <typename GT>
__global__ void __launch_bounds__(256) hier_nvls_kernel(const __grid_constant__ NvlsParams p) {
    const Geometry &g = p.geo;
    Pad *pad = pad_of(g, g.me);
    if (aborted(g)) return;
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long *>(&pad->epoch) + 1;
    const int parity = static_cast<int>(e & 1);
    // WAR: the partial half of this parity (read by the peers' reductions two epochs
    // ago) and the average half (read by the peers' machine exchange ONE epoch ago,
    // the push launch that follows every NVLS launch) are free everywhere
    bool ok = true;
    if (g.nprocs > 1 && e > 1 && threadIdx.x < g.nprocs)
        ok = spin_ge(g, &pad->done_from[threadIdx.x], e - 1);
    if (!__syncthreads_and(ok)) return;
    const long long count = g.count, nvec = (count + 3) / 4;
    const bool vec = g.vec_ok != 0;
    float *mine = p.uc + static_cast<long long>(parity) * p.cap;                         // partials
    const unsigned long long mpart = p.mc + static_cast<unsigned long long>(parity) * p.cap * 4;
    const unsigned long long mavg = p.mc + static_cast<unsigned long long>(2 + parity) * p.cap * 4;   // averages
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
    if (!nvls_sync(p, 2 * e)) return;
    // ---- reduce-scatter through the switch: this process reduces every P-th vector of the
    // CTA's range (multimem.ld_reduce adds the P partials), / L, and broadcasts it into
    // every process's average half (multimem.st) ----
    const int li = g.me - p.proc0;
    long long it = 0;
    for (long long v = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; v < nvec;
         v += static_cast<long long>(gridDim.x) * blockDim.x, ++it) {
        if (static_cast<int>(it % p.P) != li) continue;
        const unsigned long long off = static_cast<unsigned long long>(v) * 16;
        const float4 s = multimem_ld_reduce_add_v4(mpart + off);
        multimem_st_v4(mavg + off, make_float4(s.x * p.invL, s.y * p.invL, s.z * p.invL, s.w * p.invL));
    }
    if (!nvls_sync(p, 2 * e + 1)) return;
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
