// exchange_common.cuh -- device-side protocol pieces shared by the exchange
// kernels (exchange.cu: chunked kernel; exchange_fused.cuh: local-agent fused
// kernel): WAR protection of the double-buffered slots, source resolution for
// static / scheduled / per-call topologies, per-epoch descriptors.
#pragma once

#include <cuda_bf16.h>

#include "dev_common.cuh"

namespace bf {

using bf16 = __nv_bfloat16;


__device__ __forceinline__ unsigned long long *ready_ptr(const Geometry &g, unsigned long long off,
                                                         int stride, int agent, int t) {
    return at<unsigned long long>(g.peer_base[agent / g.k], off) +
           static_cast<long long>(agent % g.k) * stride + t;
}

// Wait until every process finished reading epoch e-2 (so parity e&1 is free).
__device__ __forceinline__ bool war_wait(const Geometry &g, unsigned long long e) {
    bool ok = true;
    if (g.nprocs > 1 && e > 2 && threadIdx.x < g.nprocs)
        ok = spin_ge(g, &pad_of(g, g.me)->done_from[threadIdx.x], e - 2);
    return __syncthreads_and(ok);
}

// Broadcast "this process finished reading epoch e" to every process.
__device__ __forceinline__ void publish_done(const Geometry &g, unsigned long long e) {
    // only other processes wait on done_from (war_wait); one process needs no
    // system-scope release (an idle fence.acq_rel.sys alone costs ~3.5 us)
    if (g.nprocs == 1) return;
    // one system-scope fence orders every read of this epoch before all the stores
    // (a st.release.sys per process would fence once per process)
    fence_acq_rel(true);
    for (int q = 0; q < g.nprocs; ++q) st_relaxed(&pad_of(g, q)->done_from[g.me], e, true);
}

// --------------------------------------------------------------------------
// Source resolution for one call: fills the shared table of every local agent.
//   static   : coefficients from the host's W row (Eq. 5)
//   schedule : one-peer exp-2 (R5) or inner-outer exp-2 (R27)
//              from the device round counter
//   dynamic  : declared r (Eq. 11) times the senders' s (Eq. 10) read from their
//              descriptors; push-only receivers discover their sources there;
//              topology check on mismatches.
struct SharedTab {
    float self_w[kMaxK];
    float coef[kMaxK][kMaxN];
    unsigned char src[kMaxK][kMaxN];
    int nsrc[kMaxK];
};

static __device__ bool resolve_sources(const ExchParams &p, unsigned long long e, SharedTab &st) {
    const Geometry &g = p.geo;
    const int k = g.k;
    const int parity = static_cast<int>(e & 1);
    bool ok = true;
    if (p.wmode == kWStatic) {
        for (int a = threadIdx.x; a < k; a += blockDim.x) {
            st.self_w[a] = p.tab.self_w[a];
            st.nsrc[a] = p.tab.nsrc[a];
            for (int q = 0; q < p.tab.nsrc[a]; ++q) {
                st.src[a][q] = p.tab.src[a][q];
                st.coef[a][q] = p.tab.coef[a][q];
            }
        }
    } else if (p.wmode == kWSchedule) {
        const unsigned long long round = *reinterpret_cast<volatile unsigned long long *>(
            &pad_of(g, g.me)->round);
        for (int a = threadIdx.x; a < k; a += blockDim.x) {
            int src, dst;
            sched_peers(p.sched_kind, g.n, p.sched_L, round, g.me * k + a, src, dst);
            st.self_w[a] = src < 0 ? 1.f : 0.5f;
            st.nsrc[a] = src < 0 ? 0 : 1;
            st.src[a][0] = static_cast<unsigned char>(src < 0 ? 0 : src);
            st.coef[a][0] = 0.5f;
        }
    } else {
        // one warp per local agent; lanes scan candidate senders j
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int nwarps = blockDim.x >> 5;
        for (int a = warp; a < k; a += nwarps) {
            const int gid = g.me * k + a;
            const bool has_src = p.dyn.has_src[a];
            int total = 0;
            for (int j0 = 0; j0 < g.n; j0 += 32) {
                const int j = j0 + lane;
                bool include = false;
                float c = 0.f;
                if (j < g.n && j != gid) {
                    int qdecl = -1;
                    if (has_src)
                        for (int q = 0; q < p.tab.nsrc[a]; ++q)
                            if (p.tab.src[a][q] == j) qdecl = q;
                    const bool need = !has_src || qdecl >= 0 || p.check;
                    if (need) {
                        const Desc *d = &pad_of(g, j / k)->desc[j % k][parity];
                        if (!spin_ge(g, &d->epoch, e)) {
                            ok = false;
                        } else {
                            const unsigned long long mask =
                                *reinterpret_cast<const volatile unsigned long long *>(&d->dstmask);
                            const unsigned long long hd =
                                *reinterpret_cast<const volatile unsigned long long *>(&d->has_dst);
                            const bool to_me = (mask >> gid) & 1ull;
                            const float s = to_me ? *reinterpret_cast<const volatile float *>(&d->s[gid]) : 1.f;
                            if (has_src) {
                                if (qdecl >= 0) {
                                    include = true;
                                    c = p.tab.coef[a][qdecl] * s;            // r_ij * s_ij (R1)
                                    if (p.check && hd && !to_me) ok = false;  // sender never sends to me
                                } else if (to_me && p.check) {
                                    ok = false;                               // unlisted pusher
                                }
                            } else if (to_me) {
                                include = true;                               // push-only: r = 1
                                c = s;
                            }
                        }
                    }
                }
                const unsigned int bal = __ballot_sync(0xffffffffu, include);
                if (include) {
                    const int pos = total + __popc(bal & ((1u << lane) - 1u));
                    st.src[a][pos] = static_cast<unsigned char>(j);
                    st.coef[a][pos] = c;
                }
                total += __popc(bal);
            }
            if (lane == 0) {
                st.nsrc[a] = total;
                st.self_w[a] = p.tab.self_w[a];
            }
        }
        if (!__all_sync(0xffffffffu, ok) && lane == 0) {
            const unsigned int code =
                *reinterpret_cast<volatile unsigned int *>(&pad_of(g, g.me)->abort);
            if (!code) abort_all(g, BF_ERR_TOPOLOGY);
        }
    }
    return __syncthreads_and(ok);
}

// Block 0 writes the descriptors of the local agents for this epoch.
static __device__ void write_descriptors(const ExchParams &p, unsigned long long e) {
    const Geometry &g = p.geo;
    const int parity = static_cast<int>(e & 1);
    if (blockIdx.x != 0) return;
    for (int a = threadIdx.x; a < g.k; a += blockDim.x) {
        Desc *d = &pad_of(g, g.me)->desc[a][parity];
        unsigned long long mask = 0;
        for (int q = 0; q < p.dyn.ndst[a]; ++q) {
            const int j = p.dyn.dst[a][q];
            mask |= 1ull << j;
            d->s[j] = p.dyn.s[a][q];
        }
        d->dstmask = mask;
        d->has_dst = p.dyn.has_dst[a];
        st_release_sys(&d->epoch, e);
    }
}

// Push-sum gradient tracking, u/v-step (MODE 5): the scalar weights v_j of the
// sources, combined with the step's coefficients -- v_a <- w_aa v_a + sum_j w_aj v_j
// (appendix line 1003 with v^0 = 1, so every entry of the paper's vector v is
// the same scalar).  Block 0 publishes the local agents' v in the pad for this
// epoch; every CTA reads same-process weights from p.gt_v and other processes'
// from their pads (bounded spin on the epoch tag).  Returns false on a fault.
static __device__ bool gt_weights(const ExchParams &p, unsigned long long e, const SharedTab &st, float *vnew) {
    const Geometry &g = p.geo;
    const int k = g.k, parity = static_cast<int>(e & 1);
    if (blockIdx.x == 0 && threadIdx.x < k) {
        Pad *pad = pad_of(g, g.me);
        pad->gtv[threadIdx.x][parity] = p.gt_v[threadIdx.x];
        st_release(&pad->gtv_tag[threadIdx.x][parity], e, g.nprocs > 1);
    }
    bool ok = true;
    if (threadIdx.x < k) {
        const int a = threadIdx.x;
        float acc = st.self_w[a] * p.gt_v[a];
        for (int q = 0; q < st.nsrc[a]; ++q) {
            const int j = st.src[a][q];
            float vj;
            if (j / k == g.me) {
                vj = p.gt_v[j % k];
            } else {
                Pad *pj = pad_of(g, j / k);
                if (!spin_ge(g, &pj->gtv_tag[j % k][parity], e)) {
                    ok = false;
                    break;
                }
                vj = *reinterpret_cast<volatile float *>(&pj->gtv[j % k][parity]);
            }
            acc = fmaf(st.coef[a][q], vj, acc);
        }
        vnew[a] = acc;
    }
    return __syncthreads_and(ok);
}

// Walks the items w = first, first + stride, ... as (tile t, local agent a)
// with w = t*k + a, without integer division in the loop.
struct ItemIt {
    int t, a, dt, da, k;
    __device__ ItemIt(int first, int stride, int k_) : t(first / k_), a(first % k_), dt(stride / k_),
                                                          da(stride % k_), k(k_) {}
    __device__ __forceinline__ void next() {
        t += dt;
        a += da;
        if (a >= k) {
            a -= k;
            ++t;
        }
    }
};

}  // namespace bf
