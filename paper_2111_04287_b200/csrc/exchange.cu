// exchange.cu -- the partial-averaging hot path on sm_100a.
//
// exchange_kernel: ONE persistent, cooperative launch per call that fuses
//   Eq. 4 local update (ATC)      x_half = x - lr*g          (registers)
//   publish + signal                      wire(x_half) -> own IPC slot, release flag
//   neighbour exchange (Eq. 5 / Eq. 9)    acquire peers' flags, 128-bit loads over
//                                         NVLink (other GPU) or L2 (same GPU)
//   weighted combine + store              y = w_ii x_half + sum_j w_ij wire_j (fp32 FMA)
// tile by tile (kTile elements per flag), so HBM traffic, NVLink traffic and
// the wait for the slowest neighbour overlap across the CTAs of the grid.
//
// Deadlock freedom: all CTAs are co-resident (cooperative launch), every CTA
// walks its items in increasing tile order and publishes tile t before it
// waits for anybody's tile t, and grid >= local agents; every wait is bounded
// by the context timeout.  WAR safety: slots are double-buffered by epoch
// parity and a writer overwrites parity (e&1) only after every process has
// reported (done_from) that it finished reading epoch e-2.
#include <cooperative_groups.h>
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
    for (int q = 0; q < g.nprocs; ++q) st_release_sys(&pad_of(g, q)->done_from[g.me], e);
}

// --------------------------------------------------------------------------
// Source resolution for one call: fills the shared table of every local agent.
//   static   : coefficients from the host's W row (Eq. 5)
//   schedule : one-peer exp-2 from the device round counter (R5)
//   dynamic  : declared r (Eq. 11) times the senders' s (Eq. 10) read from their
//              descriptors; push-only receivers discover their sources there;
//              topology check on mismatches.
struct SharedTab {
    float self_w[kMaxK];
    float coef[kMaxK][kMaxN];
    unsigned char src[kMaxK][kMaxN];
    int nsrc[kMaxK];
};

__device__ bool resolve_sources(const ExchParams &p, unsigned long long e, SharedTab &st) {
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
        int tau = 0;
        while ((1 << tau) < g.n) ++tau;
        for (int a = threadIdx.x; a < k; a += blockDim.x) {
            const int gid = g.me * k + a;
            if (tau == 0) {
                st.self_w[a] = 1.f;
                st.nsrc[a] = 0;
            } else {
                const int off = 1 << static_cast<int>(round % tau);
                st.self_w[a] = 0.5f;
                st.nsrc[a] = 1;
                st.src[a][0] = static_cast<unsigned char>(((gid - off) % g.n + g.n) % g.n);
                st.coef[a][0] = 0.5f;
            }
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
__device__ void write_descriptors(const ExchParams &p, unsigned long long e) {
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

#ifndef BF_LAG
#define BF_LAG 2
#endif
#ifndef BF_PSTAGES
#define BF_PSTAGES 2
#endif
#ifndef BF_NPEER
#define BF_NPEER 2
#endif
constexpr int kConsumerWarps = kThreads / 32;          // 8 consumer warps
constexpr int kExchThreads = kThreads + 96;            // + 2 producer warps + 1 signal warp

// Per-CTA shared-memory pipeline.
//   x/g ring  : SX = D + 2 stages (item i is combined while item i+D is published)
//   peer ring : SP stages of NP in-neighbour tiles
template <typename XT, typename GT, typename WT, bool HAS_G>
struct Pipe {
    static constexpr int D = BF_LAG, SX = BF_LAG + 2, SP = BF_PSTAGES, NP = BF_NPEER;
    static constexpr unsigned XB = kTile * sizeof(XT);
    static constexpr unsigned GB = HAS_G ? kTile * sizeof(GT) : 0;
    static constexpr unsigned PB = kTile * sizeof(WT);
    static constexpr unsigned XG = XB + GB;
    static constexpr unsigned BYTES = SX * XG + SP * NP * PB;
};

// exchange_kernel: warp-specialised persistent pipeline, one CTA per SM.
//   producer warp A : TMA bulk loads of this CTA's x / g tiles (x/g ring)
//   producer warp B : acquire the in-neighbours' ready flags of a tile, then
//                     LDGSTS (cp.async) of their published tiles -- over NVLink
//                     for agents on other GPUs, from L2 on this GPU (peer ring)
//   consumer warps  : iteration c publishes item c+D (adapt x - lr*g, store the
//                     wire copy in this agent's IPC slot, release its flag) and
//                     then combines item c (Eq. 5 / Eq. 9, fp32) and stores it.
// Publishing D items ahead means a neighbour's tile is normally published long
// before it is needed, so flag waits and peer-load latency leave the critical
// path.  Deadlock freedom: items are visited in increasing tile order; x/g
// loads never wait on other agents; a tile is published before anybody's wait
// for the tile of a later item; all CTAs are co-resident (cooperative launch).
// A fault never exits early: waits fail fast, garbage is computed and the fault
// is latched, so no TMA or cp.async is left in flight.
template <typename XT, typename GT, typename WT, typename YT, bool HAS_G>
__global__ void __launch_bounds__(kExchThreads, 1) exchange_kernel(const __grid_constant__ ExchParams p) {
    using P = Pipe<XT, GT, WT, HAS_G>;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ SharedTab st;
    __shared__ __align__(8) unsigned long long full_xg[P::SX], empty_xg[P::SX], published[P::SX];
    __shared__ __align__(8) unsigned long long full_pr[P::SP], empty_pr[P::SP];
    __shared__ int s_fail;
    const Geometry &g = p.geo;
    Pad *pad = pad_of(g, g.me);
    if (aborted(g)) return;
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long *>(&pad->epoch) + 1;
    const int parity = static_cast<int>(e & 1);
    const bool sys = g.nprocs > 1;   // flags of agents on other GPUs need system scope

    if (threadIdx.x == 0) {
        s_fail = 0;
        for (int i = 0; i < P::SX; ++i) {
            mbar_init(&full_xg[i], 1);
            mbar_init(&empty_xg[i], kConsumerWarps + 1);   // consumers + signal warp
            mbar_init(&published[i], kConsumerWarps);
        }
        for (int i = 0; i < P::SP; ++i) {
            mbar_init(&full_pr[i], 32);
            mbar_init(&empty_pr[i], kConsumerWarps);
        }
        fence_mbar_init();
    }
    bool ok = war_wait(g, e);
    if (p.wmode == kWDynamic) write_descriptors(p, e);
    ok = resolve_sources(p, e, st) && ok;
    if (!ok && threadIdx.x == 0) s_fail = 1;
    __syncthreads();

    const bool vec = g.vec_ok != 0;
    const long long count = g.count;
    const int k = g.k;
    const long long items = static_cast<long long>(k) * g.T;
    const int nmine = blockIdx.x < items ? static_cast<int>((items - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0;
    auto item = [&](int c) { return blockIdx.x + static_cast<long long>(c) * gridDim.x; };
    auto staged = [&](long long w) {   // TMA needs 16B-aligned rows and a full tile
        return vec && (count - static_cast<long long>(w / k) * kTile) >= kTile;
    };
    auto xs = [&](int s) { return smem + s * P::XG; };
    auto gs = [&](int s) { return smem + s * P::XG + P::XB; };
    auto ps = [&](int s, int q) { return smem + P::SX * P::XG + (s * P::NP + q) * P::PB; };
    auto slot_of = [&](int agent) {
        return at<WT>(g.peer_base[agent / k],
                      p.slot_off + (agent % k) * p.slot_agent_stride + parity * p.slot_parity_stride);
    };
    auto failed = [&]() { return *reinterpret_cast<volatile int *>(&s_fail) != 0; };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == kConsumerWarps) {
        // ===================== producer A: x / g tiles (TMA) =====================
        for (int c = 0; c < nmine; ++c) {
            const int s = c % P::SX;
            if (c >= P::SX) mbar_wait(&empty_xg[s], static_cast<unsigned>(c / P::SX - 1) & 1u);
            if (lane == 0) {
                const long long w = item(c);
                if (staged(w)) {
                    const long long off = static_cast<long long>(w % k) * count + (w / k) * kTile;
                    fence_proxy_async();
                    mbar_expect_tx(&full_xg[s], P::XG);
                    tma_load_1d(xs(s), static_cast<const XT *>(p.x) + off, P::XB, &full_xg[s]);
                    if constexpr (HAS_G) tma_load_1d(gs(s), static_cast<const GT *>(p.g) + off, P::GB, &full_xg[s]);
                } else {
                    mbar_arrive(&full_xg[s]);
                }
            }
            __syncwarp();
        }
    } else if (warp == kConsumerWarps + 1) {
        // ============ producer B: in-neighbour tiles (flag-gated cp.async) ============
        for (int c = 0; c < nmine; ++c) {
            const int s = c % P::SP;
            if (c >= P::SP) mbar_wait(&empty_pr[s], static_cast<unsigned>(c / P::SP - 1) & 1u);
            const long long w = item(c);
            const int t = static_cast<int>(w / k), a = static_cast<int>(w % k);
            const long long base = static_cast<long long>(t) * kTile;
            const int np = min(st.nsrc[a], P::NP);
            bool good = true;
            if (lane < np && !failed())
                good = spin_ge(g, ready_ptr(g, p.ready_off, p.ready_stride, st.src[a][lane], t), e, sys);
            if (!__all_sync(0xffffffffu, good) && lane == 0) s_fail = 1;
            __syncwarp();
            if (!failed()) {
                const long long rem_bytes = (count - base) * static_cast<long long>(sizeof(WT));
                for (int q = 0; q < np; ++q) {
                    const unsigned char *src = reinterpret_cast<const unsigned char *>(slot_of(st.src[a][q]) + base);
                    unsigned char *dst = ps(s, q);
#pragma unroll 4
                    for (int ch = lane; ch < static_cast<int>(P::PB / 16); ch += 32) {
                        const long long left = rem_bytes - 16ll * ch;
                        const unsigned nb = left >= 16 ? 16u : (left <= 0 ? 0u : static_cast<unsigned>(left));
                        cp_async16(dst + 16 * ch, nb ? src + 16 * ch : src, nb);
                    }
                }
            }
            cp_async_mbar_arrive_noinc(&full_pr[s]);
        }
    } else if (warp == kConsumerWarps + 2) {
        // ======== signal warp: release the ready flag of every published tile ========
        // (the release fence runs here, off the consumers' critical path)
        for (int c = 0; c < nmine; ++c) {
            const int s = c % P::SX;
            mbar_wait(&published[s], static_cast<unsigned>(c / P::SX) & 1u);
            if (lane == 0) {
                const long long w = item(c);
                st_release(ready_ptr(g, p.ready_off, p.ready_stride, g.me * k + static_cast<int>(w % k),
                                     static_cast<int>(w / k)),
                           e, sys);
                mbar_arrive(&empty_xg[s]);
            }
            __syncwarp();
        }
    } else {
        // =============================== consumers ===============================
        // x_half of item c, from the staged tiles or straight from global memory
        auto adapt = [&](int c, float (&xh)[kVecPerThread][4]) {
            const long long w = item(c);
            const int sx = c % P::SX;
            const int a = static_cast<int>(w % k);
            const long long base = (w / k) * kTile, rem = count - base;
            if (staged(w)) {
                const XT *xsm = reinterpret_cast<const XT *>(xs(sx));
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j) Vec4<XT>::load(xsm + tile_elem(j), xh[j], 4, true);
                if constexpr (HAS_G) {
                    const GT *gsm = reinterpret_cast<const GT *>(gs(sx));
#pragma unroll
                    for (int j = 0; j < kVecPerThread; ++j) {
                        float gv[4];
                        Vec4<GT>::load(gsm + tile_elem(j), gv, 4, true);
#pragma unroll
                        for (int i = 0; i < 4; ++i) xh[j][i] = fmaf(-p.lr, gv[i], xh[j][i]);
                    }
                }
            } else {
                const XT *xr = static_cast<const XT *>(p.x) + static_cast<long long>(a) * count + base;
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j)
                    Vec4<XT>::load(xr + tile_elem(j), xh[j], clamp_valid(rem, tile_elem(j)), vec);
                if constexpr (HAS_G) {
                    const GT *gr = static_cast<const GT *>(p.g) + static_cast<long long>(a) * count + base;
#pragma unroll
                    for (int j = 0; j < kVecPerThread; ++j) {
                        float gv[4];
                        Vec4<GT>::load(gr + tile_elem(j), gv, clamp_valid(rem, tile_elem(j)), vec);
#pragma unroll
                        for (int i = 0; i < 4; ++i) xh[j][i] = fmaf(-p.lr, gv[i], xh[j][i]);
                    }
                }
            }
        };
        for (int c = -P::D; c < nmine; ++c) {
            // ---- publish item c + D: Eq. 4 local update, wire copy, release flag ----
            const int cp = c + P::D;
            if (cp < nmine) {
                const long long w = item(cp);
                const int t = static_cast<int>(w / k), a = static_cast<int>(w % k);
                const long long base = static_cast<long long>(t) * kTile, rem = count - base;
                mbar_wait(&full_xg[cp % P::SX], static_cast<unsigned>(cp / P::SX) & 1u);
                float xh[kVecPerThread][4];
                adapt(cp, xh);
                WT *mine = slot_of(g.me * k + a) + base;
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j)
                    Vec4<WT>::store(mine + tile_elem(j), xh[j], clamp_valid(rem, tile_elem(j)), true);
                __syncwarp();
                if (lane == 0) mbar_arrive(&published[cp % P::SX]);   // the signal warp releases the flag
                (void)t;
            }
            if (c < 0) continue;
            // ---- combine item c: Eq. 5 / Eq. 9 in fp32 ----
            const long long w = item(c);
            const int t = static_cast<int>(w / k), a = static_cast<int>(w % k);
            const long long base = static_cast<long long>(t) * kTile, rem = count - base;
            float acc[kVecPerThread][4];
            adapt(c, acc);   // x_half again (self term uses the fp32 x_half, R18)
            const float cs = st.self_w[a];
#pragma unroll
            for (int j = 0; j < kVecPerThread; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[j][i] *= cs;
            const int ns = st.nsrc[a];
            const int np = min(ns, P::NP);
            const int sp = c % P::SP;
            mbar_wait(&full_pr[sp], static_cast<unsigned>(c / P::SP) & 1u);
            for (int q = 0; q < np; ++q) {
                const WT *psm = reinterpret_cast<const WT *>(ps(sp, q));
                const float cq = st.coef[a][q];
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j) {
                    float v[4];
                    Vec4<WT>::load(psm + tile_elem(j), v, 4, true);
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[j][i] = fmaf(cq, v[i], acc[j][i]);
                }
            }
            if (ns > np) {   // more in-neighbours than staged tiles: read the rest directly
                if (threadIdx.x < ns - np && !failed()) {
                    if (!spin_ge(g, ready_ptr(g, p.ready_off, p.ready_stride, st.src[a][np + threadIdx.x], t), e,
                                 sys))
                        s_fail = 1;
                }
                named_bar_sync(1, kThreads);
                for (int q = np; q < ns; ++q) {
                    const WT *sp2 = slot_of(st.src[a][q]) + base;
                    const float cq = st.coef[a][q];
#pragma unroll
                    for (int j = 0; j < kVecPerThread; ++j) {
                        float v[4];
                        Vec4<WT>::load_cg(sp2 + tile_elem(j), v, clamp_valid(rem, tile_elem(j)), true);
#pragma unroll
                        for (int i = 0; i < 4; ++i) acc[j][i] = fmaf(cq, v[i], acc[j][i]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&empty_xg[c % P::SX]);
                mbar_arrive(&empty_pr[sp]);
            }
            YT *yr = static_cast<YT *>(p.y) + static_cast<long long>(a) * count + base;
#pragma unroll
            for (int j = 0; j < kVecPerThread; ++j)
                Vec4<YT>::store(yr + tile_elem(j), acc[j], clamp_valid(rem, tile_elem(j)), vec);
            if (p.shadow) {
                bf16 *sr = static_cast<bf16 *>(p.shadow) + static_cast<long long>(a) * count + base;
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j)
                    Vec4<bf16>::store(sr + tile_elem(j), acc[j], clamp_valid(rem, tile_elem(j)), vec);
            }
        }
    }

    __syncthreads();
    if (s_fail) return;   // nothing is in flight any more; the fault is latched
    last_cta(pad, [&] {
        pad->epoch = e;
        if (p.wmode == kWSchedule) pad->round = pad->round + 1;
        publish_done(g, e);
    });
}

// --------------------------------------------------------------------------
// Hierarchical neighbour allreduce: leader-free, sliced.
//   A: publish x tile t -> slot, flag
//   B: agent (m,l) averages slice l over its machine's L agents (1/L, R12)
//   C: agent (m,l) combines slice l with the machine neighbours' slice l (W_M)
//   D: every agent gathers all slices of its machine's result
// Every CTA finishes a stage before starting the next, and a stage only waits
// on the previous stage, so co-resident CTAs cannot deadlock.
template <typename XT>
__global__ void __launch_bounds__(kThreads, 2) hier_kernel(const __grid_constant__ HierParams p) {
    const Geometry &g = p.geo;
    Pad *pad = pad_of(g, g.me);
    if (aborted(g)) return;
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long *>(&pad->epoch) + 1;
    const int parity = static_cast<int>(e & 1);
    if (!war_wait(g, e)) return;
    __shared__ int s_fail;
    if (threadIdx.x == 0) s_fail = 0;
    __syncthreads();

    const bool vec = g.vec_ok != 0;
    const long long count = g.count;
    const int k = g.k, L = p.L, TS = p.TS;
    auto slotA = [&](int agent) {
        return at<const XT>(g.peer_base[agent / k], p.slot_off + (agent % k) * p.slot_agent_stride +
                                                          parity * p.slot_parity_stride);
    };
    auto bufB = [&](int agent) {
        return at<float>(g.peer_base[agent / k], p.b_off + (agent % k) * p.bc_agent_stride +
                                                      parity * p.bc_parity_stride);
    };
    auto bufC = [&](int agent) {
        return at<float>(g.peer_base[agent / k], p.c_off + (agent % k) * p.bc_agent_stride +
                                                      parity * p.bc_parity_stride);
    };
    auto wait_all = [&](const unsigned long long *flag) {
        if (!spin_ge(g, flag, e)) s_fail = 1;
    };

    // ---- stage A ----
    const long long itemsA = static_cast<long long>(k) * g.T;
    for (long long w = blockIdx.x; w < itemsA; w += gridDim.x) {
        const int t = static_cast<int>(w / k), a = static_cast<int>(w % k);
        const long long base = static_cast<long long>(t) * kTile, rem = count - base;
        const XT *xr = static_cast<const XT *>(p.x) + static_cast<long long>(a) * count + base;
        XT *mine = const_cast<XT *>(slotA(g.me * k + a)) + base;
#pragma unroll
        for (int j = 0; j < kVecPerThread; ++j) {
            float v[4];
            const int vl = clamp_valid(rem, tile_elem(j));
            Vec4<XT>::load(xr + tile_elem(j), v, vl, vec);
            Vec4<XT>::store(mine + tile_elem(j), v, vl, vec);
        }
        __syncthreads();
        if (threadIdx.x == 0) st_release_sys(ready_ptr(g, p.ready_off, p.ready_stride, g.me * k + a, t), e);
    }

    // ---- stage B: slice average over the machine ----
    const long long itemsS = static_cast<long long>(k) * TS;
    for (long long w = blockIdx.x; w < itemsS; w += gridDim.x) {
        const int tt = static_cast<int>(w / k), a = static_cast<int>(w % k);
        const int gid = g.me * k + a, m = gid / L, l = gid % L;
        const int t = l * TS + tt;
        if (t >= g.T) continue;
        if (threadIdx.x < L) wait_all(ready_ptr(g, p.ready_off, p.ready_stride, m * L + threadIdx.x, t));
        __syncthreads();
        if (s_fail) return;
        const long long base = static_cast<long long>(t) * kTile, rem = count - base;
        float acc[kVecPerThread][4] = {};
        for (int lp = 0; lp < L; ++lp) {
            const XT *sp = slotA(m * L + lp) + base;
#pragma unroll
            for (int j = 0; j < kVecPerThread; ++j) {
                float v[4];
                Vec4<XT>::load_cg(sp + tile_elem(j), v, clamp_valid(rem, tile_elem(j)), vec);
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[j][i] += v[i];
            }
        }
        const float invL = 1.0f / static_cast<float>(L);
        float *bo = bufB(gid) + static_cast<long long>(tt) * kTile;
#pragma unroll
        for (int j = 0; j < kVecPerThread; ++j) {
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[j][i] *= invL;
            Vec4<float>::store(bo + tile_elem(j), acc[j], clamp_valid(rem, tile_elem(j)), true);
        }
        __syncthreads();
        if (threadIdx.x == 0) st_release_sys(ready_ptr(g, p.fb_off, p.ready_stride, gid, tt), e);
    }

    // ---- stage C: machine-level combine of the slice ----
    for (long long w = blockIdx.x; w < itemsS; w += gridDim.x) {
        const int tt = static_cast<int>(w / k), a = static_cast<int>(w % k);
        const int gid = g.me * k + a, l = gid % L;
        const int t = l * TS + tt;
        if (t >= g.T) continue;
        const int ns = p.mtab.nsrc[a];
        if (threadIdx.x < ns)
            wait_all(ready_ptr(g, p.fb_off, p.ready_stride, p.mtab.src[a][threadIdx.x] * L + l, tt));
        __syncthreads();
        if (s_fail) return;
        const long long base = static_cast<long long>(t) * kTile, rem = count - base;
        float acc[kVecPerThread][4];
        const float *own = bufB(gid) + static_cast<long long>(tt) * kTile;
        const float cs = p.mtab.self_w[a];
#pragma unroll
        for (int j = 0; j < kVecPerThread; ++j) {
            Vec4<float>::load_cg(own + tile_elem(j), acc[j], clamp_valid(rem, tile_elem(j)), true);
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[j][i] *= cs;
        }
        for (int q = 0; q < ns; ++q) {
            const float *sp = bufB(p.mtab.src[a][q] * L + l) + static_cast<long long>(tt) * kTile;
            const float c = p.mtab.coef[a][q];
#pragma unroll
            for (int j = 0; j < kVecPerThread; ++j) {
                float v[4];
                Vec4<float>::load_cg(sp + tile_elem(j), v, clamp_valid(rem, tile_elem(j)), true);
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[j][i] = fmaf(c, v[i], acc[j][i]);
            }
        }
        float *co = bufC(gid) + static_cast<long long>(tt) * kTile;
#pragma unroll
        for (int j = 0; j < kVecPerThread; ++j)
            Vec4<float>::store(co + tile_elem(j), acc[j], clamp_valid(rem, tile_elem(j)), true);
        __syncthreads();
        if (threadIdx.x == 0) st_release_sys(ready_ptr(g, p.fc_off, p.ready_stride, gid, tt), e);
    }

    // ---- stage D: gather the machine result ----
    for (long long w = blockIdx.x; w < itemsA; w += gridDim.x) {
        const int t = static_cast<int>(w / k), a = static_cast<int>(w % k);
        const int gid = g.me * k + a, m = gid / L;
        const int lo = t / TS, tt = t - lo * TS;
        const int owner = m * L + lo;
        if (threadIdx.x == 0) wait_all(ready_ptr(g, p.fc_off, p.ready_stride, owner, tt));
        __syncthreads();
        if (s_fail) return;
        const long long base = static_cast<long long>(t) * kTile, rem = count - base;
        const float *cp = bufC(owner) + static_cast<long long>(tt) * kTile;
        XT *yr = static_cast<XT *>(p.y) + static_cast<long long>(a) * count + base;
#pragma unroll
        for (int j = 0; j < kVecPerThread; ++j) {
            float v[4];
            const int vl = clamp_valid(rem, tile_elem(j));
            Vec4<float>::load_cg(cp + tile_elem(j), v, vl, true);
            Vec4<XT>::store(yr + tile_elem(j), v, vl, vec);
        }
    }

    last_cta(pad, [&] {
        pad->epoch = e;
        publish_done(g, e);
    });
}

// --------------------------------------------------------------------------
// Device barrier over all processes (P:580 bf.barrier()).
__global__ void barrier_kernel(const __grid_constant__ Geometry g, unsigned long long epoch) {
    Pad *pad = pad_of(g, g.me);
    if (threadIdx.x < g.nprocs) st_release_sys(&pad_of(g, threadIdx.x)->bar_from[g.me], epoch);
    if (threadIdx.x < g.nprocs) spin_ge(g, &pad->bar_from[threadIdx.x], epoch);
}

__global__ void set_u64_kernel(unsigned long long *dst, unsigned long long v) { *dst = v; }

// --------------------------------------------------------------------------
int max_coresident(const void *func, int threads, size_t smem) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, func, threads, smem);
    return per_sm * sms;
}

template <typename XT, typename GT, typename WT, typename YT, bool HAS_G>
static cudaError_t launch_exch_t(const ExchParams &p, int grid, cudaStream_t s) {
    auto fn = exchange_kernel<XT, GT, WT, YT, HAS_G>;
    const unsigned smem = Pipe<XT, GT, WT, HAS_G>::BYTES;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void *>(fn),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int maxg = max_coresident(reinterpret_cast<const void *>(fn), kExchThreads, smem);
    if (grid <= 0 || grid > maxg) grid = maxg;
    const long long items = static_cast<long long>(p.geo.k) * p.geo.T;
    if (grid > items) grid = static_cast<int>(items < p.geo.k ? p.geo.k : items);
    if (grid < 1) grid = 1;
    void *args[] = {const_cast<ExchParams *>(&p)};
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(fn), dim3(grid), dim3(kExchThreads), args,
                                       smem, s);
}

cudaError_t launch_exchange(const ExchParams &p, int x_kind, int g_kind, int wire_kind, int y_kind,
                            int has_g, int grid, cudaStream_t s) {
    // neighbor_allreduce: x = wire = y dtype
    if (!has_g) {
        if (x_kind == 0 && wire_kind == 0 && y_kind == 0)
            return launch_exch_t<float, float, float, float, false>(p, grid, s);
        if (x_kind == 1 && wire_kind == 1 && y_kind == 1)
            return launch_exch_t<bf16, bf16, bf16, bf16, false>(p, grid, s);
        return cudaErrorInvalidValue;
    }
    // ATC: fp32 master x and y
    if (x_kind != 0 || y_kind != 0) return cudaErrorInvalidValue;
    if (g_kind == 0 && wire_kind == 0) return launch_exch_t<float, float, float, float, true>(p, grid, s);
    if (g_kind == 0 && wire_kind == 1) return launch_exch_t<float, float, bf16, float, true>(p, grid, s);
    if (g_kind == 1 && wire_kind == 0) return launch_exch_t<float, bf16, float, float, true>(p, grid, s);
    if (g_kind == 1 && wire_kind == 1) return launch_exch_t<float, bf16, bf16, float, true>(p, grid, s);
    return cudaErrorInvalidValue;
}

cudaError_t launch_hier(const HierParams &p, int x_kind, int grid, cudaStream_t s) {
    const void *fn = x_kind == 0 ? reinterpret_cast<const void *>(hier_kernel<float>)
                                 : reinterpret_cast<const void *>(hier_kernel<bf16>);
    const int maxg = max_coresident(fn, kThreads, 0);
    if (grid <= 0 || grid > maxg) grid = maxg;
    const long long items = static_cast<long long>(p.geo.k) * p.geo.T;
    if (grid > items) grid = static_cast<int>(items < p.geo.k ? p.geo.k : items);
    if (grid < 1) grid = 1;
    void *args[] = {const_cast<HierParams *>(&p)};
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), args, 0, s);
}

cudaError_t launch_barrier(const Geometry &geo, unsigned long long epoch, cudaStream_t s) {
    barrier_kernel<<<1, 32, 0, s>>>(geo, epoch);
    return cudaGetLastError();
}

cudaError_t launch_set_u64(unsigned long long *dst, unsigned long long v, cudaStream_t s) {
    set_u64_kernel<<<1, 1, 0, s>>>(dst, v);
    return cudaGetLastError();
}

}  // namespace bf
