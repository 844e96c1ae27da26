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

// Shared-memory ring of the TMA-prefetched x / g tiles (2 stages).
template <typename XT, typename GT, bool HAS_G>
struct Ring {
    static constexpr unsigned kXBytes = kTile * sizeof(XT);
    static constexpr unsigned kGBytes = HAS_G ? kTile * sizeof(GT) : 0;
    static constexpr unsigned kBytes = 2 * (kXBytes + kGBytes);
};

template <typename XT, typename GT, typename WT, typename YT, bool HAS_G>
__global__ void __launch_bounds__(kThreads, BF_MINB) exchange_kernel(const __grid_constant__ ExchParams p) {
    using R = Ring<XT, GT, HAS_G>;
    extern __shared__ __align__(128) unsigned char ring[];
    __shared__ SharedTab st;
    __shared__ __align__(8) unsigned long long full[2];
    __shared__ int s_fail;
    const Geometry &g = p.geo;
    Pad *pad = pad_of(g, g.me);
    if (aborted(g)) return;
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long *>(&pad->epoch) + 1;
    const int parity = static_cast<int>(e & 1);
    const bool sys = g.nprocs > 1;   // flags of agents on other GPUs need system scope

    if (threadIdx.x == 0) {
        s_fail = 0;
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_mbar_init();
    }
    if (!war_wait(g, e)) return;
    if (p.wmode == kWDynamic) write_descriptors(p, e);
    if (!resolve_sources(p, e, st)) return;

    const bool vec = g.vec_ok != 0;
    const long long count = g.count;
    const int k = g.k;
    const long long items = static_cast<long long>(k) * g.T;
    // an item is staged by TMA when its rows are 16B-aligned and the tile is full
    auto staged = [&](long long w) {
        return vec && (count - static_cast<long long>(w / k) * kTile) >= kTile;
    };
    auto issue = [&](long long w, int stage) {   // thread 0 only
        const int t = static_cast<int>(w / k), a = static_cast<int>(w % k);
        const long long off = static_cast<long long>(a) * count + static_cast<long long>(t) * kTile;
        fence_proxy_async();
        mbar_expect_tx(&full[stage], R::kXBytes + R::kGBytes);
        tma_load_1d(ring + stage * R::kXBytes, static_cast<const XT *>(p.x) + off, R::kXBytes, &full[stage]);
        if constexpr (HAS_G)
            tma_load_1d(ring + 2 * R::kXBytes + stage * R::kGBytes, static_cast<const GT *>(p.g) + off,
                        R::kGBytes, &full[stage]);
    };
    unsigned phase[2] = {0u, 0u};
    if (threadIdx.x == 0 && blockIdx.x < items && staged(blockIdx.x)) issue(blockIdx.x, 0);

    int it = 0;
    for (long long w = blockIdx.x; w < items; w += gridDim.x, ++it) {
        const int t = static_cast<int>(w / k);
        const int a = static_cast<int>(w % k);
        const long long base = static_cast<long long>(t) * kTile;
        const long long rem = count - base;
        const int stage = it & 1;
        // prefetch the next item of this CTA while this one is processed
        const long long wn = w + gridDim.x;
        if (threadIdx.x == 0 && wn < items && staged(wn)) issue(wn, stage ^ 1);

        // ---- Eq. 4 local update (ATC) or plain input (neighbor_allreduce) ----
        float xh[kVecPerThread][4];
        if (staged(w)) {
            mbar_wait_b(g, &full[stage], phase[stage], &s_fail);
            phase[stage] ^= 1u;
            const XT *xs = reinterpret_cast<const XT *>(ring + stage * R::kXBytes);
#pragma unroll
            for (int j = 0; j < kVecPerThread; ++j) Vec4<XT>::load(xs + tile_elem(j), xh[j], 4, true);
            if constexpr (HAS_G) {
                const GT *gs = reinterpret_cast<const GT *>(ring + 2 * R::kXBytes + stage * R::kGBytes);
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j) {
                    float gv[4];
                    Vec4<GT>::load(gs + tile_elem(j), gv, 4, true);
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

        // ---- publish the wire copy into this agent's slot, release flag ----
        WT *mine = at<WT>(g.peer_base[g.me], p.slot_off + a * p.slot_agent_stride +
                                                 parity * p.slot_parity_stride) + base;
#pragma unroll
        for (int j = 0; j < kVecPerThread; ++j)
            Vec4<WT>::store(mine + tile_elem(j), xh[j], clamp_valid(rem, tile_elem(j)), vec);
        __syncthreads();
        if (threadIdx.x == 0)
            st_release(ready_ptr(g, p.ready_off, p.ready_stride, g.me * k + a, t), e, sys);

        // ---- wait for the in-neighbours' tile t ----
        const int ns = st.nsrc[a];
        if (threadIdx.x < ns) {
            if (!spin_ge(g, ready_ptr(g, p.ready_off, p.ready_stride, st.src[a][threadIdx.x], t), e, sys))
                s_fail = 1;
        }
        __syncthreads();
        if (s_fail) {
            // drain the in-flight prefetch before the CTA exits (its smem may be reused)
            if (threadIdx.x == 0 && wn < items && staged(wn)) {
                volatile int no_fail = 0;
                mbar_wait_b(g, &full[stage ^ 1], phase[stage ^ 1], &no_fail);
            }
            return;
        }

        // ---- Eq. 5 / Eq. 9 weighted combine in fp32 ----
        float acc[kVecPerThread][4];
        const float cs = st.self_w[a];
#pragma unroll
        for (int j = 0; j < kVecPerThread; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[j][i] = cs * xh[j][i];
        for (int q = 0; q < ns; ++q) {
            const int src = st.src[a][q];
            const float c = st.coef[a][q];
            const WT *sp = at<const WT>(g.peer_base[src / k],
                                        p.slot_off + (src % k) * p.slot_agent_stride +
                                            parity * p.slot_parity_stride) + base;
            float v[kVecPerThread][4];
#pragma unroll
            for (int j = 0; j < kVecPerThread; ++j)
                Vec4<WT>::load_cg(sp + tile_elem(j), v[j], clamp_valid(rem, tile_elem(j)), vec);
#pragma unroll
            for (int j = 0; j < kVecPerThread; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[j][i] = fmaf(c, v[j][i], acc[j][i]);
        }

        // ---- store (cast) ----
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

    last_cta(pad, [&] {
        pad->epoch = e;
        if (p.wmode == kWSchedule) pad->round = pad->round + 1;
        publish_done(g, e);
    });
}

#ifndef BF_LAG
#define BF_LAG 3
#endif
#ifndef BF_PSTAGES
#define BF_PSTAGES 3
#endif
#ifndef BF_CSTAGES
#define BF_CSTAGES 2
#endif
#ifndef BF_NPEER
#define BF_NPEER 2
#endif
constexpr int kConsumerWarps = kThreads / 32;          // 8 consumer warps
constexpr int kExchThreads = kThreads + 96;            // + 2 producer warps + 1 signal warp
constexpr int kPub = 16;                               // ring of "published" notifications

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

// Per-CTA shared-memory pipelines.
//   publish ring (PS stages): x / g tile of an item to publish (DRAM reads in flight)
//   combine ring (CS stages): the tiles combined for an item.  When the wire copy
//   IS the fp32 x_half (fp32 wire, or neighbor_allreduce) the self term is the
//   agent's own published tile, staged like a neighbour's (an L2 hit); for ATC
//   with a bf16 wire the stage re-reads x / g to recompute the fp32 x_half (R18).
template <typename XT, typename GT, typename WT, bool HAS_G>
struct Pipe {
    static constexpr int D = BF_LAG, PS = BF_PSTAGES, CS = BF_CSTAGES, NP = BF_NPEER;
    static constexpr bool SELF_XG = HAS_G && sizeof(WT) < 4;
    static constexpr unsigned XB = kTile * sizeof(XT);
    static constexpr unsigned GB = HAS_G ? kTile * sizeof(GT) : 0;
    static constexpr unsigned PB = kTile * sizeof(WT);
    static constexpr unsigned XG = XB + GB;
    static constexpr int NT = NP + (SELF_XG ? 0 : 1);               // staged tiles per combine stage
    static constexpr unsigned CST = (SELF_XG ? XG : 0) + NT * PB;
    static constexpr unsigned BYTES = PS * XG + CS * CST;
};

// exchange_pipe_kernel: warp-specialised persistent pipeline, one CTA per SM
// (alternative to exchange_kernel, selected with BF_EXCH=pipe).
//   producer A : TMA bulk loads of the x / g tiles of items to publish
//   producer B : TMA bulk loads of the x / g tiles of items to combine (L2 hits,
//                they were published D items earlier), then acquire the
//                in-neighbours' ready flags of the tile and LDGSTS (cp.async)
//                their published tiles -- over NVLink for agents on other GPUs,
//                from L2 for agents on this GPU
//   signal     : releases the ready flag of every published tile (the release
//                fence runs off the consumers' critical path)
//   consumers  : iteration c publishes item c+D (Eq. 4 adapt, wire copy into
//                this agent's IPC slot) and combines item c (Eq. 5 / Eq. 9,
//                fp32) from shared memory.
// Publishing D items ahead means a neighbour's tile is normally published long
// before anybody needs it.  Deadlock freedom: items are visited in increasing
// tile order; publish-side loads never wait on other agents; a tile is
// published before its owner waits on the tile of any later item; all CTAs are
// co-resident (cooperative launch) and grid >= local agents.  A fault never
// exits early: waits fail fast, garbage is computed, the fault is latched, and
// no TMA or cp.async is left in flight.
template <typename XT, typename GT, typename WT, typename YT, bool HAS_G>
__global__ void __launch_bounds__(kExchThreads, 1) exchange_pipe_kernel(const __grid_constant__ ExchParams p) {
    using P = Pipe<XT, GT, WT, HAS_G>;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ SharedTab st;
    __shared__ __align__(8) unsigned long long fullP[P::PS], emptyP[P::PS];
    __shared__ __align__(8) unsigned long long published[kPub], signaled[kPub];
    __shared__ __align__(8) unsigned long long fullC[P::CS], emptyC[P::CS];
    __shared__ int s_fail, drain_fail;
    volatile int *const fail = &s_fail;
    const Geometry &g = p.geo;
    Pad *pad = pad_of(g, g.me);
    if (aborted(g)) return;
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long *>(&pad->epoch) + 1;
    const int parity = static_cast<int>(e & 1);
    const bool sys = g.nprocs > 1;   // flags of agents on other GPUs need system scope

    if (threadIdx.x == 0) {
        s_fail = 0;
        drain_fail = 0;
        for (int i = 0; i < P::PS; ++i) {
            mbar_init(&fullP[i], 1);
            mbar_init(&emptyP[i], kConsumerWarps);
        }
        for (int i = 0; i < kPub; ++i) {
            mbar_init(&published[i], kConsumerWarps);
            mbar_init(&signaled[i], 1);
        }
        for (int i = 0; i < P::CS; ++i) {
            mbar_init(&fullC[i], 1 + 32);                 // TMA / plain arrive + 32 cp.async lanes
            mbar_init(&emptyC[i], kConsumerWarps);
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
    const int items = k * g.T;
    const int nfull = static_cast<int>(count / kTile);   // tiles that are full
    const int nmine = static_cast<int>(blockIdx.x) < items
                          ? (items - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                                static_cast<int>(gridDim.x)
                          : 0;
    auto staged = [&](int t) { return vec && t < nfull; };   // TMA needs 16B-aligned rows and a full tile
    unsigned char *const ringP = smem;
    unsigned char *const ringC = smem + P::PS * P::XG;
    auto xP = [&](int s) { return ringP + s * P::XG; };
    auto xC = [&](int s) { return ringC + s * P::CST; };
    auto tC = [&](int s, int q) { return ringC + s * P::CST + (P::SELF_XG ? P::XG : 0) + q * P::PB; };
    auto slot_of = [&](int agent) {
        return at<WT>(g.peer_base[agent / k],
                      p.slot_off + (agent % k) * p.slot_agent_stride + parity * p.slot_parity_stride);
    };
    auto failed = [&]() { return *reinterpret_cast<volatile int *>(&s_fail) != 0; };
    auto tma_xg = [&](int t, int a, unsigned char *dst, unsigned long long *bar) {   // lane 0 only
        const long long off = static_cast<long long>(a) * count + static_cast<long long>(t) * kTile;
        fence_proxy_async();
        mbar_expect_tx(bar, P::XG);
        tma_load_1d(dst, static_cast<const XT *>(p.x) + off, P::XB, bar);
        if constexpr (HAS_G) tma_load_1d(dst + P::XB, static_cast<const GT *>(p.g) + off, P::GB, bar);
    };
    // agent whose published tile is staged in tile slot q of a combine stage
    auto staged_agent = [&](int a, int q) {
        if constexpr (P::SELF_XG) return static_cast<int>(st.src[a][q]);
        return q == 0 ? g.me * k + a : static_cast<int>(st.src[a][q - 1]);
    };
    auto n_staged = [&](int a) { return min(st.nsrc[a], P::NP) + (P::SELF_XG ? 0 : 1); };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == kConsumerWarps) {
        // ====================== producer A: publish-side x / g ======================
        ItemIt it(blockIdx.x, gridDim.x, k);
        int issued = 0;
        for (int c = 0; c < nmine; ++c, it.next()) {
            const int s = c % P::PS;
            bool okw = true;   // lane 0 waits, the warp follows its verdict (no divergent break)
            if (c >= P::PS && lane == 0) okw = mbar_wait_b(g, &emptyP[s], static_cast<unsigned>(c / P::PS - 1) & 1u, fail);
            if (!__shfl_sync(0xffffffffu, okw, 0)) break;
            issued = c + 1;
            if (lane == 0) {
                if (staged(it.t))
                    tma_xg(it.t, it.a, xP(s), &fullP[s]);
                else
                    mbar_arrive(&fullP[s]);
            }
            __syncwarp();
        }
        // drain: every armed phase completes before the CTA can exit
        if (lane == 0)
            for (int c = max(0, issued - P::PS); c < issued; ++c)
                mbar_wait_b(g, &fullP[c % P::PS], static_cast<unsigned>(c / P::PS) & 1u, &drain_fail);
    } else if (warp == kConsumerWarps + 1) {
        // ========== producer B: the published tiles combined for each item ==========
        ItemIt it(blockIdx.x, gridDim.x, k);
        int issued = 0;
        for (int c = 0; c < nmine; ++c, it.next()) {
            const int s = c % P::CS;
            bool okw = true;
            if (c >= P::CS && lane == 0) okw = mbar_wait_b(g, &emptyC[s], static_cast<unsigned>(c / P::CS - 1) & 1u, fail);
            if (!__shfl_sync(0xffffffffu, okw, 0)) break;
            issued = c + 1;
            const int t = it.t, a = it.a;
            const long long base = static_cast<long long>(t) * kTile;
            if (lane == 0) {
                if (P::SELF_XG && staged(t))
                    tma_xg(t, a, xC(s), &fullC[s]);
                else
                    mbar_arrive(&fullC[s]);
            }
            const int nt = n_staged(a);
            bool good = true;
            if (lane < nt && !failed())
                good = spin_ge(g, ready_ptr(g, p.ready_off, p.ready_stride, staged_agent(a, lane), t), e, sys);
            if (!__all_sync(0xffffffffu, good) && lane == 0) s_fail = 1;
            __syncwarp();
            if (!failed()) {
                const long long rem_bytes = (count - base) * static_cast<long long>(sizeof(WT));
                for (int q = 0; q < nt; ++q) {
                    const unsigned char *src =
                        reinterpret_cast<const unsigned char *>(slot_of(staged_agent(a, q)) + base);
                    unsigned char *dst = tC(s, q);
#pragma unroll 4
                    for (int ch = lane; ch < static_cast<int>(P::PB / 16); ch += 32) {
                        const long long left = rem_bytes - 16ll * ch;
                        const unsigned nb = left >= 16 ? 16u : (left <= 0 ? 0u : static_cast<unsigned>(left));
                        cp_async16(dst + 16 * ch, nb ? src + 16 * ch : src, nb);
                    }
                }
            }
            cp_async_mbar_arrive_noinc(&fullC[s]);
        }
        if (lane == 0)
            for (int c = max(0, issued - P::CS); c < issued; ++c)
                mbar_wait_b(g, &fullC[c % P::CS], static_cast<unsigned>(c / P::CS) & 1u, &drain_fail);
    } else if (warp == kConsumerWarps + 2) {
        // ======== signal warp: release the ready flags of published tiles ========
        // One release fence covers every tile already published (batch), so the
        // fence cost is paid per batch, not per tile, and never by the consumers.
        if (lane == 0) {
            ItemIt it(blockIdx.x, gridDim.x, k);
            int c = 0;
            while (c < nmine) {
                const bool okp = mbar_wait_b(g, &published[c % kPub], static_cast<unsigned>(c / kPub) & 1u, fail);
                int c_end = c + 1;
                while (okp && c_end < nmine && c_end - c < kPub / 2 &&
                       mbar_test(&published[c_end % kPub], static_cast<unsigned>(c_end / kPub) & 1u))
                    ++c_end;
                if (okp) fence_acq_rel(sys);
                for (int i = c; i < c_end; ++i, it.next()) {
                    if (okp) st_relaxed(ready_ptr(g, p.ready_off, p.ready_stride, g.me * k + it.a, it.t), e, sys);
                    mbar_arrive(&signaled[i % kPub]);
                }
                c = c_end;
            }
        }
        __syncwarp();
    } else {
        // =============================== consumers ===============================
        // x_half of item (t, a) from a staged x/g tile, or straight from global memory
        auto adapt = [&](int t, int a, const unsigned char *stage, float (&xh)[kVecPerThread][4]) {
            const long long base = static_cast<long long>(t) * kTile, rem = count - base;
            if (staged(t)) {
                const XT *xsm = reinterpret_cast<const XT *>(stage);
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j) Vec4<XT>::load(xsm + tile_elem(j), xh[j], 4, true);
                if constexpr (HAS_G) {
                    const GT *gsm = reinterpret_cast<const GT *>(stage + P::XB);
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
        ItemIt itP(blockIdx.x, gridDim.x, k);   // next item to publish
        ItemIt itC(blockIdx.x, gridDim.x, k);   // next item to combine
        for (int c = -P::D; c < nmine; ++c) {
            // ---- publish item c + D: Eq. 4 local update, wire copy into the slot ----
            const int cp = c + P::D;
            if (cp >= 0 && cp < nmine) {
                const int s = cp % P::PS;
                const int t = itP.t, a = itP.a;
                const long long base = static_cast<long long>(t) * kTile, rem = count - base;
                mbar_wait_b(g, &fullP[s], static_cast<unsigned>(cp / P::PS) & 1u, fail);
                float xh[kVecPerThread][4];
                adapt(t, a, xP(s), xh);
                __syncwarp();
                if (lane == 0) mbar_arrive(&emptyP[s]);   // x / g consumed: producer A may refill
                WT *mine = slot_of(g.me * k + a) + base;
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j)
                    Vec4<WT>::store(mine + tile_elem(j), xh[j], clamp_valid(rem, tile_elem(j)), true);
                __syncwarp();
                if (lane == 0) {
                    if (cp >= kPub)   // the signal warp has consumed the notification kPub items back
                        mbar_wait_b(g, &signaled[cp % kPub], static_cast<unsigned>(cp / kPub - 1) & 1u, fail);
                    mbar_arrive(&published[cp % kPub]);   // the signal warp releases the flag
                }
                itP.next();
            }
            if (c < 0) continue;
            // ---- combine item c: Eq. 5 / Eq. 9 in fp32 ----
            const int t = itC.t, a = itC.a;
            itC.next();
            const long long base = static_cast<long long>(t) * kTile, rem = count - base;
            const int s = c % P::CS;
            mbar_wait_b(g, &fullC[s], static_cast<unsigned>(c / P::CS) & 1u, fail);
            float acc[kVecPerThread][4];
            const float cs = st.self_w[a];
            int q0 = 0;
            if constexpr (P::SELF_XG) {
                adapt(t, a, xC(s), acc);   // fp32 x_half for the self term (R18)
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[j][i] *= cs;
            } else {
                // own published tile == the fp32 x_half (fp32 wire) or x itself
                const WT *sm0 = reinterpret_cast<const WT *>(tC(s, 0));
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j) {
                    Vec4<WT>::load(sm0 + tile_elem(j), acc[j], 4, true);
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[j][i] *= cs;
                }
                q0 = 1;
            }
            const int ns = st.nsrc[a];
            const int np = min(ns, P::NP);
            for (int q = 0; q < np; ++q) {
                const WT *psm = reinterpret_cast<const WT *>(tC(s, q0 + q));
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
            if (lane == 0) mbar_arrive(&emptyC[s]);
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
// exchange_chunk_kernel (kernel 2, default): chunk-granular synchronisation.
// The tiles are grouped into chunks of CT tiles (per agent).  Every CTA walks
// its items (grid-stride, tile-major) twice: it PUBLISHES them (Eq. 4 adapt,
// wire copy into the IPC slot) and COMBINES them (Eq. 5 / Eq. 9), the combine
// of chunk c running after the CTA has published everything up to chunk c+1.
// A CTA that has published all its items of a chunk bumps the chunk's counter;
// the CTA that completes the count releases the chunk flag once (system scope
// if other GPUs read it).  A combine waits once per chunk for the chunk flags
// of every process -- no per-tile flag traffic, no per-tile fences, and the
// one-chunk lag means the flags are normally already set.
// Deadlock freedom: a CTA never waits while holding an un-counted chunk that a
// waiter needs (it publishes chunk c+1 before waiting for chunk c), and all CTAs
// are co-resident (cooperative launch).
template <typename XT, typename GT, typename WT, typename YT, bool HAS_G>
__global__ void __launch_bounds__(kThreads, BF_MINB) exchange_chunk_kernel(const __grid_constant__ ExchParams p) {
    using R = Ring<XT, GT, HAS_G>;
    extern __shared__ __align__(128) unsigned char ring[];
    __shared__ SharedTab st;
    __shared__ __align__(8) unsigned long long full[2];
    __shared__ int s_fail;
    const Geometry &g = p.geo;
    Pad *pad = pad_of(g, g.me);
    if (aborted(g)) return;
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long *>(&pad->epoch) + 1;
    const int parity = static_cast<int>(e & 1);
    const bool sys = g.nprocs > 1;
    if (threadIdx.x == 0) {
        s_fail = 0;
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_mbar_init();
    }
    bool ok = war_wait(g, e);
    if (p.wmode == kWDynamic) write_descriptors(p, e);
    ok = resolve_sources(p, e, st) && ok;
    if (!ok) return;   // fault latched; nothing in flight yet

    const bool vec = g.vec_ok != 0;
    const long long count = g.count;
    const int k = g.k, G = gridDim.x;
    const int items = k * g.T;
    const int CT = p.chunk_tiles;
    const int NC = (g.T + CT - 1) / CT;
    const int nfull = static_cast<int>(count / kTile);
    const int nmine = static_cast<int>(blockIdx.x) < items ? (items - static_cast<int>(blockIdx.x) + G - 1) / G : 0;
    unsigned *cnt = at<unsigned>(g.peer_base[g.me], p.ccnt_off);
    unsigned long long *cflag = at<unsigned long long>(g.peer_base[g.me], p.cflag_off);
    auto staged = [&](int t) { return vec && t < nfull; };
    auto slot_of = [&](int agent) {
        return at<WT>(g.peer_base[agent / k],
                      p.slot_off + (agent % k) * p.slot_agent_stride + parity * p.slot_parity_stride);
    };
#ifndef BF_HINTS
#define BF_HINTS 1
#endif
    // BF_HINTS: 0 none, 1 streaming data evict-first, 2 + published tiles evict-last
    const unsigned long long pol_stream = BF_HINTS >= 1 ? policy_evict_first() : policy_evict_normal();
    const unsigned long long pol_keep = BF_HINTS >= 2 ? policy_evict_last() : policy_evict_normal();
    auto issue = [&](const ItemIt &it, int stage) {   // thread 0: TMA of the x / g tiles of a publish item
        const long long off = static_cast<long long>(it.a) * count + static_cast<long long>(it.t) * kTile;
        fence_proxy_async();
        mbar_expect_tx(&full[stage], R::kXBytes + R::kGBytes);
        tma_load_1d_hint(ring + stage * R::kXBytes, static_cast<const XT *>(p.x) + off, R::kXBytes, &full[stage],
                         pol_stream);
        if constexpr (HAS_G)
            tma_load_1d_hint(ring + 2 * R::kXBytes + stage * R::kGBytes, static_cast<const GT *>(p.g) + off,
                             R::kGBytes, &full[stage], pol_stream);
    };
    // x_half of (t, a) from global memory (unstaged publish items, bf16-wire self terms)
    auto adapt_global = [&](int t, int a, float (&xh)[kVecPerThread][4]) {
        const long long base = static_cast<long long>(t) * kTile, rem = count - base;
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
    };

    int counted = 0;   // this CTA has counted chunks [0, counted)
    auto count_upto = [&](int c_excl) {   // uniform
        __syncthreads();   // every slot store of this CTA for those chunks is issued (CTA scope)
        if (threadIdx.x == 0) {
            __threadfence();   // ... and visible at GPU scope before the counters
            for (int c = counted; c < c_excl; ++c) {
                const unsigned old = atomicAdd(&cnt[c], 1u);
                if (old == static_cast<unsigned>(G) - 1) {   // last CTA of this GPU for chunk c
                    cnt[c] = 0;
                    fence_acq_rel(sys);
                    st_relaxed(&cflag[c], e, sys);
                }
            }
        }
        counted = c_excl;
    };

    ItemIt pub(blockIdx.x, G, k), comb(blockIdx.x, G, k);
    int mp = 0, mc = 0, waited = -1, it_pub = 0;
    unsigned phase[2] = {0u, 0u};
    if (threadIdx.x == 0 && nmine > 0 && staged(pub.t)) issue(pub, 0);
    if (nmine == 0) count_upto(NC);
    bool failed = false;
    while (mp < nmine || mc < nmine) {
        const bool do_pub = mp < nmine && (mc >= nmine || pub.t / CT <= comb.t / CT + 1);
        if (do_pub) {
            // ---- publish item mp ----
            const int t = pub.t, a = pub.a;
            const long long base = static_cast<long long>(t) * kTile, rem = count - base;
            const int stage = it_pub & 1;
            ItemIt nxt = pub;
            nxt.next();
            // every warp has finished reading stage^1 (item mp-1) and has waited on its
            // phase before thread 0 re-arms it: a barrier can never run two phases ahead
            __syncthreads();
            if (threadIdx.x == 0 && mp + 1 < nmine && staged(nxt.t)) issue(nxt, stage ^ 1);
            float xh[kVecPerThread][4];
            if (staged(t)) {
                mbar_wait_b(g, &full[stage], phase[stage], &s_fail);
                phase[stage] ^= 1u;
                const XT *xs = reinterpret_cast<const XT *>(ring + stage * R::kXBytes);
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j) Vec4<XT>::load(xs + tile_elem(j), xh[j], 4, true);
                if constexpr (HAS_G) {
                    const GT *gs = reinterpret_cast<const GT *>(ring + 2 * R::kXBytes + stage * R::kGBytes);
#pragma unroll
                    for (int j = 0; j < kVecPerThread; ++j) {
                        float gv[4];
                        Vec4<GT>::load(gs + tile_elem(j), gv, 4, true);
#pragma unroll
                        for (int i = 0; i < 4; ++i) xh[j][i] = fmaf(-p.lr, gv[i], xh[j][i]);
                    }
                }
            } else {
                adapt_global(t, a, xh);
            }
            WT *mine = slot_of(g.me * k + a) + base;
#pragma unroll
            for (int j = 0; j < kVecPerThread; ++j)
                Vec4<WT>::store_hint(mine + tile_elem(j), xh[j], clamp_valid(rem, tile_elem(j)), true, pol_keep);
            ++it_pub;
            ++mp;
            pub = nxt;
            const int next_chunk = mp < nmine ? pub.t / CT : NC;
            if (next_chunk > counted) count_upto(next_chunk);
        } else {
            // ---- combine item mc (its chunk's flags: once per chunk) ----
            const int t = comb.t, a = comb.a;
            const int cc = t / CT;
            if (cc != waited) {
                bool good = true;
                if (threadIdx.x < g.nprocs && !failed)
                    good = spin_ge(g, at<unsigned long long>(g.peer_base[threadIdx.x], p.cflag_off) + cc, e, sys);
                failed = !__syncthreads_and(good) || failed;
                waited = cc;
            }
            const long long base = static_cast<long long>(t) * kTile, rem = count - base;
            float acc[kVecPerThread][4];
            const float cs = st.self_w[a];
            if constexpr (HAS_G && sizeof(WT) < 4) {
                adapt_global(t, a, acc);   // fp32 x_half for the self term (R18); L2 hit
            } else {
                const WT *own = slot_of(g.me * k + a) + base;   // == fp32 x_half (or x)
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j)
                    Vec4<WT>::load_cg(own + tile_elem(j), acc[j], clamp_valid(rem, tile_elem(j)), true);
            }
#pragma unroll
            for (int j = 0; j < kVecPerThread; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[j][i] *= cs;
            const int ns = st.nsrc[a];
            for (int q = 0; q < ns; ++q) {
                const WT *sp = slot_of(st.src[a][q]) + base;
                const float c = st.coef[a][q];
                float v[kVecPerThread][4];
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j)
                    Vec4<WT>::load_cg(sp + tile_elem(j), v[j], clamp_valid(rem, tile_elem(j)), true);
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[j][i] = fmaf(c, v[j][i], acc[j][i]);
            }
            if (p.awc) {   // AWC (Eq. 16): x_i <- sum_j w_ij x_j - lr * g_i
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j) {
                    float gv[4];
                    const long long off = static_cast<long long>(a) * count + base + tile_elem(j);
                    if (p.g_bf16)
                        Vec4<bf16>::load(static_cast<const bf16 *>(p.g) + off, gv, clamp_valid(rem, tile_elem(j)), vec);
                    else
                        Vec4<float>::load(static_cast<const float *>(p.g) + off, gv, clamp_valid(rem, tile_elem(j)),
                                          vec);
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[j][i] = fmaf(-p.lr, gv[i], acc[j][i]);
                }
            }
            YT *yr = static_cast<YT *>(p.y) + static_cast<long long>(a) * count + base;
#pragma unroll
            for (int j = 0; j < kVecPerThread; ++j)
                Vec4<YT>::store_hint(yr + tile_elem(j), acc[j], clamp_valid(rem, tile_elem(j)), vec, pol_stream);
            if (p.shadow) {
                bf16 *sr = static_cast<bf16 *>(p.shadow) + static_cast<long long>(a) * count + base;
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j)
                    Vec4<bf16>::store_hint(sr + tile_elem(j), acc[j], clamp_valid(rem, tile_elem(j)), vec, pol_stream);
            }
            comb.next();
            ++mc;
        }
    }
    if (counted < NC) count_upto(NC);
    if (failed) return;
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
    const int kind = p.kernel;
    const bool pipe = kind == 1;
    const void *fn = pipe ? reinterpret_cast<const void *>(exchange_pipe_kernel<XT, GT, WT, YT, HAS_G>)
                          : (kind == 2 ? reinterpret_cast<const void *>(exchange_chunk_kernel<XT, GT, WT, YT, HAS_G>)
                                       : reinterpret_cast<const void *>(exchange_kernel<XT, GT, WT, YT, HAS_G>));
    const unsigned smem = pipe ? Pipe<XT, GT, WT, HAS_G>::BYTES : Ring<XT, GT, HAS_G>::kBytes;
    const int threads = pipe ? kExchThreads : kThreads;
    static bool attr_set[3] = {false, false, false};
    if (!attr_set[kind]) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_set[kind] = true;
    }
    const int maxg = max_coresident(fn, threads, smem);
    if (grid <= 0 || grid > maxg) grid = maxg;
    const long long items = static_cast<long long>(p.geo.k) * p.geo.T;
    if (grid > items) grid = static_cast<int>(items < p.geo.k ? p.geo.k : items);
    if (grid < 1) grid = 1;
    void *args[] = {const_cast<ExchParams *>(&p)};
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(threads), args, smem, s);
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
