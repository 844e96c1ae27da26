// exchange.cu -- the partial-averaging hot path on sm_100a: the chunked
// exchange kernel (kernel 2, any number of local agents), the dispatch to the
// local-agent fused kernel (kernel 3, exchange_fused.cuh), the hierarchical
// kernel and the device barrier.
//
// Every exchange is ONE persistent, cooperative launch per call that fuses
//   Eq. 4 local update (ATC)      x_half = x - lr*g          (registers)
//   publish + signal                      wire(x_half) -> own IPC slot, release flag
//   neighbour exchange (Eq. 5 / Eq. 9)    acquire peers' flags, loads over
//                                         NVLink (other GPU) or L2 (same GPU)
//   weighted combine + store              y = w_ii x_half + sum_j w_ij wire_j (fp32 FMA)
// chunk by chunk, so HBM traffic, NVLink traffic and the wait for the slowest
// neighbour overlap across the CTAs of the grid.
//
// Deadlock freedom: all CTAs are co-resident (cooperative launch), every CTA
// walks its items in increasing tile order and publishes chunk c+1 before it
// waits for anybody's chunk c; every wait is bounded by the context timeout.
// WAR safety: slots are double-buffered by epoch parity and a writer
// overwrites parity (e&1) only after every process has reported (done_from)
// that it finished reading epoch e-2.
#include <cuda_bf16.h>

#include "exchange_common.cuh"

namespace bf {

cudaError_t launch_fused_nar(const ExchParams &p, int x_kind, int grid, cudaStream_t s);
cudaError_t launch_fused_atc(const ExchParams &p, int g_kind, int wire_kind, int grid, cudaStream_t s);
cudaError_t launch_fused_awc(const ExchParams &p, int g_kind, int wire_kind, int grid, cudaStream_t s);
cudaError_t launch_fused_ed(const ExchParams &p, int g_kind, int wire_kind, int grid, cudaStream_t s);
cudaError_t launch_fused_gt(const ExchParams &p, int wire_kind, int grid, cudaStream_t s);

// Shared-memory ring of the TMA-prefetched x / g tiles (2 stages).
template <typename XT, typename GT, bool HAS_G>
struct Ring {
    static constexpr unsigned kXBytes = kTile * sizeof(XT);
    static constexpr unsigned kGBytes = HAS_G ? kTile * sizeof(GT) : 0;
    static constexpr unsigned kBytes = 2 * (kXBytes + kGBytes);
};

// --------------------------------------------------------------------------
// exchange_chunk_kernel (kernel 2): chunk-granular synchronisation.
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
// Gradient row a of the hierarchical ATC / AWC step, fp32 or bf16.
static __device__ __forceinline__ void load_grad(const HierParams &p, int a, long long off, float v[4], int vl,
                                                 bool vec) {
    if (p.g_bf16)
        Vec4<bf16>::load(static_cast<const bf16 *>(p.g) + static_cast<long long>(a) * p.geo.count + off, v, vl, vec);
    else
        Vec4<float>::load(static_cast<const float *>(p.g) + static_cast<long long>(a) * p.geo.count + off, v, vl, vec);
}

// Hierarchical neighbour allreduce: leader-free, sliced.
//   A: publish x tile t -> slot, flag (H-ATC: x - lr g), only for agents a
//      machine member on another process reads; local members read x in B
//   B: agent (m,l) averages slice l over its machine's L agents (1/L, R12)
//   C: agent (m,l) combines slice l with the machine neighbours' slice l (W_M)
//   D: every agent gathers all slices of its machine's result (H-AWC: - lr g)
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
        if (!((p.pubA >> a) & 1u)) continue;   // no member of its machine on another process
        const long long base = static_cast<long long>(t) * kTile, rem = count - base;
        const XT *xr = static_cast<const XT *>(p.x) + static_cast<long long>(a) * count + base;
        XT *mine = const_cast<XT *>(slotA(g.me * k + a)) + base;
#pragma unroll
        for (int j = 0; j < kVecPerThread; ++j) {
            float v[4];
            const int vl = clamp_valid(rem, tile_elem(j));
            Vec4<XT>::load(xr + tile_elem(j), v, vl, vec);
            if (p.hmode == 1) {   // H-ATC: publish the adapted x - lr g (Eq. 17)
                float gv[4];
                load_grad(p, a, base + tile_elem(j), gv, vl, vec);
#pragma unroll
                for (int i = 0; i < 4; ++i) v[i] = fmaf(-p.lr, gv[i], v[i]);
            }
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
        // members on another process: their published copy (stage A flag)
        if (threadIdx.x < L && (m * L + static_cast<int>(threadIdx.x)) / k != g.me)
            wait_all(ready_ptr(g, p.ready_off, p.ready_stride, m * L + threadIdx.x, t));
        __syncthreads();
        if (s_fail) return;
        const long long base = static_cast<long long>(t) * kTile, rem = count - base;
        float acc[kVecPerThread][4] = {};
        for (int lp = 0; lp < L; ++lp) {
            const int j_agent = m * L + lp;
            if (j_agent / k == g.me) {   // member on this process: straight from x (adapted as in stage A)
                const int aj = j_agent % k;
                const XT *xr = static_cast<const XT *>(p.x) + static_cast<long long>(aj) * count + base;
#pragma unroll
                for (int j = 0; j < kVecPerThread; ++j) {
                    float v[4];
                    const int vl = clamp_valid(rem, tile_elem(j));
                    Vec4<XT>::load(xr + tile_elem(j), v, vl, vec);
                    if (p.hmode == 1) {
                        float gv[4];
                        load_grad(p, aj, base + tile_elem(j), gv, vl, vec);
#pragma unroll
                        for (int i = 0; i < 4; ++i) v[i] = fmaf(-p.lr, gv[i], v[i]);
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[j][i] += v[i];
                }
                continue;
            }
            const XT *sp = slotA(j_agent) + base;
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
            if (p.hmode == 2) {   // H-AWC: combine, then subtract lr g (Eq. 16)
                float gv[4];
                load_grad(p, a, base + tile_elem(j), gv, vl, vec);
#pragma unroll
                for (int i = 0; i < 4; ++i) v[i] = fmaf(-p.lr, gv[i], v[i]);
            }
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
    const void *fn = reinterpret_cast<const void *>(exchange_chunk_kernel<XT, GT, WT, YT, HAS_G>);
    const unsigned smem = Ring<XT, GT, HAS_G>::kBytes;
    static int maxg = 0;   // co-resident CTAs of this instantiation (queried once)
    if (maxg == 0) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        maxg = max_coresident(fn, kThreads, smem);
    }
    if (grid <= 0 || grid > maxg) grid = maxg;
    const long long items = static_cast<long long>(p.geo.k) * p.geo.T;
    if (grid > items) grid = static_cast<int>(items < p.geo.k ? p.geo.k : items);
    if (grid < 1) grid = 1;
    void *args[] = {const_cast<ExchParams *>(&p)};
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), args, smem, s);
}

bool fused_supported(int k, int nprocs) { return k == 1 || k == 2 || k == 4 || (k == 8 && nprocs == 1); }

static cudaError_t launch_fused(const ExchParams &p, int x_kind, int g_kind, int wire_kind, int y_kind, int has_g,
                                int grid, cudaStream_t s) {
    if (p.gt) {   // push-sum gradient tracking: fp32 tensors
        if (x_kind != 0 || y_kind != 0 || g_kind != 0) return cudaErrorInvalidValue;
        return launch_fused_gt(p, wire_kind, grid, s);
    }
    if (p.awc) {   // AWC: fp32 master x, wire = the x value in the wire dtype
        if (x_kind != 0 || y_kind != 0) return cudaErrorInvalidValue;
        return launch_fused_awc(p, p.g_bf16 ? 1 : 0, wire_kind, grid, s);
    }
    if (!has_g) {
        if (x_kind != wire_kind || x_kind != y_kind) return cudaErrorInvalidValue;
        return launch_fused_nar(p, x_kind, grid, s);
    }
    if (p.psi) {   // Exact-Diffusion
        if (x_kind != 0 || y_kind != 0) return cudaErrorInvalidValue;
        return launch_fused_ed(p, g_kind, wire_kind, grid, s);
    }
    if (x_kind != 0 || y_kind != 0) return cudaErrorInvalidValue;
    return launch_fused_atc(p, g_kind, wire_kind, grid, s);
}

cudaError_t launch_exchange(const ExchParams &p, int x_kind, int g_kind, int wire_kind, int y_kind,
                            int has_g, int grid, cudaStream_t s) {
    if (p.kernel == 3) return launch_fused(p, x_kind, g_kind, wire_kind, y_kind, has_g, grid, s);
    // kernel 2 (chunked): any number of local agents
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
