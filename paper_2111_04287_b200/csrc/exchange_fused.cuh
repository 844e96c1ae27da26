// exchange_fused.cuh -- the local-agent fused exchange kernel (kernel 3) and its
// launch templates; instantiated per operation in fused_nar.cu (MODE 0),
// fused_atc.cu (MODE 1) and fused_awc.cu (MODE 2) so they compile in parallel.
#pragma once

#include <cstdlib>
#include <type_traits>

#include "exchange_common.cuh"

namespace bf {

// --------------------------------------------------------------------------
// exchange_fused_kernel (kernel 3, default when the process hosts K = 1, 2, 4
// or 8 agents).  The K agents of one process share one GPU, so their part of
// the exchange never has to leave the SM: a consumer thread loads the same
// 4-element vector of x (and g) of ALL K local agents into registers, forms
// every x_half there (Eq. 4), and combines each agent's local sources straight
// from those registers (Eq. 5 / Eq. 9) -- the K x K local block of W is applied
// in registers.  Only sources on OTHER processes go through the published slots:
//   * a local agent whose x_half is read by another process (pub mask)
//     publishes its wire copy kLead sub-items ahead of the combine;
//   * synchronisation is pairwise between CTAs, not global: sub-item s is
//     handled by CTA s mod G on every process (same grid everywhere), so CTA b
//     only ever needs what CTA b of the source process published.  CTA b
//     releases a progress counter prog[b] = e * 2^24 + (sub-items published)
//     every kBatch sub-items -- no chunk barrier over all CTAs of both GPUs,
//     so a slow CTA delays only its peer;
//   * two warps per CTA do all cross-GPU work off the consumers' path:
//     - a signal warp turns the consumers' "batch published" mbarrier arrivals
//       into system-scope releases of prog[b].  The fence.acq_rel.sys drains
//       the SM's outstanding stores: BF_STATS measured 8-36 us per fence under
//       load, so no warp that moves data may execute it;
//     - a producer warp (lane 0, a non-blocking poll loop) pulls the remote
//       sources' tiles over NVLink with TMA bulk copies (cp.async.bulk, peer
//       addresses of the CUDA-IPC mappings) into a ring of NSLOT shared-memory
//       slots, up to NSLOT tiles ahead of the consumers, so the NVLink latency
//       (calibrated 2.7 us one way) never stalls the HBM stream of the local
//       agents.
// HBM traffic per agent-element drops from x + g + publish + x (16 B fp32) to
// x + g + x (12 B) for every agent without remote readers -- at N = 1 that is
// every agent.
//   MODE 0: neighbor_allreduce (x is the wire value)
//   MODE 1: ATC  (Eq. 4-5, Eq. 17):  y_a = sum_b w_ab (x_b - lr g_b)
//   MODE 2: AWC  (Eq. 16):           y_a = sum_b w_ab x_b - lr g_a
//   MODE 3: Exact-Diffusion (appendix ed-1..ed-3): psi = x - lr g (stored over
//           psi_prev), phi = psi + x - psi_prev, y_a = sum_b w_ab phi_b
//   MODE 4: push-sum gradient tracking, y-step (appendix):
//           y_a = sum_b w_ab (y_b + g_b - g2_b)    (x = y, g = g^(k+1), g2 = g^(k))
//   MODE 5: push-sum gradient tracking, u/v-step (lines 1002-1004):
//           u_a = sum_b w_ab (u_b - lr y_b)  (x = u, g = y),  v_a = sum_b w_ab v_b
//           (scalar weights, gt_weights), x_out_a = u_a / v_a
// Summation order (R18): self, local sources in (a - b) mod K order, then the
// remote sources in table order; a neighbour's term always uses the value as it
// travels on the wire (bf16 RNE for a bf16 wire), the self term the fp32 value.
// Deadlock freedom: consumers publish sub-item m + kLead before they consume
// sub-item m; the communication warp never blocks (it polls), so releases
// always follow publication; every wait is bounded by the context timeout.
// BF_STATS=1 (a diagnostic build, never the default library) records per-CTA
// timings into ExchParams::stats[blockIdx.x * 8 + i]: 0 kernel ns, 1 consumer
// ns waiting for remote tiles, 2 comm ns blocked on peers' progress, 3 comm ns
// blocked on ring slots, 4 fence ns, 5 fences, 6 progress polls, 7 prologue ns.
#ifndef BF_STATS
#define BF_STATS 0
#endif
#if BF_STATS
#define BF_STAT(expr) expr
#else
#define BF_STAT(expr)
#endif
// elements per thread-vector: 16-byte accesses of the x dtype (4 fp32, 8 bf16);
// a sub-item is one vector per consumer thread (1024 fp32 / 2048 bf16 elements)
template <typename XT>
struct FusedVec {
    static constexpr int V = sizeof(XT) >= 4 ? 4 : 8;
};
#ifndef BF_RING_KB
#define BF_RING_KB 64
#endif
// remote-tile ring: BF_RING_KB of shared memory per CTA (2 CTAs per SM fit), as
// many slots as tiles fit -- 16 fp32, 32 bf16 tiles of 1024 elements (measured: a
// 96 KB ring changed nothing for exp-2 and slowed one-peer at N = 2 by 4%)
constexpr int kRingBytes = BF_RING_KB * 1024;
constexpr int kMaxSlot = 64;
#ifndef BF_SLOTX_PUB_STREAM
#define BF_SLOTX_PUB_STREAM 0   // 1: the publish loads of x / g evict-first when the combine reads the slot back
#endif
#ifndef BF_REVERSE
#define BF_REVERSE 1
#endif
#ifndef BF_REVERSE_X
#define BF_REVERSE_X 0   // also across processes (the pull path; every process flips with the epoch)
#endif
#ifndef BF_LEAD
#define BF_LEAD 24
#endif
#ifndef BF_BATCH
#define BF_BATCH 8
#endif
constexpr int kLead = BF_LEAD;             // sub-items published ahead of the combine
constexpr int kBatch = BF_BATCH;           // sub-items per progress release
constexpr int kProgShift = 24;             // prog = epoch << 24 | sub-items published
constexpr int kPubRing = 16;               // "batch published" mbarriers (ring)
// K = 8 local agents (N = 1 of the 8-agent configs) has no remote sources: no
// producer warp, and the 128-register budget of 2 x 256 threads per SM holds
// the 16 vectors in flight per thread without spilling.
// K <= 2 keep too few bytes in flight per thread with one sub-item: they
// combine U = 2 sub-items per iteration (all loads issued first).
template <int K, int XBYTES = 4>
struct FusedCfg {
    static constexpr bool kRing = K < 8;
    static constexpr int kThreadsPerCta = kThreads + (kRing ? 64 : 0);   // 8 consumer warps (+ producer, signal)
    static constexpr int kUnroll = K <= 2 ? 2 : 1;
};

template <int K>
struct LocalMix {
    float c[K][K];                     // c[a][b]: weight of local agent b in agent a's combine
    float rc[K * kMaxN];               // remote entries, agent-major: weight ...
    unsigned char rs[K * kMaxN];       // ... and global source agent (push-only views: up to n - 1 each)
    int rbeg[K + 1];                   // entries of agent a: [rbeg[a], rbeg[a+1])
    unsigned pub;                      // bit a: agent a's x_half is read by another process
    unsigned procs;                    // bit q: process q hosts a remote source
};

template <typename XT, typename GT, typename WT, typename YT, int MODE, int K>
__global__ void __launch_bounds__(FusedCfg<K>::kThreadsPerCta, (K >= 2 ? 2 : 3))
    exchange_fused_kernel(const __grid_constant__ ExchParams p) {
    constexpr bool HAS_G = MODE != 0;
    constexpr int U = FusedCfg<K, sizeof(XT)>::kUnroll;
    constexpr int V = FusedVec<XT>::V;         // elements per thread-vector (16-byte x accesses)
    constexpr int kSubT = kThreads * V;        // elements per sub-item
    constexpr unsigned kSlotBytes = kSubT * sizeof(WT);
    constexpr int kNSlot = kRingBytes / kSlotBytes < kMaxSlot ? kRingBytes / kSlotBytes : kMaxSlot;
    extern __shared__ __align__(128) unsigned char ring[];
    __shared__ SharedTab st;
    __shared__ LocalMix<K> lm;
    __shared__ __align__(8) unsigned long long full[kNSlot], empty[kNSlot], pubbar[kPubRing];
    __shared__ int s_fail;
    __shared__ int s_released;   // batches released by the communication warp
    volatile int *const fail = &s_fail;
    const Geometry &g = p.geo;
    Pad *pad = pad_of(g, g.me);
    if (aborted(g)) return;
    BF_STAT(const unsigned long long t_k0 = globaltimer();)
    BF_STAT(unsigned long long *const stat = p.stats ? p.stats + blockIdx.x * 8 : nullptr;)
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long *>(&pad->epoch) + 1;
    const int parity = static_cast<int>(e & 1);
    const bool sys = g.nprocs > 1;
    if (threadIdx.x == 0) {
        s_fail = 0;
        s_released = 0;
        if (sys) {   // the ring and the publish barriers exist only across processes
            for (int i = 0; i < kNSlot; ++i) {
                mbar_init(&full[i], 1);
                mbar_init(&empty[i], kThreads / 32);
            }
            for (int i = 0; i < kPubRing; ++i) mbar_init(&pubbar[i], kThreads);   // every consumer thread arrives
            fence_mbar_init();
        }
    }
    bool ok = war_wait(g, e);
    if (p.wmode == kWDynamic) write_descriptors(p, e);
    ok = resolve_sources(p, e, st) && ok;
    if (!ok) return;   // fault latched; nothing in flight yet
    __shared__ float s_vnew[K];
    if constexpr (MODE == 5) {
        if (!gt_weights(p, e, st, s_vnew)) return;
    }

    // ---- split every agent's sources into the local block and the remote list ----
    if (threadIdx.x == 0) {
        unsigned procs = 0;
        int nr = 0;
        for (int a = 0; a < K; ++a) {
            for (int b = 0; b < K; ++b) lm.c[a][b] = 0.f;
            lm.c[a][a] = st.self_w[a];
            lm.rbeg[a] = nr;
            for (int q = 0; q < st.nsrc[a]; ++q) {
                const int src = st.src[a][q];
                if (src / K == g.me) {
                    lm.c[a][src % K] += st.coef[a][q];
                } else {
                    lm.rs[nr] = static_cast<unsigned char>(src);
                    lm.rc[nr] = st.coef[a][q];
                    procs |= 1u << (src / K);
                    ++nr;
                }
            }
        }
        lm.rbeg[K] = nr;
        lm.procs = procs;
        unsigned pub = 0;
        if (g.nprocs > 1) {
            if (p.wmode == kWStatic) {
                pub = p.pub_mask;
            } else if (p.wmode == kWSchedule) {   // agent a pushes to its scheduled dst (R5, R27)
                const unsigned long long round = *reinterpret_cast<volatile unsigned long long *>(&pad->round);
                for (int a = 0; a < K; ++a) {
                    int src, dst;
                    sched_peers(p.sched_kind, g.n, p.sched_L, round, g.me * K + a, src, dst);
                    if (dst >= 0 && dst / K != g.me) pub |= 1u << a;
                }
            } else {
                pub = (1u << K) - 1u;   // pull-only readers are not known to the sender
            }
        }
        lm.pub = pub;
    }
    __syncthreads();
    BF_STAT(if (stat && threadIdx.x == 0) stat[7] = globaltimer() - t_k0;)

    const bool vec = g.vec_ok != 0;
    const long long count = g.count;
    const int G = gridDim.x;
    const int S = static_cast<int>((count + kSubT - 1) / kSubT);
    const int nmine = static_cast<int>(blockIdx.x) < S ? (S - static_cast<int>(blockIdx.x) + G - 1) / G : 0;
    const int nrt = lm.rbeg[K];   // remote tiles per sub-item
    auto slot_of = [&](int agent) {
        return at<WT>(g.peer_base[agent / K],
                      p.slot_off + (agent % K) * p.slot_agent_stride + parity * p.slot_parity_stride);
    };
    // One process (HBM-bound): odd epochs walk the sub-items backwards, so a step starts
    // on the lines the previous step wrote last -- still in the 126 MB L2 -- instead of
    // the ones it wrote first (BF_REVERSE=0 at build time keeps the forward walk).  Only the
    // in-place updates (ATC, AWC, ED, GT): neighbor_allreduce writes y, not the x the next call
    // reads, and walked backwards it measured slower (hierarchical 4x2 0.271 -> 0.283 ms;
    // ATC 0.410 -> 0.398 ms with it, profiles/r02c_fused_reverse_ab_n1.txt)
    const bool reverse = BF_REVERSE && MODE != 0 && (g.nprocs == 1 || BF_REVERSE_X) && (e & 1);
    auto sub = [&](int m) {
        const int s = static_cast<int>(blockIdx.x) + m * G;
        return reverse ? S - 1 - s : s;
    };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == kThreads / 32 + 1) {
        // ================ signal warp (lane 0): system-scope releases ================
        const int nbatch = lm.pub ? (nmine + kBatch - 1) / kBatch : 0;
        if (FusedCfg<K>::kRing && lane == 0 && nbatch > 0) {
            unsigned long long *prog = at<unsigned long long>(g.peer_base[g.me], p.prog_off) + blockIdx.x;
            volatile int *released = &s_released;
            for (int rb = 0; rb < nbatch; ++rb) {
                if (!mbar_wait_acq_b(g, &pubbar[rb % kPubRing], static_cast<unsigned>(rb / kPubRing) & 1u, fail)) break;
                const int done = min((rb + 1) * kBatch, nmine);
                BF_STAT(const unsigned long long tf = globaltimer();)
                fence_acq_rel(true);   // the consumers' slot stores, visible system-wide ...
                BF_STAT(if (stat) { stat[4] += globaltimer() - tf; stat[5] += 1; })
                st_relaxed(prog, (e << kProgShift) | static_cast<unsigned long long>(done), true);   // ... first
                *released = rb + 1;
            }
        }
    } else if (warp == kThreads / 32) {
        // ============ producer warp (lane 0): TMA pulls of the remote tiles ============
        if (FusedCfg<K>::kRing && lane == 0 && nrt > 0) {
            long long issued = 0;              // ring entries issued
            const long long total = static_cast<long long>(nmine) * nrt;
            unsigned long long seen[kMaxP];    // last acquired progress of each source process
            for (int q = 0; q < kMaxP; ++q) seen[q] = 0;
            unsigned long long t_idle = globaltimer();
            BF_STAT(unsigned long long t_mark = t_idle;)
            unsigned it = 0;
            while (issued < total && !*fail) {
                bool progressed = false;
                // pull the remote tiles of the next sub-items while ring slots are free
                BF_STAT(int why = 0;)   // 1: blocked on a ring slot, 2: blocked on a peer's progress
                while (issued < total) {
                    const int m = static_cast<int>(issued / nrt), i = static_cast<int>(issued % nrt);
                    const int sl = static_cast<int>(issued % kNSlot);
                    if (issued >= kNSlot && !mbar_test(&empty[sl], static_cast<unsigned>(issued / kNSlot - 1) & 1u)) {
                        BF_STAT(why = 1;)
                        break;   // slot still being read
                    }
                    if (i == 0) {   // a new sub-item: every source process must have published it
                        const unsigned long long need = (e << kProgShift) | static_cast<unsigned long long>(m + 1);
                        bool ready = true, acquired = false;
                        for (int q = 0; q < g.nprocs && ready; ++q) {
                            if (!((lm.procs >> q) & 1u) || seen[q] >= need) continue;
                            seen[q] = ld_acquire_sys(at<unsigned long long>(g.peer_base[q], p.prog_off) + blockIdx.x);
                            ready = seen[q] >= need;
                            acquired = true;
                            BF_STAT(if (stat) stat[6] += 1;)
                        }
                        if (acquired) fence_proxy_async_global();   // acquire before the async-proxy reads
                        if (!ready) {
                            BF_STAT(why = 2;)
                            break;
                        }
                    }
                    const long long base = static_cast<long long>(sub(m)) * kSubT;
                    const long long left = count - base;
                    const unsigned bytes =
                        (static_cast<unsigned>((left < kSubT ? left : kSubT) * sizeof(WT)) + 15u) & ~15u;
                    mbar_expect_tx(&full[sl], bytes);
                    tma_load_1d(ring + sl * kSlotBytes, slot_of(lm.rs[i]) + base, bytes, &full[sl]);
                    ++issued;
                    progressed = true;
                }
                BF_STAT(const unsigned long long now = globaltimer();
                        if (stat && !progressed && why) stat[why == 1 ? 3 : 2] += now - t_mark;
                        t_mark = now;)
                if (progressed) {
                    t_idle = globaltimer();
                } else {   // nothing to do right now: bounded idle
                    if ((++it & 63u) == 0) {
                        const unsigned code = ld_relaxed_sys_u32(&pad->abort);
                        if (code) {
                            if (g.host_err) *g.host_err = code;
                            *fail = 1;
                        } else if (globaltimer() - t_idle > g.timeout_ns) {
                            abort_all(g, BF_ERR_TIMEOUT);
                            *fail = 1;
                        }
                    }
                    __nanosleep(32);
                }
            }
            // drain: no bulk copy may be in flight when the CTA exits
            volatile int no_fail = 0;
            for (long long i = issued > kNSlot ? issued - kNSlot : 0; i < issued; ++i)
                mbar_wait_b(g, &full[i % kNSlot], static_cast<unsigned>(i / kNSlot) & 1u, &no_fail);
        }
    } else {
        // ============================ consumer warps ============================
        const unsigned pub = lm.pub;
        const unsigned long long pol_stream = policy_evict_first();
        const unsigned long long pol_keep = policy_evict_normal();
        // fp32-wire neighbor_allreduce / ATC: an agent another process reads takes its x_half
        // in the combine back from its own slot (stored kLead sub-items earlier by this thread,
        // bit-identical, 4 B and often still in L2) instead of re-reading x and g (8 B)
        constexpr bool SLOTX = (MODE == 0 || MODE == 1) && std::is_same<XT, float>::value &&
                               std::is_same<WT, float>::value && FusedCfg<K>::kRing;
        const unsigned long long pol_pub = BF_SLOTX_PUB_STREAM && SLOTX ? pol_stream : pol_keep;   // x / g of the publish
        auto xrow = [&](int a) { return static_cast<const XT *>(p.x) + static_cast<long long>(a) * count; };
        auto grow = [&](int a) { return static_cast<const GT *>(p.g) + static_cast<long long>(a) * count; };
        unsigned long long *prog = at<unsigned long long>(g.peer_base[g.me], p.prog_off) + blockIdx.x;
        // batch b published: every consumer thread arrives with release semantics after its
        // own slot stores; the signal warp acquires the completed phase and turns it into the
        // system-scope release (fence.acq_rel.sys is cumulative over what it acquired)
        auto batch_done = [&](int b) {
            if (b >= kPubRing) {   // the ring slot's previous phase must have been released
                volatile int *released = &s_released;
                while (*released <= b - kPubRing && !*fail) __nanosleep(64);
            }
            mbar_arrive_release(&pubbar[b % kPubRing]);
        };
        if (sys && pub == 0 && threadIdx.x == 0)   // nothing of this process is read remotely
            st_relaxed(prog, (e << kProgShift) | static_cast<unsigned long long>(nmine), true);

        long long consumed = 0;   // remote ring entries consumed
        int mp = 0, mc = 0;
        while (mc < nmine) {
            if (FusedCfg<K>::kRing && pub && mp < nmine && mp <= mc + kLead) {
                // ---- publish sub-item mp for the agents with remote readers ----
                const long long base = static_cast<long long>(sub(mp)) * kSubT;
                const int e0 = threadIdx.x * V;
                const int valid = clamp_valid_v<V>(count - base, e0);
#pragma unroll
                for (int a = 0; a < K; ++a) {
                    if (!((pub >> a) & 1u)) continue;
                    float v[V];
                    VecN<XT, V>::load_hint(xrow(a) + base + e0, v, valid, vec, pol_pub);
                    if constexpr (MODE == 1 || MODE == 5) {
                        float gv[V];
                        VecN<GT, V>::load_hint(grow(a) + base + e0, gv, valid, vec, pol_pub);
#pragma unroll
                        for (int i = 0; i < V; ++i) v[i] = fmaf(-p.lr, gv[i], v[i]);
                    }
                    if constexpr (MODE == 4) {   // GT y-step: y + g - g_prev
                        float gv[V], hv[V];
                        VecN<GT, V>::load_hint(grow(a) + base + e0, gv, valid, vec, pol_keep);
                        VecN<float, V>::load_hint(p.g2 + static_cast<long long>(a) * count + base + e0, hv, valid, vec,
                                                  pol_keep);
#pragma unroll
                        for (int i = 0; i < V; ++i) v[i] = (v[i] + gv[i]) - hv[i];
                    }
                    if constexpr (MODE == 3) {   // Exact-Diffusion: phi = (x - lr g) + x - psi_prev
                        float gv[V], pv[V];
                        VecN<GT, V>::load_hint(grow(a) + base + e0, gv, valid, vec, pol_keep);
                        VecN<float, V>::load_hint(p.psi + static_cast<long long>(a) * count + base + e0, pv, valid,
                                                  vec, pol_keep);
#pragma unroll
                        for (int i = 0; i < V; ++i) v[i] = (fmaf(-p.lr, gv[i], v[i]) + v[i]) - pv[i];
                    }
                    VecN<WT, V>::store_hint(slot_of(g.me * K + a) + base + e0, v, valid, true, pol_keep);
                }
                ++mp;
                if (mp % kBatch == 0 || mp == nmine) batch_done((mp - 1) / kBatch);
                continue;
            }
            // ---- combine sub-items mc .. mc + U - 1 ----
            const int nu = min(U, nmine - mc);
            const int e0 = threadIdx.x * V;
            float xv[U][K][V];
            float gv[U][HAS_G ? K : 1][V];
            {
                // every local load of the group is issued (raw) before the first use
                typename VecN<XT, V>::Raw xr[U][K];
                typename VecN<GT, V>::Raw gr[U][HAS_G ? K : 1];
                // third stream: Exact-Diffusion psi^(k-1) (MODE 3), gradient tracking g^(k) (MODE 4)
                constexpr bool THIRD = MODE == 3 || MODE == 4;
                const float *third = MODE == 3 ? p.psi : p.g2;
                typename VecN<float, THIRD ? V : 4>::Raw pr[U][THIRD ? K : 1];
                // one branch per group: the common case is a straight line of vector loads
                bool fast = vec;
#pragma unroll
                for (int u = 0; u < U; ++u)
                    fast = fast && u < nu && clamp_valid_v<V>(count - static_cast<long long>(sub(mc + u)) * kSubT, e0) == V;
                if (fast) {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const long long base = static_cast<long long>(sub(mc + u)) * kSubT + e0;
#pragma unroll
                        for (int a = 0; a < K; ++a) {
                            const XT *src = xrow(a) + base;
                            if constexpr (SLOTX)
                                if ((pub >> a) & 1u) src = reinterpret_cast<const XT *>(slot_of(g.me * K + a)) + base;
                            VecN<XT, V>::load_raw_fast(src, xr[u][a], pol_stream);
                        }
                        if constexpr (HAS_G) {
#pragma unroll
                            for (int a = 0; a < K; ++a) {
                                if (SLOTX && ((pub >> a) & 1u)) {
                                    gr[u][a] = typename VecN<GT, V>::Raw{};
                                    continue;
                                }
                                VecN<GT, V>::load_raw_fast(grow(a) + base, gr[u][a], pol_stream);
                            }
                        }
                        if constexpr (THIRD) {
#pragma unroll
                            for (int a = 0; a < K; ++a)
                                VecN<float, V>::load_raw_fast(third + static_cast<long long>(a) * count + base, pr[u][a],
                                                              pol_stream);
                        }
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        // a slot of the group past the end (u >= nu) runs with valid = 0: no memory access
                        const long long base = static_cast<long long>(sub(mc + u)) * kSubT;
                        const int valid = u < nu ? clamp_valid_v<V>(count - base, e0) : 0;
#pragma unroll
                        for (int a = 0; a < K; ++a) {
                            const XT *src = xrow(a) + base + e0;
                            if constexpr (SLOTX)
                                if ((pub >> a) & 1u) src = reinterpret_cast<const XT *>(slot_of(g.me * K + a)) + base + e0;
                            VecN<XT, V>::load_raw(src, xr[u][a], valid, pol_stream);
                        }
                        if constexpr (HAS_G) {
#pragma unroll
                            for (int a = 0; a < K; ++a) {
                                if (SLOTX && ((pub >> a) & 1u)) {
                                    gr[u][a] = typename VecN<GT, V>::Raw{};
                                    continue;
                                }
                                VecN<GT, V>::load_raw(grow(a) + base + e0, gr[u][a], valid, pol_stream);
                            }
                        }
                        if constexpr (THIRD) {
#pragma unroll
                            for (int a = 0; a < K; ++a)
                                VecN<float, V>::load_raw(third + static_cast<long long>(a) * count + base + e0, pr[u][a],
                                                         valid, pol_stream);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int a = 0; a < K; ++a) {
                        VecN<XT, V>::unpack(xr[u][a], xv[u][a]);
                        if constexpr (HAS_G) VecN<GT, V>::unpack(gr[u][a], gv[u][a]);
                        if constexpr (MODE == 4) {   // GT y-step: y + g - g_prev
                            float hv[V];
                            VecN<float, V>::unpack(pr[u][a], hv);
#pragma unroll
                            for (int i = 0; i < V; ++i) xv[u][a][i] = (xv[u][a][i] + gv[u][a][i]) - hv[i];
                        }
                        if constexpr (MODE == 3) {   // psi_prev kept in gv's place after use below
                            float pv[V];
                            VecN<float, V>::unpack(pr[u][a], pv);
                            // psi = x - lr g (ed-1, the new state); phi = psi + x - psi_prev (ed-2)
#pragma unroll
                            for (int i = 0; i < V; ++i) {
                                const float psi = fmaf(-p.lr, gv[u][a][i], xv[u][a][i]);
                                gv[u][a][i] = psi;
                                xv[u][a][i] = (psi + xv[u][a][i]) - pv[i];
                            }
                        }
                    }
            }
            for (int u = 0; u < nu; ++u) {
                const long long base = static_cast<long long>(sub(mc + u)) * kSubT;
                const int valid = clamp_valid_v<V>(count - base, e0);
                if constexpr (MODE == 1 || MODE == 5) {
#pragma unroll
                    for (int a = 0; a < K; ++a) {
                        if (SLOTX && ((pub >> a) & 1u)) continue;   // read back adapted from the slot
#pragma unroll
                        for (int i = 0; i < V; ++i) xv[u][a][i] = fmaf(-p.lr, gv[u][a][i], xv[u][a][i]);   // Eq. 4
                    }
                }
                if constexpr (MODE == 3) {   // store psi^(k) over psi^(k-1) (same elements, same thread)
#pragma unroll
                    for (int a = 0; a < K; ++a)
                        VecN<float, V>::store_hint(p.psi + static_cast<long long>(a) * count + base + e0, gv[u][a], valid,
                                                   vec, pol_stream);
                }
#pragma unroll
                for (int a = 0; a < K; ++a) {
                    float acc[V];
                    const float cs = lm.c[a][a];
#pragma unroll
                    for (int i = 0; i < V; ++i) acc[i] = cs * xv[u][a][i];
#pragma unroll
                    for (int d = 1; d < K; ++d) {
                        const int b = (a + K - d) % K;
                        const float c = lm.c[a][b];
                        if (c != 0.f) {
#pragma unroll
                            for (int i = 0; i < V; ++i)   // MODE 0: x is already a wire value
                                acc[i] = fmaf(c, MODE == 0 ? xv[u][b][i] : VecN<WT, V>::wire(xv[u][b][i]), acc[i]);
                        }
                    }
                    if constexpr (FusedCfg<K>::kRing) {
                        for (int i = lm.rbeg[a]; i < lm.rbeg[a + 1]; ++i) {   // remote sources from the TMA ring
                            const long long idx = consumed + i;
                            const int sl = static_cast<int>(idx % kNSlot);
                            BF_STAT(const unsigned long long tw = globaltimer();)
                            mbar_wait_b(g, &full[sl], static_cast<unsigned>(idx / kNSlot) & 1u, fail);
                            BF_STAT(if (stat && threadIdx.x == 0) stat[1] += globaltimer() - tw;)
                            float v[V];
                            VecN<WT, V>::load(reinterpret_cast<const WT *>(ring + sl * kSlotBytes) + e0, v, valid, true);
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&empty[sl]);
                            const float c = lm.rc[i];
#pragma unroll
                            for (int j = 0; j < V; ++j) acc[j] = fmaf(c, v[j], acc[j]);
                        }
                    }
                    if constexpr (MODE == 2) {   // AWC (Eq. 16)
#pragma unroll
                        for (int i = 0; i < V; ++i) acc[i] = fmaf(-p.lr, gv[u][a][i], acc[i]);
                    }
                    YT *yr = static_cast<YT *>(p.y) + static_cast<long long>(a) * count + base + e0;
                    VecN<YT, V>::store_hint(yr, acc, valid, vec, pol_stream);
                    if (p.shadow) {
                        bf16 *sr = static_cast<bf16 *>(p.shadow) + static_cast<long long>(a) * count + base + e0;
                        VecN<bf16, V>::store_hint(sr, acc, valid, vec, pol_stream);
                    }
                    if constexpr (MODE == 5) {   // x = u / v (appendix)
                        const float vn = s_vnew[a];
#pragma unroll
                        for (int i = 0; i < V; ++i) acc[i] = acc[i] / vn;
                        VecN<float, V>::store_hint(p.x_out + static_cast<long long>(a) * count + base + e0, acc, valid,
                                                   vec, pol_stream);
                    }
                }
                consumed += nrt;
            }
            mc += nu;
        }
    }
    __syncthreads();
    BF_STAT(if (stat && threadIdx.x == 0) stat[0] = globaltimer() - t_k0;)
    if (*fail) return;   // nothing is in flight any more; the fault is latched
    last_cta(pad, [&] {
        if constexpr (MODE == 5)
            for (int a = 0; a < K; ++a) p.gt_v[a] = s_vnew[a];
        pad->epoch = e;
        if (p.wmode == kWSchedule) pad->round = pad->round + 1;
        publish_done(g, e);
    });
}

template <typename XT, typename GT, typename WT, typename YT, int MODE, int K>
static cudaError_t launch_fused_k(const ExchParams &p, int grid, cudaStream_t s) {
    const void *fn = reinterpret_cast<const void *>(exchange_fused_kernel<XT, GT, WT, YT, MODE, K>);
    // the remote-tile ring is only needed when other processes exist
    const bool ringed = FusedCfg<K>::kRing && p.geo.nprocs > 1;
    if (!FusedCfg<K>::kRing && p.geo.nprocs > 1) return cudaErrorInvalidValue;
    constexpr int kSubT = kThreads * FusedVec<XT>::V;
    const unsigned smem = ringed ? kRingBytes : 0;
    static int maxg[2] = {0, 0};   // co-resident CTAs of this instantiation (queried once per smem size)
    if (maxg[ringed] == 0) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kRingBytes);
        if (e != cudaSuccess) return e;
        maxg[ringed] = max_coresident(fn, FusedCfg<K>::kThreadsPerCta, smem);
    }
    const long long subs = (p.geo.count + kSubT - 1) / kSubT;
    static const int grid_env = getenv("BF_FUSED_GRID") ? atoi(getenv("BF_FUSED_GRID")) : 0;   // tuning
    if (grid <= 0 && grid_env > 0) grid = grid_env;
    if (grid <= 0 || grid > maxg[ringed]) grid = maxg[ringed];
    // across GPUs: 2 CTAs per SM (measured at K = 1: 444 CTAs 0.272 ms, 296 CTAs 0.227 ms,
    // 222 CTAs 0.255 ms per C4-sized step -- more CTAs only add pairwise synchronisation)
    if (ringed && grid_env <= 0) {
        static int two_per_sm = 0;
        if (two_per_sm == 0) {
            int dev = 0, sms = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            two_per_sm = 2 * sms;
        }
        if (grid > two_per_sm) grid = two_per_sm;
    }
    if (grid > subs) grid = static_cast<int>(subs);
    if (grid > kMaxGrid) grid = kMaxGrid;
    if (grid < 1) grid = 1;
    void *args[] = {const_cast<ExchParams *>(&p)};
    // one process: no CTA of the launch ever waits for another, so a plain launch
    // (lower launch latency) is enough; across processes CTA b waits for CTA b of
    // the peers, so every CTA must be resident: cooperative launch
    if (p.geo.nprocs == 1)
        return cudaLaunchKernel(fn, dim3(grid), dim3(FusedCfg<K>::kThreadsPerCta), args, smem, s);
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(FusedCfg<K>::kThreadsPerCta), args, smem, s);
}

}  // namespace bf

#include "exchange_push.cuh"
#include "exchange_ll.cuh"

namespace bf {

template <typename XT, typename GT, typename WT, typename YT, int MODE>
static cudaError_t launch_fused_t(const ExchParams &p, int grid, cudaStream_t s) {
    if (p.ll) {
        switch (p.geo.k) {
            case 1: return launch_ll_k<XT, GT, WT, YT, MODE, 1>(p, s);
            case 2: return launch_ll_k<XT, GT, WT, YT, MODE, 2>(p, s);
            case 4: return launch_ll_k<XT, GT, WT, YT, MODE, 4>(p, s);
            default: return cudaErrorInvalidValue;
        }
    }
    switch (p.geo.k) {
        case 1: return p.push ? launch_push_k<XT, GT, WT, YT, MODE, 1>(p, grid, s)
                              : launch_fused_k<XT, GT, WT, YT, MODE, 1>(p, grid, s);
        case 2: return p.push ? launch_push_k<XT, GT, WT, YT, MODE, 2>(p, grid, s)
                              : launch_fused_k<XT, GT, WT, YT, MODE, 2>(p, grid, s);
        case 4: return p.push ? launch_push_k<XT, GT, WT, YT, MODE, 4>(p, grid, s)
                              : launch_fused_k<XT, GT, WT, YT, MODE, 4>(p, grid, s);
        case 8: return launch_fused_k<XT, GT, WT, YT, MODE, 8>(p, grid, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace bf
