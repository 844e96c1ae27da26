// exchange_push.cuh -- the cross-GPU PUSH variant of the local-agent fused kernel
// (kernel 3 with ExchParams::push), for processes hosting K = 1 or 2 agents (the
// 8-GPU shape of the paper, one agent per GPU, and 8 agents over 4 GPUs).
//
// The pull kernel (exchange_fused.cuh) publishes every wire copy into the
// writer's own HBM and the reader pulls it over NVLink after acquiring the
// writer's progress word across NVLink: the two GPUs' CTAs pace each other
// through ~5 us system-scope round trips, and the writer reads x and g twice
// (once to publish kLead sub-items ahead, once to combine).  Here:
//   * the WRITER stores wire(x_half) straight into each reader process's inbox
//     (remote NVLink stores, posted: no round trip on the data path) and, per
//     batch of sub-items, releases a progress word that lives in the READER's
//     heap (pflag[writer process][CTA]);
//   * the READER polls its own local memory for the progress word and reads the
//     inbox tiles from its local HBM / L2 (the NVLink writes land in its L2);
//   * each sub-item is read from HBM once: the local part of every combine
//     (self term, same-process sources, AWC / ED terms) is formed while the
//     sub-item is published and parked in shared memory for kLag sub-items, until
//     the remote tiles of that sub-item have arrived, then the remote terms are
//     added and y is stored.
// HBM per agent-element at K = 1 (fp32 ATC): x + g read, y write, inbox landing
// write + read (often an L2 hit) = 16-20 B, against 28 B for the pull kernel.
// Same pairwise CTA pairing as the pull kernel (sub-item s -> CTA s mod G on every
// process), same WAR protection of the double-buffered inbox (done_from), same
// summation order (R18: self, same-process sources in (a - b) mod K order, remote
// sources in table order), so results are bitwise those of the pull kernel --
// except AWC, whose -lr g_a joins the parked local part before the remote terms.
// Static and scheduled topologies only (a push needs the writer to know its
// readers; pull-only per-call views keep the pull kernel).
//
// Hierarchical modes (R12; caption P:869) when every machine lies inside
// one process (machine size L divides agents_per_proc): a "machine agent" is a
// whole machine, K = machines per process, and each sub-item of machine agent a
// reads its L rows a*L + l:
//   MODE 6: hierarchical neighbor_allreduce  y_row = sum_m' W_M[m][m'] mean(x of m')
//   MODE 7: H-ATC  the mean of fp32(x - lr g) over the machine's rows (Eq. 17)
//   MODE 8: H-AWC  y_row = sum_m' W_M[m][m'] mean(x of m') - lr g_row (Eq. 16)
// The machine average crosses NVLink once per reader process; the broadcast back
// to the L rows is the store of the combine.
#pragma once

namespace bf {

#ifndef BF_PUSH_SMEM_KB
#define BF_PUSH_SMEM_KB 96
#endif
#ifndef BF_PUSH_LAG
#define BF_PUSH_LAG 16
#endif
#ifndef BF_PUSH_BATCH
#define BF_PUSH_BATCH 4
#endif
// signal warps: a system-scope release fence waits for every store the SM issued
// before it -- BF_STATS measured ~14 us per fence at K = 1 with NVLink stores in
// flight, so one warp fencing batch after batch paces the whole exchange (fence
// time ~ 90% of the kernel).  NSIG warps fence different batches concurrently
// (batch rb -> warp rb mod NSIG): the latency stays, the throughput of releases
// scales; progress words are raised with a remote atomic max, so a later batch's
// release overtaking an earlier one never moves a word backwards.
// (measured at N = 2: K = 1 one-peer 0.233 ms with one signal warp, 0.201 with 4,
// 0.193-0.195 with 8; K = 2 is best with 4 -- 8 more warps cost it registers)
#ifndef BF_PUSH_REVERSE
#define BF_PUSH_REVERSE 1
#endif
#ifndef BF_PUSH_PREFETCH
#define BF_PUSH_PREFETCH 1   // K >= 4: issue sub-item m's x / g loads before the combine of sub-item m - kLag
#endif
#ifndef BF_PUSH_PREFETCH_MINK
#define BF_PUSH_PREFETCH_MINK 2   // smallest K with the prefetch (K = 2 one-peer: 0.294 -> 0.286 ms at N = 2; K = 1 slower)
#endif
#ifndef BF_PUSH_PREFETCH_GT5
#define BF_PUSH_PREFETCH_GT5 0   // 1: the prefetch also for the GT u/v-step (two streams, like ATC)
#endif
#ifndef BF_PUSH_K4_MINB
#define BF_PUSH_K4_MINB 2   // CTAs per SM of the K = 4 push kernel (1: 192 KB lag, 4 signal warps;
                            // measured N = 2 exp-2: 2 per SM 0.72 ms, 1 per SM 0.78 ms)
#endif
#ifndef BF_PUSH_NSIG
#define BF_PUSH_NSIG 0   // 0: 8 for K = 1, 4 for K = 2
#endif

template <int K, int V>
struct PushCfg {
    // K <= 2: 2 CTAs per SM, 96 KB each; K = 4 holds 4 agents' partial combines per
    // sub-item: 1 CTA per SM with 192 KB (a deeper lag, and no register cap of 2 CTAs)
    static constexpr int kMinB = K >= 4 ? BF_PUSH_K4_MINB : 2;
    static constexpr int kSmemKB = K >= 4 && BF_PUSH_K4_MINB == 1 ? 2 * BF_PUSH_SMEM_KB : BF_PUSH_SMEM_KB;
    // sub-items between the publish of a sub-item and its combine: as many as the
    // shared-memory budget holds (K agents x V floats per thread per sub-item)
    static constexpr int kPerSub = K * kThreads * V * 4;
    static constexpr int kByBytes = kSmemKB * 1024 / kPerSub;
    static constexpr int kLag = kByBytes < BF_PUSH_LAG ? (kByBytes < 2 ? 2 : kByBytes) : BF_PUSH_LAG;
    static constexpr int kSmem = kLag * kPerSub;
    static constexpr int kSig = BF_PUSH_NSIG > 0 ? BF_PUSH_NSIG : (K == 1 ? 8 : (K >= 4 && kMinB == 2 ? 2 : 4));
    static constexpr int kThreadsPerCta = kThreads + 32 * (1 + kSig);   // consumers + poll + signal warps
    // sub-items per progress release.  Deadlock freedom: the combine of sub-item m - kLag
    // runs before sub-item m is pushed, and needs the peer's batch holding m - kLag released,
    // i.e. pushed up to its end -- so a batch may not span more than kLag sub-items
    // (bf16 at K = 4: kLag = 3 -> batches of 3)
    static constexpr int kBatch = BF_PUSH_BATCH < kLag ? BF_PUSH_BATCH : kLag;
    static_assert(kPubRing % kSig == 0, "a publish-barrier slot must always map to the same signal warp");
    static_assert(kBatch >= 1 && kBatch <= kLag, "a batch must fit in the lag");
};
#ifndef BF_PUSH_FIRST
#define BF_PUSH_FIRST 0   // 1: the first batch is a single sub-item (an early first release)
#endif
// batches of B sub-items: with BF_PUSH_FIRST, batch 0 = sub-item 0, batch b >= 1 = sub-items
// 1 + (b-1)B .. bB; else batch b = sub-items bB .. (b+1)B - 1
template <int B>
__device__ __forceinline__ int push_nbatch(int nmine) {
    return BF_PUSH_FIRST ? (nmine > 0 ? 1 + (nmine - 1 + B - 1) / B : 0) : (nmine + B - 1) / B;
}
template <int B>
__device__ __forceinline__ int push_batch_end(int b, int nmine) {   // sub-items covered by batches 0..b
    return min(BF_PUSH_FIRST ? 1 + b * B : (b + 1) * B, nmine);
}
template <int B>
__device__ __forceinline__ int push_batch_of(int m) {
    return BF_PUSH_FIRST ? (m == 0 ? 0 : 1 + (m - 1) / B) : m / B;
}

__device__ __forceinline__ void red_max_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("red.relaxed.sys.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int K>
struct PushMix {
    float c[K][K];                 // local block of W (registers)
    float rc[K * kMaxN];           // remote sources, agent-major: weight ...
    unsigned char rs[K * kMaxN];   // ... and global source agent
    int rbeg[K + 1];
    unsigned procs_in;             // processes hosting a remote source of a local agent
    unsigned procs_out[K];         // per local agent: processes it pushes to
    unsigned procs_out_all;
};

__device__ __forceinline__ unsigned ld_acquire_cta_shared(const int *p) {
    unsigned v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta_shared(int *p, int v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

template <typename XT, typename GT, typename WT, typename YT, int MODE, int K>
__global__ void __launch_bounds__(PushCfg<K, FusedVec<XT>::V>::kThreadsPerCta, PushCfg<K, FusedVec<XT>::V>::kMinB)
    exchange_push_kernel(const __grid_constant__ ExchParams p) {
    constexpr bool HAS_G = MODE != 0 && MODE != 6;
    constexpr bool HIER = MODE >= 6;
    constexpr int V = FusedVec<XT>::V;
    constexpr int kSubT = kThreads * V;
    constexpr int L = PushCfg<K, V>::kLag;
    constexpr int kPushSig = PushCfg<K, V>::kSig;
    constexpr int B = PushCfg<K, V>::kBatch;
    extern __shared__ __align__(16) float lag[];   // [L][K][kThreads][V]: partial combines, thread-private
    __shared__ SharedTab st;
    __shared__ PushMix<K> lm;
    __shared__ __align__(8) unsigned long long pubbar[kPubRing];
    __shared__ int s_fail, s_ready;
    __shared__ int s_rel[kPubRing];   // last batch whose publish barrier phase a signal warp has consumed
    volatile int *const fail = &s_fail;
    const Geometry &g = p.geo;
    Pad *pad = pad_of(g, g.me);
    if (aborted(g)) return;
    // BF_STATS (diagnostic build): 0 kernel ns, 1 consumer ns waiting for remote tiles,
    // 2 ns until the first remote batch was seen, 3 ns until the consumer loop ended,
    // 4 release-fence ns, 5 fences, 6 progress polls, 7 prologue ns
    BF_STAT(const unsigned long long t_k0 = globaltimer();)
    BF_STAT(unsigned long long *const stat = p.stats ? p.stats + blockIdx.x * 8 : nullptr;)
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long *>(&pad->epoch) + 1;
    const int parity = static_cast<int>(e & 1);
    if (threadIdx.x == 0) {
        s_fail = 0;
        s_ready = 0;
        for (int i = 0; i < kPubRing; ++i) s_rel[i] = i - kPubRing;
        for (int i = 0; i < kPubRing; ++i) mbar_init(&pubbar[i], kThreads);
        fence_mbar_init();
    }
    bool ok = war_wait(g, e);
    ok = resolve_sources(p, e, st) && ok;
    if (!ok) return;
    __shared__ float s_vnew[K];
    if constexpr (MODE == 5) {
        if (!gt_weights(p, e, st, s_vnew)) return;
    }

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
        lm.procs_in = procs;
        unsigned all = 0;
        for (int a = 0; a < K; ++a) {
            unsigned out = 0;
            if (p.wmode == kWStatic) {
                out = p.pushq[a];
            } else {   // kWSchedule: the scheduled destination (R5, R27)
                const unsigned long long round = *reinterpret_cast<volatile unsigned long long *>(&pad->round);
                int src, dst;
                sched_peers(p.sched_kind, g.n, p.sched_L, round, g.me * K + a, src, dst);
                if (dst >= 0 && dst / K != g.me) out = 1u << (dst / K);
            }
            lm.procs_out[a] = out;
            all |= out;
        }
        lm.procs_out_all = all;
    }
    __syncthreads();
    BF_STAT(if (stat && threadIdx.x == 0) stat[7] = globaltimer() - t_k0;)

    const bool vec = g.vec_ok != 0;
    const long long count = g.count;
    const int G = gridDim.x;
    const int S = static_cast<int>((count + kSubT - 1) / kSubT);
    const int nmine = static_cast<int>(blockIdx.x) < S ? (S - static_cast<int>(blockIdx.x) + G - 1) / G : 0;
    const int nrt = lm.rbeg[K];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // odd epochs walk the sub-items backwards on every process (the pairing of CTA b with
    // the peers' CTA b is unchanged): a step starts on the lines the previous one left in L2
    // (measured at N = 4: K = 2 exp-2 0.680 -> 0.660 ms; K = 1 one-peer 0.187 -> 0.191 ms; at N = 2
    // K = 4 it costs: exp-2 0.71 -> 0.80 ms, profiles/r02_push_k4_knobs_n2.txt -- so K = 2 only)
    // ATC only: Exact-Diffusion walked backwards at K = 2 measured 0.81 ms against 0.37 ms
    // forward (N = 2, profiles/r02c_ed_ab_n2.txt)
    const bool reverse = BF_PUSH_REVERSE && K == 2 && MODE == 1 && (e & 1);
    auto sub = [&](int m) {
        const int s = static_cast<int>(blockIdx.x) + m * G;
        return reverse ? S - 1 - s : s;
    };
    // inbox of source agent j in process q's heap, this epoch's parity
    auto inbox = [&](int q, int j) {
        return at<WT>(g.peer_base[q], p.inbox_off + static_cast<unsigned long long>(j) * p.inbox_agent_stride +
                                          parity * p.inbox_parity_stride);
    };
    // progress word of writer process w for CTA b, in reader process q's heap
    auto pflag = [&](int q, int w) {
        return at<unsigned long long>(g.peer_base[q], p.pflag_off) + static_cast<long long>(w) * kMaxGrid + blockIdx.x;
    };

    if (warp >= kThreads / 32 + 1) {
        // ============ signal warps (lane 0): system-scope releases, batch rb -> warp rb mod NSIG ============
        const int sw = warp - (kThreads / 32 + 1);
        const int nbatch = lm.procs_out_all ? push_nbatch<B>(nmine) : 0;
        if (lane == 0) {
            volatile int *rel = s_rel;
            for (int rb = sw; rb < nbatch; rb += kPushSig) {
                if (!mbar_wait_acq_b(g, &pubbar[rb % kPubRing], static_cast<unsigned>(rb / kPubRing) & 1u, fail)) break;
                rel[rb % kPubRing] = rb;   // the barrier slot may take its next phase
                const int done = push_batch_end<B>(rb, nmine);
                BF_STAT(const unsigned long long tf = globaltimer();)
#ifndef BF_PUSH_NOFENCE   // diagnostic builds only (timing of the protocol without its fence; results may be stale)
                fence_acq_rel(true);   // the consumers' remote inbox stores, visible system-wide ...
#endif
                BF_STAT(if (stat) { atomicAdd(stat + 4, globaltimer() - tf); atomicAdd(stat + 5, 1ull); })
                for (int q = 0; q < g.nprocs; ++q)   // ... before the progress word in every reader's heap
                    if ((lm.procs_out_all >> q) & 1u)
                        red_max_sys(pflag(q, g.me), (e << kProgShift) | static_cast<unsigned long long>(done));
            }
        }
    } else if (warp == kThreads / 32) {
        // ===== poll warp (lane 0): local progress words of the writers -> s_ready =====
        if (lane == 0 && nrt > 0 && nmine > 0) {
            unsigned long long seen[kMaxP];
            for (int q = 0; q < kMaxP; ++q) seen[q] = 0;
            int ready = 0;
            unsigned long long t_idle = globaltimer();
            unsigned it = 0;
            while (ready < nmine && !*fail) {
                int lo = nmine;
                for (int q = 0; q < g.nprocs; ++q) {
                    if (!((lm.procs_in >> q) & 1u)) continue;
                    const unsigned long long need = (e << kProgShift) | static_cast<unsigned long long>(ready + 1);
                    if (seen[q] < need) {
                        seen[q] = ld_acquire_sys(pflag(g.me, q));
                        BF_STAT(if (stat) stat[6] += 1;)
                    }
                    const long long c = static_cast<long long>(seen[q]) - static_cast<long long>(e << kProgShift);
                    lo = min(lo, c <= 0 ? 0 : static_cast<int>(c));
                }
                if (lo > ready) {
                    BF_STAT(if (stat && ready == 0) stat[2] = globaltimer() - t_k0;)
                    ready = lo;
                    st_release_cta_shared(&s_ready, ready);
                    t_idle = globaltimer();
                } else {
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
                    __nanosleep(64);
                }
            }
        }
    } else {
        // ============================ consumer warps ============================
        const unsigned long long pol_stream = policy_evict_first();
        const XT *xbase = static_cast<const XT *>(p.x_alt && ((e - 1) & 1) ? p.x_alt : p.x);
        auto xrow = [&](int a) { return xbase + static_cast<long long>(a) * count; };
        auto grow = [&](int a) { return static_cast<const GT *>(p.g) + static_cast<long long>(a) * count; };
        const int HL = HIER ? p.hier_L : 1;   // rows written per (machine) agent
        const int HLin = HIER && p.hier_in ? p.hier_in : HL;   // rows averaged (1: x is the machine average)
        const float invL = 1.0f / static_cast<float>(HLin);
        const int e0 = threadIdx.x * V;
        float *mylag = lag + static_cast<long long>(threadIdx.x) * V;   // + (slot * K + a) * kSubT
        if (lm.procs_out_all == 0 && nrt == 0) {
            // nothing crosses processes for this process (e.g. a schedule round inside it)
        }
        int slot = 0;
        // non-hierarchical modes: the x / g loads of sub-item m are issued before the
        // combine of sub-item m - L, so their HBM latency overlaps the inbox reads
        // (measured at N = 2: K = 4 exp-2 0.715 -> 0.704 ms; K = 1 one-peer 0.183 -> 0.195 ms, so K >= 4 only)
        // (neighbor_allreduce / ATC / AWC only: Exact-Diffusion and the GT steps read a third
        // stream and were slower with it at K = 4 -- E 0.776 -> 0.96 ms, GT 1.47 -> 1.69 ms, N = 2)
        constexpr bool PREFETCH = !HIER && (MODE <= 2 || (BF_PUSH_PREFETCH_GT5 && MODE == 5)) && BF_PUSH_PREFETCH &&
                                  K >= BF_PUSH_PREFETCH_MINK;
        for (int m = 0; m < nmine + L; ++m, slot = slot + 1 == L ? 0 : slot + 1) {
            const int mc = m - L;
            typename VecN<XT, V>::Raw xraw[PREFETCH ? K : 1];
            typename VecN<GT, V>::Raw graw[PREFETCH && HAS_G ? K : 1];
            if constexpr (PREFETCH) {
                if (m < nmine) {
                    const long long base = static_cast<long long>(sub(m)) * kSubT;
                    const int valid = clamp_valid_v<V>(count - base, e0);
                    if (vec && valid == V) {
#pragma unroll
                        for (int a = 0; a < K; ++a) VecN<XT, V>::load_raw_fast(xrow(a) + base + e0, xraw[a], pol_stream);
                        if constexpr (HAS_G) {
#pragma unroll
                            for (int a = 0; a < K; ++a) VecN<GT, V>::load_raw_fast(grow(a) + base + e0, graw[a], pol_stream);
                        }
                    } else {
#pragma unroll
                        for (int a = 0; a < K; ++a) VecN<XT, V>::load_raw(xrow(a) + base + e0, xraw[a], valid, pol_stream);
                        if constexpr (HAS_G) {
#pragma unroll
                            for (int a = 0; a < K; ++a) VecN<GT, V>::load_raw(grow(a) + base + e0, graw[a], valid, pol_stream);
                        }
                    }
                }
            }
            // ---------------- combine sub-item mc: local part (smem) + remote tiles (inbox) ----------------
            if (mc >= 0) {
                const long long base = static_cast<long long>(sub(mc)) * kSubT;
                const int valid = clamp_valid_v<V>(count - base, e0);
                if (nrt > 0) {
                    if (static_cast<int>(ld_acquire_cta_shared(&s_ready)) <= mc) {
                        const unsigned long long t0 = globaltimer();
                        while (static_cast<int>(ld_acquire_cta_shared(&s_ready)) <= mc) {
                            if (*fail) break;
                            if (globaltimer() - t0 > g.timeout_ns + 1000000000ull) {   // the poll warp times out first
                                *fail = 1;
                                break;
                            }
                            __nanosleep(32);
                        }
                        BF_STAT(if (stat && threadIdx.x == 0) stat[1] += globaltimer() - t0;)
                    }
                    if (*fail) break;
                }
#pragma unroll
                for (int a = 0; a < K; ++a) {
                    float acc[V];
                    const float *lp = mylag + static_cast<long long>(slot * K + a) * kSubT;
#pragma unroll
                    for (int i = 0; i < V; i += 4) {
                        const float4 t = *reinterpret_cast<const float4 *>(lp + i);
                        acc[i] = t.x, acc[i + 1] = t.y, acc[i + 2] = t.z, acc[i + 3] = t.w;
                    }
                    // H-AWC at K >= 2: the first two g rows of the broadcast are loaded before the remote
                    // tiles (4x2 at N = 2: 0.595 -> 0.557 ms; K = 1, short of registers, got slower)
                    float g2[MODE == 8 ? 2 : 1][V];
                    auto load_g2 = [&](int l0) {
#pragma unroll
                        for (int u = 0; u < 2; ++u)
                            if (l0 + u < HL)
                                VecN<GT, V>::load_hint(static_cast<const GT *>(p.g) +
                                                           (static_cast<long long>(a) * HL + l0 + u) * count + base + e0,
                                                       g2[u], valid, vec, pol_stream);
                    };
                    constexpr bool kG2Early = MODE == 8 && K >= 2;
                    if constexpr (kG2Early) load_g2(0);
                    const int rb = lm.rbeg[a], re = lm.rbeg[a + 1];
                    for (int i0 = rb; i0 < re; i0 += 4) {   // up to 4 remote tiles in flight
                        float v[4][V];
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (i0 + u < re) VecN<WT, V>::load_cg(inbox(g.me, lm.rs[i0 + u]) + base + e0, v[u], valid, true);
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (i0 + u < re) {
                                const float c = lm.rc[i0 + u];
#pragma unroll
                                for (int j = 0; j < V; ++j) acc[j] = fmaf(c, v[u][j], acc[j]);
                            }
                    }
                    if constexpr (MODE == 8) {   // H-AWC: broadcast to the machine's rows, - lr g per row;
                        // the g rows are loaded 2 at a time before their first use (4 spill); rows 0-1
                        // were issued before the remote tiles
                        for (int l0 = 0; l0 < HL; l0 += 2) {
                            if (l0 > 0 || !kG2Early) load_g2(l0);
#pragma unroll
                            for (int u = 0; u < 2; ++u)
                                if (l0 + u < HL) {
                                    const long long row = static_cast<long long>(a) * HL + l0 + u;
                                    float out[V];
#pragma unroll
                                    for (int i = 0; i < V; ++i) out[i] = fmaf(-p.lr, g2[u][i], acc[i]);
                                    VecN<YT, V>::store_hint(static_cast<YT *>(p.y) + row * count + base + e0, out, valid,
                                                            vec, pol_stream);
                                }
                        }
                    } else if constexpr (HIER) {   // broadcast to the machine's rows
                        for (int l = 0; l < HL; ++l) {
                            const long long row = static_cast<long long>(a) * HL + l;
                            VecN<YT, V>::store_hint(static_cast<YT *>(p.y) + row * count + base + e0, acc, valid, vec,
                                                    pol_stream);
                        }
                    } else {
                        YT *yr = static_cast<YT *>(p.y) + static_cast<long long>(a) * count + base + e0;
                        VecN<YT, V>::store_hint(yr, acc, valid, vec, pol_stream);
                        if (p.shadow) {
                            bf16 *sr = static_cast<bf16 *>(p.shadow) + static_cast<long long>(a) * count + base + e0;
                            VecN<bf16, V>::store_hint(sr, acc, valid, vec, pol_stream);
                        }
                    }
                    if constexpr (MODE == 5) {   // x = u / v (appendix)
                        const float vn = s_vnew[a];
#pragma unroll
                        for (int i = 0; i < V; ++i) acc[i] = acc[i] / vn;
                        VecN<float, V>::store_hint(p.x_out + static_cast<long long>(a) * count + base + e0, acc, valid,
                                                   vec, pol_stream);
                    }
                }
            }
            // ---------------- publish sub-item m and park the local part of its combine ----------------
            if (m < nmine) {
                const long long base = static_cast<long long>(sub(m)) * kSubT;
                const int valid = clamp_valid_v<V>(count - base, e0);
                float xv[K][V];
                float gv[HAS_G && !HIER ? K : 1][V];
                if constexpr (HIER) {   // the machine average of the L rows (R12), H-ATC: of x - lr g
#pragma unroll
                    for (int a = 0; a < K; ++a) {
                        float sum[V];
#pragma unroll
                        for (int i = 0; i < V; ++i) sum[i] = 0.f;
#pragma unroll 4
                        for (int l = 0; l < HLin; ++l) {
                            const long long row = static_cast<long long>(a) * HLin + l;
                            float r[V];
                            VecN<XT, V>::load_hint(xrow(0) + row * count + base + e0, r, valid, vec, pol_stream);
                            if constexpr (MODE == 7) {
                                float gr[V];
                                VecN<GT, V>::load_hint(grow(0) + row * count + base + e0, gr, valid, vec, pol_stream);
#pragma unroll
                                for (int i = 0; i < V; ++i) r[i] = fmaf(-p.lr, gr[i], r[i]);
                            }
#pragma unroll
                            for (int i = 0; i < V; ++i) sum[i] += r[i];
                        }
#pragma unroll
                        for (int i = 0; i < V; ++i) xv[a][i] = sum[i] * invL;
                    }
                } else if constexpr (PREFETCH) {
#pragma unroll
                    for (int a = 0; a < K; ++a) VecN<XT, V>::unpack(xraw[a], xv[a]);
                } else {
#pragma unroll
                    for (int a = 0; a < K; ++a) VecN<XT, V>::load_hint(xrow(a) + base + e0, xv[a], valid, vec, pol_stream);
                }
                if constexpr (HAS_G && !HIER) {
                    if constexpr (PREFETCH) {
#pragma unroll
                        for (int a = 0; a < K; ++a) VecN<GT, V>::unpack(graw[a], gv[a]);
                    } else {
#pragma unroll
                        for (int a = 0; a < K; ++a) VecN<GT, V>::load_hint(grow(a) + base + e0, gv[a], valid, vec, pol_stream);
                    }
                }
                if constexpr (MODE == 1 || MODE == 5) {   // Eq. 4 (GT: u - lr y)
#pragma unroll
                    for (int a = 0; a < K; ++a)
#pragma unroll
                        for (int i = 0; i < V; ++i) xv[a][i] = fmaf(-p.lr, gv[a][i], xv[a][i]);
                }
                if constexpr (MODE == 4) {   // GT y-step: y + g - g_prev
#pragma unroll
                    for (int a = 0; a < K; ++a) {
                        float hv[V];
                        VecN<float, V>::load_hint(p.g2 + static_cast<long long>(a) * count + base + e0, hv, valid, vec,
                                                  pol_stream);
#pragma unroll
                        for (int i = 0; i < V; ++i) xv[a][i] = (xv[a][i] + gv[a][i]) - hv[i];
                    }
                }
                if constexpr (MODE == 3) {   // Exact-Diffusion: psi = x - lr g (stored), phi = psi + x - psi_prev
#pragma unroll
                    for (int a = 0; a < K; ++a) {
                        float pv[V];
                        float *pr = p.psi + static_cast<long long>(a) * count + base + e0;
                        VecN<float, V>::load_hint(pr, pv, valid, vec, pol_stream);
                        float psi[V];
#pragma unroll
                        for (int i = 0; i < V; ++i) {
                            psi[i] = fmaf(-p.lr, gv[a][i], xv[a][i]);
                            xv[a][i] = (psi[i] + xv[a][i]) - pv[i];
                        }
                        VecN<float, V>::store_hint(pr, psi, valid, vec, pol_stream);
                    }
                }
                // wire copies into every reader process's inbox (NVLink stores)
#pragma unroll
                for (int a = 0; a < K; ++a) {
                    const unsigned out = lm.procs_out[a];
                    if (!out) continue;
                    for (int q = 0; q < g.nprocs; ++q)
#ifndef BF_PUSH_LOCALSTORE
                        if ((out >> q) & 1u) VecN<WT, V>::store(inbox(q, g.me * K + a) + base + e0, xv[a], valid, true);
#else   // diagnostic builds only: the wire copy lands in the writer's own heap (timing of the remote stores)
                        if ((out >> q) & 1u) VecN<WT, V>::store(inbox(g.me, g.me * K + a) + base + e0, xv[a], valid, true);
#endif
                }
                // local part of every combine: self, then same-process sources ((a - b) mod K)
#pragma unroll
                for (int a = 0; a < K; ++a) {
                    float acc[V];
                    const float cs = lm.c[a][a];
#pragma unroll
                    for (int i = 0; i < V; ++i) acc[i] = cs * xv[a][i];
#pragma unroll
                    for (int d = 1; d < K; ++d) {
                        const int b = (a + K - d) % K;
                        const float c = lm.c[a][b];
                        if (c != 0.f) {
#pragma unroll
                            for (int i = 0; i < V; ++i)
                                acc[i] = fmaf(c, MODE == 0 ? xv[b][i] : VecN<WT, V>::wire(xv[b][i]), acc[i]);
                        }
                    }
                    float *lp = mylag + static_cast<long long>(slot * K + a) * kSubT;
#pragma unroll
                    for (int i = 0; i < V; i += 4) *reinterpret_cast<float4 *>(lp + i) = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
                }
                if constexpr (MODE == 2) {   // AWC (Eq. 16): the remote terms come later; -lr g is local (per row for H-AWC)
#pragma unroll
                    for (int a = 0; a < K; ++a) {
                        float *lp = mylag + static_cast<long long>(slot * K + a) * kSubT;
#pragma unroll
                        for (int i = 0; i < V; ++i) lp[i] = fmaf(-p.lr, gv[a][i], lp[i]);
                    }
                }
                if (lm.procs_out_all && (push_batch_end<B>(push_batch_of<B>(m), nmine) == m + 1)) {
                    const int b = push_batch_of<B>(m);
                    if (b >= kPubRing) {   // the slot's previous phase must have been consumed by its signal warp
                        volatile int *rel = s_rel;
                        while (rel[b % kPubRing] < b - kPubRing && !*fail) __nanosleep(64);
                    }
                    mbar_arrive_release(&pubbar[b % kPubRing]);
                }
            }
        }
    }
    BF_STAT(if (stat && threadIdx.x == 0) stat[3] = globaltimer() - t_k0;)
    __syncthreads();
    BF_STAT(if (stat && threadIdx.x == 0) stat[0] = globaltimer() - t_k0;)
    if (*fail) return;
    last_cta(pad, [&] {
        if constexpr (MODE == 5)
            for (int a = 0; a < K; ++a) p.gt_v[a] = s_vnew[a];
        pad->epoch = e;
        if (p.wmode == kWSchedule) pad->round = pad->round + 1;
        publish_done(g, e);
    });
}

template <typename XT, typename GT, typename WT, typename YT, int MODE, int K>
static cudaError_t launch_push_k(const ExchParams &p, int grid, cudaStream_t s) {
    using Cfg = PushCfg<K, FusedVec<XT>::V>;
    const void *fn = reinterpret_cast<const void *>(exchange_push_kernel<XT, GT, WT, YT, MODE, K>);
    constexpr int kSubT = kThreads * FusedVec<XT>::V;
    static int maxg = 0;
    if (maxg == 0) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
        if (e != cudaSuccess) return e;
        maxg = max_coresident(fn, Cfg::kThreadsPerCta, Cfg::kSmem);
        if (maxg <= 0) return cudaErrorInvalidConfiguration;
    }
    static const int grid_env = getenv("BF_FUSED_GRID") ? atoi(getenv("BF_FUSED_GRID")) : 0;   // tuning
    if (grid <= 0 && grid_env > 0) grid = grid_env;
    if (grid <= 0 || grid > maxg) grid = maxg;
    const long long subs = (p.geo.count + kSubT - 1) / kSubT;
    if (grid > subs) grid = static_cast<int>(subs);
    if (grid > kMaxGrid) grid = kMaxGrid;
    if (grid < 1) grid = 1;
    void *args[] = {const_cast<ExchParams *>(&p)};
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(Cfg::kThreadsPerCta), args, Cfg::kSmem, s);
}

}  // namespace bf
