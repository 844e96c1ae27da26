// exchange_ll.cuh -- the small-message variant of the cross-GPU exchange
// (C1 / C2 sizes: latency-bound, "O(1) latency").
//
// Every element travels with its epoch: the writer stores (epoch << 32 | bits of
// the wire value) as one 64-bit word -- single-copy atomic -- straight into the
// reader's LL inbox over NVLink, and the reader spins on its own inbox words
// until they carry this epoch.  No fence and no progress word on the data path:
// the push kernel's fence (~1-3 us idle, a round trip for the remote stores)
// plus the progress word's flight (~2.7 us one way) collapse into the data's own
// flight.  Twice the bytes on the wire: measured at N = 2, the tagged words win up
// to ~2 MB per agent (1 MB fp32: 16.9 vs 19.9 us pushed; 4 MB: 30.4 vs 27.7 us).
// WAR protection of the double-buffered inbox and the epoch / round / done
// bookkeeping are those of the other exchange kernels; stale words of epoch e-2
// carry another tag.  Static and scheduled topologies (the writer must know its
// readers), MODE 0 / 1 / 2 (neighbor_allreduce, ATC, AWC), K = 1, 2, 4.
#pragma once

namespace bf {

constexpr int kLLThreads = 256;

__device__ __forceinline__ void st_ll2(unsigned long long *p, unsigned long long a, unsigned long long b) {
    asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_ll2(const unsigned long long *p, unsigned long long &a, unsigned long long &b) {
    asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

template <typename XT, typename GT, typename WT, typename YT, int MODE, int K>
__global__ void __launch_bounds__(kLLThreads) exchange_ll_kernel(const __grid_constant__ ExchParams p) {
    constexpr bool HAS_G = MODE != 0;
    constexpr int V = 4;   // elements per thread-vector (fp32: 16 B, bf16: 8 B)
    __shared__ SharedTab st;
    __shared__ PushMix<K> lm;
    __shared__ int s_fail;
    const Geometry &g = p.geo;
    Pad *pad = pad_of(g, g.me);
    if (aborted(g)) return;
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long *>(&pad->epoch) + 1;
    const int parity = static_cast<int>(e & 1);
    const unsigned long long tag = (e & 0xffffffffull) << 32;
    if (threadIdx.x == 0) s_fail = 0;
    bool ok = war_wait(g, e);
    ok = resolve_sources(p, e, st) && ok;
    if (!ok) return;
    if (threadIdx.x == 0) {
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
                    ++nr;
                }
            }
        }
        lm.rbeg[K] = nr;
        for (int a = 0; a < K; ++a) {
            unsigned out = 0;
            if (p.wmode == kWStatic) {
                out = p.pushq[a];
            } else {
                const unsigned long long round = *reinterpret_cast<volatile unsigned long long *>(&pad->round);
                int src, dst;
                sched_peers(p.sched_kind, g.n, p.sched_L, round, g.me * K + a, src, dst);
                if (dst >= 0 && dst / K != g.me) out = 1u << (dst / K);
            }
            lm.procs_out[a] = out;
        }
    }
    __syncthreads();
    const long long count = g.count;
    const bool vec = g.vec_ok != 0;
    // LL inbox words of source agent j in process q's heap: [j][parity][element]
    auto ll = [&](int q, int j) {
        return at<unsigned long long>(g.peer_base[q], p.ll_off + (static_cast<unsigned long long>(j) * 2 + parity) *
                                                                  p.ll_stride);
    };
    const long long nvec = (count + V - 1) / V;
    volatile int *fail = &s_fail;
    for (long long v = static_cast<long long>(blockIdx.x) * kLLThreads + threadIdx.x; v < nvec;
         v += static_cast<long long>(gridDim.x) * kLLThreads) {
        const long long e0 = v * V;
        const int valid = clamp_valid_v<V>(count - e0, 0);
        float xv[K][V];
        float gv[HAS_G ? K : 1][V];
#pragma unroll
        for (int a = 0; a < K; ++a) VecN<XT, V>::load(static_cast<const XT *>(p.x) + a * count + e0, xv[a], valid, vec);
        if constexpr (HAS_G) {
#pragma unroll
            for (int a = 0; a < K; ++a) VecN<GT, V>::load(static_cast<const GT *>(p.g) + a * count + e0, gv[a], valid, vec);
        }
        if constexpr (MODE == 1) {
#pragma unroll
            for (int a = 0; a < K; ++a)
#pragma unroll
                for (int i = 0; i < V; ++i) xv[a][i] = fmaf(-p.lr, gv[a][i], xv[a][i]);   // Eq. 4
        }
        // tagged wire words to every reader process (no fence: the tag orders them)
#pragma unroll
        for (int a = 0; a < K; ++a) {
            const unsigned out = lm.procs_out[a];
            if (!out) continue;
            unsigned long long w[V];
#pragma unroll
            for (int i = 0; i < V; ++i) w[i] = tag | __float_as_uint(MODE == 0 ? xv[a][i] : VecN<WT, V>::wire(xv[a][i]));
            for (int q = 0; q < g.nprocs; ++q) {
                if (!((out >> q) & 1u)) continue;
                unsigned long long *dst = ll(q, g.me * K + a) + e0;
                st_ll2(dst, w[0], w[1]);
                st_ll2(dst + 2, w[2], w[3]);
            }
        }
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
            for (int r = lm.rbeg[a]; r < lm.rbeg[a + 1]; ++r) {   // remote sources: spin on the tagged words
                const unsigned long long *src = ll(g.me, lm.rs[r]) + e0;
                unsigned long long w[V];
                const unsigned long long t0 = globaltimer();
                unsigned it = 0;
                while (true) {
                    ld_ll2(src, w[0], w[1]);
                    ld_ll2(src + 2, w[2], w[3]);
                    bool ready = true;
#pragma unroll
                    for (int i = 0; i < V; ++i) ready = ready && (i >= valid || (w[i] & 0xffffffff00000000ull) == tag);
                    if (ready) break;
                    if ((++it & 255u) == 0) {
                        if (*fail || ld_relaxed_sys_u32(&pad->abort)) {
                            *fail = 1;
                            break;
                        }
                        if (globaltimer() - t0 > g.timeout_ns) {
                            abort_all(g, BF_ERR_TIMEOUT);
                            *fail = 1;
                            break;
                        }
                    }
                }
                if (*fail) break;
                const float c = lm.rc[r];
#pragma unroll
                for (int i = 0; i < V; ++i) acc[i] = fmaf(c, __uint_as_float(static_cast<unsigned>(w[i])), acc[i]);
            }
            if constexpr (MODE == 2) {   // AWC (Eq. 16)
#pragma unroll
                for (int i = 0; i < V; ++i) acc[i] = fmaf(-p.lr, gv[a][i], acc[i]);
            }
            VecN<YT, V>::store(static_cast<YT *>(p.y) + a * count + e0, acc, valid, vec);
            if (p.shadow) VecN<bf16, V>::store(static_cast<bf16 *>(p.shadow) + a * count + e0, acc, valid, vec);
        }
        if (*fail) break;
    }
    __syncthreads();
    if (*fail) {
        if (g.host_err && threadIdx.x == 0) {
            const unsigned code = ld_relaxed_sys_u32(&pad->abort);
            if (code) *g.host_err = code;
        }
        return;
    }
    last_cta(pad, [&] {
        pad->epoch = e;
        if (p.wmode == kWSchedule) pad->round = pad->round + 1;
        publish_done(g, e);
    });
}

template <typename XT, typename GT, typename WT, typename YT, int MODE, int K>
static cudaError_t launch_ll_k(const ExchParams &p, cudaStream_t s) {
    if constexpr (MODE > 2) {
        return cudaErrorInvalidValue;
    } else {
        const long long nvec = (p.geo.count + 3) / 4;
        long long grid = (nvec + kLLThreads - 1) / kLLThreads;
        if (grid > 296) grid = 296;
        exchange_ll_kernel<XT, GT, WT, YT, MODE, K><<<static_cast<int>(grid), kLLThreads, 0, s>>>(p);
        return cudaGetLastError();
    }
}

}  // namespace bf
