// window.cu -- one-sided windows for asynchronous push-sum
// on sm_100a.
//
// Protocol (single producer / single consumer per slot, no remote
// read-modify-write, no lock):
//   producer i -> consumer j owns slot (j, q_in) in j's heap, two halves.
//   payload m lands in half m&1 only if the consumer has consumed payload
//   m-2 (consumed >= delivered-1); the producer then releases
//   version = m+1 into j's heap.  Otherwise the payload stays in i's fp32
//   outbox and later payloads accumulate onto it (sender-side accumulation).
//   The consumer's collect sums the payloads consumed..version-1, then
//   releases consumed = version into i's heap.
// Decisions are snapshotted by CTA 0 of the streaming kernel and published to the
// other CTAs through a per-window gate (win_gate), so every CTA acts on the same
// decision -- one launch per operation.  Nothing here waits on another
// agent, so these kernels can run on a single GPU for any number of agents.
#include <cuda_bf16.h>

#include "dev_common.cuh"

namespace bf {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ unsigned long long esize(const WinParams &p) { return p.dtype == 0 ? 4 : 2; }

__device__ __forceinline__ bool active(const WinParams &p, int a) {
    return (p.agent_mask >> a) & 1ull;
}

// ---- snapshot gate ---------------------------------------------------------
// The decisions of one launch (push: deliver or keep in the outbox; collect: the
// (consumed, version) window of every slot) must be the same in every CTA while
// peers keep moving the counters, so CTA 0 takes them and the others wait for it.
// ctl[0] = last snapshot taken, ctl[1] = last launch finished (written by the last
// CTA): a launch's number is ctl[1] + 1, read by every CTA at its start -- ctl[1]
// changes only at the end of a launch, and launches of one window are stream
// ordered -- so no host counter is involved (CUDA-graph capturable).  The grid
// is co-resident (cooperative launch).  Returns the launch number, 0 on a fault.
static __device__ __noinline__ bool win_wait_snapshot(const Geometry &g, const unsigned long long *flag,
                                                      unsigned long long want) {
    return spin_ge(g, flag, want, false);
}

template <typename F>
__device__ unsigned long long win_gate(const WinParams &p, unsigned long long *ctl, F snapshot) {
    __shared__ unsigned long long s_want;
    __shared__ int s_ok;
    if (threadIdx.x == 0) {
        s_want = *reinterpret_cast<volatile unsigned long long *>(&ctl[1]) + 1;
        s_ok = 1;
    }
    __syncthreads();
    const unsigned long long want = s_want;
    if (blockIdx.x == 0) {
        snapshot();
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            st_release_gpu(&ctl[0], want);
        }
    } else if (threadIdx.x == 0) {
        s_ok = win_wait_snapshot(p.geo, &ctl[0], want) ? 1 : 0;
    }
    __syncthreads();
    return s_ok ? want : 0ull;
}

// ---- push side ------------------------------------------------------------
__device__ __noinline__ void win_push_decide(const WinParams &p) {
    const Geometry &g = p.geo;
    const unsigned long long me = g.peer_base[g.me];
    for (int idx = threadIdx.x; idx < g.k * kMaxS; idx += blockDim.x) {
        const int a = idx / kMaxS, q = idx % kMaxS;
        if (!active(p, a) || q >= p.nout[a]) continue;
        const int qo = p.out_q[a][q];
        const unsigned long long cons =
            ld_acquire_sys(at<unsigned long long>(me, p.consumed_off) + a * p.maxdout + qo);
        const unsigned long long dlv = at<unsigned long long>(me, p.delivered_off)[a * p.maxdout + qo];
        const bool deliver = static_cast<long long>(cons) >= static_cast<long long>(dlv) - 1;
        at<unsigned long long>(me, p.dec_off)[a * p.maxdout + qo] = deliver ? 1ull : 0ull;
    }
}

// Elements per thread-vector (16-byte accesses of the window dtype), vectors per
// thread per item, and elements per item (the window kernels' own tile):
// element of vector j of this thread: (j*kThreads + tid)*V.  NV = 8 keeps 8
// independent 16-byte loads of every stream in flight per thread (the r01 tile of
// 4096 elements gave 2 per bf16 thread: ncu showed 48-55% of DRAM peak, latency-bound).
// (BF_WIN_BYTES / 16 fp32 vectors, half as many 8 x bf16 vectors, per stream; the fp32 outbox streams of a backlogged
// destination are walked vector by vector -- the rare path.)
#ifndef BF_WIN_BYTES
#define BF_WIN_BYTES 128   // bytes of each stream in flight per thread
#endif
#ifndef BF_WIN_COLLECT_REVERSE
#define BF_WIN_COLLECT_REVERSE 1
#endif
#ifndef BF_WIN_PUSH_BYTES
#define BF_WIN_PUSH_BYTES BF_WIN_BYTES   // the push kernel holds one stream (x): tuning variant
#endif
template <typename T, int BYTES = BF_WIN_BYTES>
struct WinVec {
    static constexpr int V = sizeof(T) >= 4 ? 4 : 8;
    static constexpr int NV = BYTES / 16 / (sizeof(T) >= 4 ? 1 : 2);   // 32 fp32 values per stream
    static constexpr int TILE = NV * kThreads * V;
};
template <int V>
__device__ __forceinline__ int win_elem(int j) { return (j * kThreads + threadIdx.x) * V; }
template <typename T, int BYTES = BF_WIN_BYTES>
__host__ __device__ __forceinline__ long long win_items(int k, long long count) {
    return static_cast<long long>(k) * ((count + WinVec<T, BYTES>::TILE - 1) / WinVec<T, BYTES>::TILE);
}

// all NV raw vectors of one stream of an item, issued before any use
template <typename T, int V, int NV>
__device__ __forceinline__ void win_load_raw(const T *base, typename VecN<T, V>::Raw (&r)[NV], long long rem,
                                             bool vec) {
    if (vec && rem >= static_cast<long long>(NV) * kThreads * V) {
        const unsigned long long pol = policy_evict_normal();
#pragma unroll
        for (int j = 0; j < NV; ++j) VecN<T, V>::load_raw_fast(base + win_elem<V>(j), r[j], pol);
    } else {
#pragma unroll
        for (int j = 0; j < NV; ++j)
            VecN<T, V>::load_raw(base + win_elem<V>(j), r[j], clamp_valid_v<V>(rem, win_elem<V>(j)), 0ull);
    }
}

// min CTAs per SM for the streaming window kernels (0 = no bound; tuning variants: -DBF_WIN_COLLECT_MINB=6)
#ifndef BF_WIN_PUSH_MINB
#define BF_WIN_PUSH_MINB 3   // C5 A/B: r01 (4-element tiles) 4 per SM best; r02 (128 B per stream) 3 per SM 5.73 -> 5.59 ms
#endif
#ifndef BF_WIN_COLLECT_MINB
#define BF_WIN_COLLECT_MINB 3    // 3 CTAs/SM (80 registers); -1: 4 for bf16, 3 for fp32
#endif
// BF_WIN_HINTS=1: x / out / slot streams carry an L2 evict-first policy (tuning variant)
#ifndef BF_WIN_HINTS
#define BF_WIN_HINTS 0
#endif
#if BF_WIN_HINTS
#define WIN_LD(T_, V_, p_, v_, n_, vec_) VecN<T_, V_>::load_hint(p_, v_, n_, vec_, policy_evict_first())
#define WIN_ST(T_, V_, p_, v_, n_, vec_) VecN<T_, V_>::store_hint(p_, v_, n_, vec_, policy_evict_first())
#else
#define WIN_LD(T_, V_, p_, v_, n_, vec_) VecN<T_, V_>::load(p_, v_, n_, vec_)
#define WIN_ST(T_, V_, p_, v_, n_, vec_) VecN<T_, V_>::store(p_, v_, n_, vec_)
#endif
#if BF_WIN_PUSH_MINB > 0
#define BF_PUSH_LB __launch_bounds__(kThreads, BF_WIN_PUSH_MINB)
#else
#define BF_PUSH_LB __launch_bounds__(kThreads)
#endif
// C5 round at N = 1 (340M bf16 x 8): 2 CTAs/SM (125 registers) 6.32 ms, 3 per SM 5.73 ms,
// 4 per SM 5.70 ms (0.89 of the HBM roofline; profiles/r02_window_collect_ab.txt); with
// the snapshot gate folded in (win_gate), 4 per SM spills: 5.90 ms, 3 per SM 5.72 ms
#if BF_WIN_COLLECT_MINB > 0
#define BF_COLLECT_LB __launch_bounds__(kThreads, BF_WIN_COLLECT_MINB)
#elif BF_WIN_COLLECT_MINB < 0
#define BF_COLLECT_LB __launch_bounds__(kThreads, sizeof(T) == 2 ? 4 : 3)
#else
#define BF_COLLECT_LB __launch_bounds__(kThreads)
#endif
// SGD = true: the gradient-in-window variant (SGP-style, bf_win_accumulate_grad):
// x_half = x - lr g (Eq. 4) replaces x before the payloads and the self scaling.
template <typename T, bool SGD>
__global__ void BF_PUSH_LB win_push_kernel(const __grid_constant__ WinParams p) {
    constexpr int V = WinVec<T, BF_WIN_PUSH_BYTES>::V, NV = WinVec<T, BF_WIN_PUSH_BYTES>::NV,
                  TILE = WinVec<T, BF_WIN_PUSH_BYTES>::TILE;
    const Geometry &g = p.geo;
    const unsigned long long me = g.peer_base[g.me];
    Pad *pad = pad_of(g, g.me);
    const long long count = g.count;
    const bool vec = g.vec_ok != 0;
    const int k = g.k;
    unsigned long long *ctl = at<unsigned long long>(me, p.ctl_off);   // [0..1]: push gate
    const unsigned long long launch = win_gate(p, ctl, [&] { win_push_decide(p); });
    if (!launch) return;
    const unsigned long long *dec = at<unsigned long long>(me, p.dec_off);
    const unsigned long long *dlv = at<unsigned long long>(me, p.delivered_off);
    const unsigned int *obv = at<unsigned int>(me, p.obvalid_off);
    const long long items = win_items<T, BF_WIN_PUSH_BYTES>(k, count);
    for (long long w = blockIdx.x; w < items; w += gridDim.x) {
        const int t = static_cast<int>(w / k), a = static_cast<int>(w % k);
        if (!active(p, a)) continue;
        const long long base = static_cast<long long>(t) * TILE, rem = count - base;
        T *xr = static_cast<T *>(p.x) + static_cast<long long>(a) * count + base;
        typename VecN<T, V>::Raw xraw[NV];
        win_load_raw<T, V, NV>(xr, xraw, rem, vec);
        typename VecN<T, V>::Raw graw[SGD ? NV : 1];
        if constexpr (SGD)
            win_load_raw<T, V, NV>(static_cast<const T *>(p.g) + static_cast<long long>(a) * count + base, graw, rem, vec);
        // x (or x - lr g) of vector j as fp32
        auto xval = [&](int j, float *xv) {
            VecN<T, V>::unpack(xraw[j], xv);
            if constexpr (SGD) {
                float gv[V];
                VecN<T, V>::unpack(graw[j], gv);
#pragma unroll
                for (int i = 0; i < V; ++i) xv[i] = fmaf(-p.lr, gv[i], xv[i]);
            }
        };
        for (int q = 0; q < p.nout[a]; ++q) {
            const int qo = p.out_q[a][q], dst = p.out_dst[a][q], qin = p.out_qin[a][q];
            const float s = p.out_s[a][q];
            const int ci = a * p.maxdout + qo;
            const bool deliver = dec[ci] != 0;
            const bool use_ob = obv[ci] != 0 && !p.overwrite;
            float *ob = at<float>(me, p.outbox_off) + static_cast<long long>(ci) * p.cpad + base;
            T *slot = at<T>(g.peer_base[dst / k],
                            p.slot_off + ((static_cast<unsigned long long>(dst % k) * p.maxdin + qin) * 2 +
                                          (dlv[ci] & 1ull)) * p.cpad * esize(p)) + base;
            // payload = (outbox +) s * x  (push-side scaling, Eq. 10)
            if (use_ob) {   // a backlogged payload to this destination: add onto its outbox
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    const int vl = clamp_valid_v<V>(rem, win_elem<V>(j));
                    float ov[V], xv[V];
                    VecN<float, V>::load(ob + win_elem<V>(j), ov, vl, true);
                    xval(j, xv);
#pragma unroll
                    for (int i = 0; i < V; ++i) ov[i] = fmaf(s, xv[i], ov[i]);
                    if (deliver) {
                        WIN_ST(T, V, slot + win_elem<V>(j), ov, vl, vec);
                        if (p.ef) {   // keep the wire rounding residual (bf16) in the outbox (R24)
                            float r[V];
#pragma unroll
                            for (int i = 0; i < V; ++i) r[i] = ov[i] - (sizeof(T) == 2 ? bf2f(f2bf(ov[i])) : ov[i]);
                            VecN<float, V>::store(ob + win_elem<V>(j), r, vl, true);
                        }
                    } else {
                        VecN<float, V>::store(ob + win_elem<V>(j), ov, vl, true);
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    const int vl = clamp_valid_v<V>(rem, win_elem<V>(j));
                    float pay[V];
                    xval(j, pay);
#pragma unroll
                    for (int i = 0; i < V; ++i) pay[i] = s * pay[i];
                    if (deliver) {
                        WIN_ST(T, V, slot + win_elem<V>(j), pay, vl, vec);
                        if (p.ef) {
                            float r[V];
#pragma unroll
                            for (int i = 0; i < V; ++i) r[i] = pay[i] - (sizeof(T) == 2 ? bf2f(f2bf(pay[i])) : pay[i]);
                            VecN<float, V>::store(ob + win_elem<V>(j), r, vl, true);
                        }
                    } else {
                        VecN<float, V>::store(ob + win_elem<V>(j), pay, vl, true);
                    }
                }
            }
        }
        const float sw = p.self_w[a];
        if (sw != 1.0f || SGD) {   // x <- self_weight * x (R8)
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                float xv[V];
                xval(j, xv);
#pragma unroll
                for (int i = 0; i < V; ++i) xv[i] *= sw;
                WIN_ST(T, V, xr + win_elem<V>(j), xv, clamp_valid_v<V>(rem, win_elem<V>(j)), vec);
            }
        }
    }

    // last CTA: p lane, version release, control state
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned int prev = atomicAdd(&pad->done_ctr, 1u);
        if (prev == gridDim.x - 1) {
            __threadfence_system();
            pad->done_ctr = 0;
            ctl[1] = launch;   // this launch is finished: the next one takes launch + 1
            unsigned long long *dlvw = at<unsigned long long>(me, p.delivered_off);
            unsigned int *obvw = at<unsigned int>(me, p.obvalid_off);
            double *P = at<double>(me, p.p_off);
            double *pout = at<double>(me, p.pout_off);
            for (int a = 0; a < k; ++a) {
                if (!active(p, a)) continue;
                for (int q = 0; q < p.nout[a]; ++q) {
                    const int qo = p.out_q[a][q], dst = p.out_dst[a][q], qin = p.out_qin[a][q];
                    const int ci = a * p.maxdout + qo;
                    const bool deliver = dec[ci] != 0;
                    const bool use_ob = obvw[ci] != 0 && !p.overwrite;
                    const double pv = (use_ob ? pout[ci] : 0.0) + p.out_sd[a][q] * P[a];
                    if (deliver) {
                        const unsigned long long m = dlvw[ci];
                        const unsigned long long slot_idx =
                            static_cast<unsigned long long>(dst % k) * p.maxdin + qin;
                        if (p.with_p)
                            at<double>(g.peer_base[dst / k], p.pslot_off)[slot_idx * 2 + (m & 1)] = pv;
                        __threadfence_system();
                        st_release_sys(at<unsigned long long>(g.peer_base[dst / k], p.version_off) + slot_idx,
                                       m + 1);
                        dlvw[ci] = m + 1;
                        obvw[ci] = p.ef ? 1u : 0u;
                        pout[ci] = 0.0;
                    } else {
                        pout[ci] = pv;
                        obvw[ci] = 1u;
                    }
                }
                P[a] *= p.self_wd[a];
            }
        }
    }
}

// ---- consumer side ----------------------------------------------------------
__device__ __noinline__ void win_collect_decide(const WinParams &p) {
    const Geometry &g = p.geo;
    const unsigned long long me = g.peer_base[g.me];
    for (int idx = threadIdx.x; idx < g.k * kMaxS; idx += blockDim.x) {
        const int b = idx / kMaxS, q = idx % kMaxS;
        if (!active(p, b) || q >= p.nin[b]) continue;
        const int ci = b * p.maxdin + q;
        const unsigned long long v = ld_acquire_sys(at<unsigned long long>(me, p.version_off) + ci);
        const unsigned long long c = at<unsigned long long>(me, p.conslocal_off)[ci];
        unsigned long long *snap = at<unsigned long long>(me, p.snap_off);
        snap[ci * 2] = c;
        snap[ci * 2 + 1] = v;
    }
}

// update == 0: update_then_collect (x += sum of ready payloads, R9)
// update == 1: win_update (out = self*x + sum r_j * latest payload, R10)
template <typename T>
__global__ void BF_COLLECT_LB win_collect_kernel(const __grid_constant__ WinParams p, int update) {
    const Geometry &g = p.geo;
    const unsigned long long me = g.peer_base[g.me];
    Pad *pad = pad_of(g, g.me);
    const long long count = g.count;
    const bool vec = g.vec_ok != 0;
    const int k = g.k;
    unsigned long long *ctl = at<unsigned long long>(me, p.ctl_off) + 2;   // [2..3]: collect gate
    const unsigned long long launch = win_gate(p, ctl, [&] { win_collect_decide(p); });
    if (!launch) return;
    const unsigned long long *snap = at<unsigned long long>(me, p.snap_off);
    // per-CTA acquire of the producers' versions (orders the slot reads below)
    for (int idx = threadIdx.x; idx < k * p.maxdin; idx += blockDim.x)
        (void)ld_acquire_sys(at<unsigned long long>(me, p.version_off) + idx);
    __syncthreads();
    constexpr int V = WinVec<T>::V, NV = WinVec<T>::NV, TILE = WinVec<T>::TILE;
    const long long items = win_items<T>(k, count);
    // the collect walks the items backwards: it starts on the x / slot lines the push
    // kernel wrote last (still in L2), and the next push (forwards) on the ones it wrote last
    for (long long wi = blockIdx.x; wi < items; wi += gridDim.x) {
        const long long w = BF_WIN_COLLECT_REVERSE ? items - 1 - wi : wi;
        const int t = static_cast<int>(w / k), b = static_cast<int>(w % k);
        if (!active(p, b)) continue;
        const long long base = static_cast<long long>(t) * TILE, rem = count - base;
        const T *xr = static_cast<const T *>(p.x) + static_cast<long long>(b) * count + base;
        T *outr = static_cast<T *>(p.out) + static_cast<long long>(b) * count + base;
        const float sw = update ? p.self_w[b] : 1.0f;
        // the first payload of the first in-neighbour is loaded together with x
        // (the common one-payload case has every load in flight before the first use)
        const T *pre_h = nullptr;
        float pre_r = 1.0f;
        if (p.nin[b] > 0) {
            const int ci = b * p.maxdin;
            const unsigned long long c0 = snap[ci * 2], v0 = snap[ci * 2 + 1];
            const unsigned long long m0 = update ? v0 - 1 : c0;
            if (update || c0 < v0) {
                pre_h = at<const T>(me, p.slot_off + (static_cast<unsigned long long>(ci) * 2 + (m0 & 1)) * p.cpad *
                                                         esize(p)) + base;
                pre_r = update ? p.in_r[b][0] : 1.0f;
            }
        }
        float acc[NV][V];
        {
            typename VecN<T, V>::Raw xraw[NV], praw[NV];
            win_load_raw<T, V, NV>(xr, xraw, rem, vec);
            if (pre_h) win_load_raw<T, V, NV>(pre_h, praw, rem, vec);
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                VecN<T, V>::unpack(xraw[j], acc[j]);
#pragma unroll
                for (int i = 0; i < V; ++i) acc[j][i] *= sw;
            }
            if (pre_h) {
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    float v4[V];
                    VecN<T, V>::unpack(praw[j], v4);
#pragma unroll
                    for (int i = 0; i < V; ++i) acc[j][i] = fmaf(pre_r, v4[i], acc[j][i]);
                }
            }
        }
        for (int q = 0; q < p.nin[b]; ++q) {
            const int ci = b * p.maxdin + q;
            const unsigned long long c = snap[ci * 2], v = snap[ci * 2 + 1];
            const float r = update ? p.in_r[b][q] : 1.0f;
            // update: the latest complete payload v-1 (v == 0: the initial copy in half 1);
            // collect: every delivered payload c..v-1, in order.
            const unsigned long long m_first = update ? v - 1 : c;
            const unsigned long long m_end = update ? v : v;
            for (unsigned long long m = m_first; update ? (m == m_first) : (m < m_end);
                 m = update ? m_first + 1 : m + 1) {
                const T *h = at<const T>(me, p.slot_off + (static_cast<unsigned long long>(ci) * 2 + (m & 1)) *
                                                              p.cpad * esize(p)) + base;
                if (h != pre_h) {   // (pre_h was added first: it is the first of this order)
                    typename VecN<T, V>::Raw hraw[NV];
                    win_load_raw<T, V, NV>(h, hraw, rem, vec);
#pragma unroll
                    for (int j = 0; j < NV; ++j) {
                        float v4[V];
                        VecN<T, V>::unpack(hraw[j], v4);
#pragma unroll
                        for (int i = 0; i < V; ++i) acc[j][i] = fmaf(r, v4[i], acc[j][i]);
                    }
                }
                if (update) break;
            }
        }
#pragma unroll
        for (int j = 0; j < NV; ++j)
            WIN_ST(T, V, outr + win_elem<V>(j), acc[j], clamp_valid_v<V>(rem, win_elem<V>(j)), vec);
    }

    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int prev = atomicAdd(&pad->done_ctr, 1u);
        if (prev == gridDim.x - 1) {
            __threadfence();
            pad->done_ctr = 0;
            ctl[1] = launch;
            unsigned long long *cl = at<unsigned long long>(me, p.conslocal_off);
            double *P = at<double>(me, p.p_off);
            const double *ps = at<const double>(me, p.pslot_off);
            for (int b = 0; b < k; ++b) {
                if (!active(p, b)) continue;
                for (int q = 0; q < p.nin[b]; ++q) {
                    const int ci = b * p.maxdin + q;
                    const unsigned long long c = snap[ci * 2], v = snap[ci * 2 + 1];
                    if (!update && p.with_p)
                        for (unsigned long long m = c; m < v; ++m) P[b] += ps[ci * 2 + (m & 1)];
                    cl[ci] = v;
                    const int src = p.in_src[b][q];
                    st_release_sys(at<unsigned long long>(g.peer_base[src / k], p.consumed_off) +
                                       (src % k) * p.maxdout + p.in_qout[b][q],
                                   v);
                }
            }
        }
    }
}

// ---- neighbor_win_get: pull the in-neighbours' window tensors ---------
// Needs the window tensor in the symmetric heap (bf_alloc): agent j's tensor is
// then at peer_base[j / k] + x_off + (j % k) * count * es in every process.
// For each selected in-neighbour (in_r[a][q] != 0): my slot (a, q), half
// version & 1, <- in_r * x_j; win_get_finish then releases version + 1, so
// win_update sees the fetched value as the latest complete payload (R26).
template <typename T>
__global__ void __launch_bounds__(kThreads) win_get_kernel(const __grid_constant__ WinParams p,
                                                           unsigned long long x_off) {
    constexpr int V = WinVec<T>::V, NV = WinVec<T>::NV, TILE = WinVec<T>::TILE;
    const Geometry &g = p.geo;
    const unsigned long long me = g.peer_base[g.me];
    const long long count = g.count;
    const bool vec = g.vec_ok != 0;
    const int k = g.k;
    const unsigned long long *ver = at<unsigned long long>(me, p.version_off);
    const long long items = win_items<T>(k, count);
    for (long long w = blockIdx.x; w < items; w += gridDim.x) {
        const int t = static_cast<int>(w / k), a = static_cast<int>(w % k);
        if (!active(p, a)) continue;
        const long long base = static_cast<long long>(t) * TILE, rem = count - base;
        for (int q = 0; q < p.nin[a]; ++q) {
            const float r = p.in_r[a][q];
            if (r == 0.f) continue;
            const int j = p.in_src[a][q];
            const int ci = a * p.maxdin + q;
            const T *xj = at<const T>(g.peer_base[j / k], x_off + static_cast<unsigned long long>(j % k) * count *
                                                                 esize(p)) + base;
            T *slot = at<T>(me, p.slot_off + (static_cast<unsigned long long>(ci) * 2 + (ver[ci] & 1ull)) * p.cpad *
                                                 esize(p)) + base;
            float v[NV][V];
#pragma unroll
            for (int jv = 0; jv < NV; ++jv)
                VecN<T, V>::load_cg(xj + win_elem<V>(jv), v[jv], clamp_valid_v<V>(rem, win_elem<V>(jv)), vec);
#pragma unroll
            for (int jv = 0; jv < NV; ++jv) {
#pragma unroll
                for (int i = 0; i < V; ++i) v[jv][i] *= r;
                VecN<T, V>::store(slot + win_elem<V>(jv), v[jv], clamp_valid_v<V>(rem, win_elem<V>(jv)), vec);
            }
        }
    }
}

__global__ void win_get_finish(const __grid_constant__ WinParams p) {
    const Geometry &g = p.geo;
    const unsigned long long me = g.peer_base[g.me];
    __threadfence();   // every slot store of the copy kernel (stream-ordered before) is visible
    for (int idx = threadIdx.x; idx < g.k * kMaxS; idx += blockDim.x) {
        const int a = idx / kMaxS, q = idx % kMaxS;
        if (!active(p, a) || q >= p.nin[a] || p.in_r[a][q] == 0.f) continue;
        unsigned long long *v = at<unsigned long long>(me, p.version_off) + a * p.maxdin + q;
        st_release_gpu(v, *v + 1);
    }
}

static int stream_grid(long long items) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long g = static_cast<long long>(sms) * 4;
    if (items < g) g = items;
    return g < 1 ? 1 : static_cast<int>(g);
}

// grid of a window streaming kernel: every CTA the SMs can hold (occupancy), at
// most one per item
template <typename F>
static int occ_grid(F fn, long long items) {
    // co-resident CTAs, cached per kernel (instantiations of one signature share F)
    static const void *fns[16] = {};
    static int occ[16] = {};
    const void *f = reinterpret_cast<const void *>(fn);
    int slot = 0;
    while (slot < 15 && fns[slot] && fns[slot] != f) ++slot;
    if (fns[slot] != f) {
        fns[slot] = f;
        occ[slot] = max_coresident(f, kThreads, 0);
    }
    const int maxg = occ[slot];
    long long g = maxg > 0 ? maxg : stream_grid(items);
    if (items < g) g = items;
    return g < 1 ? 1 : static_cast<int>(g);
}

// cooperative launch: CTAs 1.. wait for CTA 0's snapshot, so every CTA is resident
template <typename K>
static cudaError_t coop(K kernel, int grid, cudaStream_t s, const WinParams &p) {
    void *args[] = {const_cast<WinParams *>(&p)};
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(kernel), dim3(grid), dim3(kThreads), args, 0, s);
}
template <typename K>
static cudaError_t coop2(K kernel, int grid, cudaStream_t s, const WinParams &p, int update) {
    void *args[] = {const_cast<WinParams *>(&p), &update};
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(kernel), dim3(grid), dim3(kThreads), args, 0, s);
}

cudaError_t launch_win_push(const WinParams &p, int grid, cudaStream_t s) {
    const long long items = p.dtype == 0 ? win_items<float, BF_WIN_PUSH_BYTES>(p.geo.k, p.geo.count)
                                         : win_items<bf16, BF_WIN_PUSH_BYTES>(p.geo.k, p.geo.count);
    if (p.g) {
        if (grid <= 0)
            grid = p.dtype == 0 ? occ_grid(win_push_kernel<float, true>, items) : occ_grid(win_push_kernel<bf16, true>, items);
        return p.dtype == 0 ? coop(win_push_kernel<float, true>, grid, s, p) : coop(win_push_kernel<bf16, true>, grid, s, p);
    }
    if (grid <= 0)
        grid = p.dtype == 0 ? occ_grid(win_push_kernel<float, false>, items) : occ_grid(win_push_kernel<bf16, false>, items);
    return p.dtype == 0 ? coop(win_push_kernel<float, false>, grid, s, p) : coop(win_push_kernel<bf16, false>, grid, s, p);
}

cudaError_t launch_win_get(const WinParams &p, unsigned long long x_off, cudaStream_t s) {
    if (p.dtype == 0)
        win_get_kernel<float><<<occ_grid(win_get_kernel<float>, win_items<float>(p.geo.k, p.geo.count)), kThreads, 0,
                                s>>>(p, x_off);
    else
        win_get_kernel<bf16><<<occ_grid(win_get_kernel<bf16>, win_items<bf16>(p.geo.k, p.geo.count)), kThreads, 0,
                               s>>>(p, x_off);
    win_get_finish<<<1, 256, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_win_collect(const WinParams &p, int update, int grid, cudaStream_t s) {
    if (grid <= 0)
        grid = p.dtype == 0 ? occ_grid(win_collect_kernel<float>, win_items<float>(p.geo.k, p.geo.count))
                            : occ_grid(win_collect_kernel<bf16>, win_items<bf16>(p.geo.k, p.geo.count));
    return p.dtype == 0 ? coop2(win_collect_kernel<float>, grid, s, p, update)
                        : coop2(win_collect_kernel<bf16>, grid, s, p, update);
}

}  // namespace bf
