// dev_common.cuh -- device helpers for the sm_100a kernels: system-scope
// acquire/release flags (cross-GPU over NVLink through CUDA-IPC mappings),
// bounded spins, 4-element vector loads/stores for fp32 / bf16.
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

#include "bf_internal.h"

namespace bf {

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys_u32(unsigned int *p, unsigned int v) {
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_relaxed_sys_u32(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Flags read by other GPUs need system scope; flags only read on this GPU
// (every agent on one GPU) take the cheaper GPU scope.
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long *p, bool sys) {
    return sys ? ld_acquire_sys(p) : ld_acquire_gpu(p);
}
__device__ __forceinline__ void st_release(unsigned long long *p, unsigned long long v, bool sys) {
    if (sys)
        st_release_sys(p, v);
    else
        st_release_gpu(p, v);
}

__device__ __forceinline__ void fence_acq_rel(bool sys) {
    if (sys)
        asm volatile("fence.acq_rel.sys;" ::: "memory");
    else
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p, bool sys) {
    unsigned long long v;
    if (sys)
        asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v, bool sys) {
    if (sys)
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else
        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---- TMA bulk copies + mbarriers (sm_90+ async proxy; SASS UBLKCP / SYNCS) ----
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// order generic-proxy accesses (e.g. an acquire of a peer's flag) before later
// async-proxy (TMA) accesses of global memory
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *smem_dst, const void *gsrc, unsigned bytes,
                                            unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// L2 cache policies (createpolicy): streaming data evict-first, published
// tiles evict-last so that the neighbours' re-reads hit L2.
__device__ __forceinline__ unsigned long long policy_evict_first() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ unsigned long long policy_evict_normal() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_load_1d_hint(void *smem_dst, const void *gsrc, unsigned bytes,
                                                 unsigned long long *bar, unsigned long long pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void st_hint_v4f(float *p, const float v[4], unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v[0]), "f"(v[1]),
                 "f"(v[2]), "f"(v[3]), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void st_hint_v2u(void *p, unsigned a, unsigned b, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(a), "r"(b), "l"(pol)
                 : "memory");
}
// 128-bit / 64-bit loads with an L2 eviction policy, bypassing L1 (streamed once)
__device__ __forceinline__ float4 ld_hint_v4f(const float *p, unsigned long long pol) {
    float4 v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint2 ld_hint_v2u(const void *p, unsigned long long pol) {
    uint2 v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "LAB_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LAB_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_release(unsigned long long *bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_acquire(unsigned long long *bar, unsigned phase) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 16-byte LDGSTS with zero fill beyond src_bytes (0..16); generic-proxy global
// read, so it is valid on CUDA-IPC peer mappings (NVLink) as well as local HBM.
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc, unsigned src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)), "l"(gsrc),
                 "r"(src_bytes)
                 : "memory");
}
// arrive on `bar` when all prior cp.async of this thread have completed
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(unsigned long long *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Kernel prologue check: a fault raised earlier (here or by a peer) stops the
// kernel and is latched in the host-visible error word.
__device__ __forceinline__ bool aborted(const Geometry &g) {
    const unsigned int code = *reinterpret_cast<volatile unsigned int *>(
        &reinterpret_cast<Pad *>(g.peer_base[g.me])->abort);
    if (code && g.host_err && threadIdx.x == 0) *g.host_err = code;
    return code != 0;
}

template <typename T>
__device__ __forceinline__ T *at(unsigned long long base, unsigned long long off) {
    return reinterpret_cast<T *>(base + off);
}

__device__ __forceinline__ Pad *pad_of(const Geometry &g, int proc) {
    return reinterpret_cast<Pad *>(g.peer_base[proc]);
}

// Raise an abort in every process (so peers stop waiting quickly) and latch
// the code in the host-mapped error word.
static __device__ __noinline__ void abort_all(const Geometry &g, unsigned int code) {
    for (int q = 0; q < g.nprocs; ++q) st_relaxed_sys_u32(&pad_of(g, q)->abort, code);
    if (g.host_err) *g.host_err = code;
    __threadfence_system();
}

// Spin until *flag >= target.  Bounded by the context timeout and by the
// abort word of this process.  Returns false on timeout / abort.
__device__ __forceinline__ bool spin_ge(const Geometry &g, const unsigned long long *flag,
                                        unsigned long long target, bool sys = true) {
    if (ld_acquire(flag, sys) >= target) return true;
    const unsigned long long t0 = globaltimer();
    const unsigned int *abort_w = &pad_of(g, g.me)->abort;
    unsigned int it = 0;
    while (true) {
        if (ld_acquire(flag, sys) >= target) return true;
        if ((++it & 63u) == 0) {
            const unsigned int code = ld_relaxed_sys_u32(abort_w);
            if (code) {   // raised by a peer: latch it for this process's host too
                if (g.host_err) *g.host_err = code;
                return false;
            }
            if (globaltimer() - t0 > g.timeout_ns) {
                abort_all(g, BF_ERR_TIMEOUT);
                return false;
            }
        }
        __nanosleep(32);
    }
}

// Bounded mbarrier wait: returns false (and fails the CTA) on timeout or when
// *fail is already set, so a protocol fault can never hang the GPU.
__device__ __forceinline__ bool mbar_try(unsigned long long *bar, unsigned phase) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
// non-blocking test of a phase
__device__ __forceinline__ bool mbar_test(unsigned long long *bar, unsigned phase) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool mbar_wait_b(const Geometry &g, unsigned long long *bar, unsigned phase,
                                            volatile int *fail) {
    if (mbar_try(bar, phase)) return true;
    const unsigned long long t0 = globaltimer();
    while (true) {
        if (mbar_try(bar, phase)) return true;
        if (*fail) return false;
        if (globaltimer() - t0 > g.timeout_ns) {
            *fail = 1;
            abort_all(g, BF_ERR_TIMEOUT);
            return false;
        }
    }
}

// bounded wait with explicit acquire semantics (pairs with mbar_arrive_release)
__device__ __forceinline__ bool mbar_wait_acq_b(const Geometry &g, unsigned long long *bar, unsigned phase,
                                                volatile int *fail) {
    if (mbar_try_acquire(bar, phase)) return true;
    const unsigned long long t0 = globaltimer();
    while (true) {
        if (mbar_try_acquire(bar, phase)) return true;
        if (*fail) return false;
        if (globaltimer() - t0 > g.timeout_ns) {
            *fail = 1;
            abort_all(g, BF_ERR_TIMEOUT);
            return false;
        }
    }
}

// ---- 4-element vector access --------------------------------------------
// fp32: one 16-byte access; bf16: one 8-byte access.  `valid` < 4 takes the
// guarded scalar path (ragged tail / unaligned rows).
template <typename T>
struct Vec4;

template <>
struct Vec4<float> {
    static __device__ __forceinline__ void load(const float *p, float v[4], int valid, bool vec) {
        if (vec && valid == 4) {
            float4 q = *reinterpret_cast<const float4 *>(p);
            v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) v[i] = i < valid ? p[i] : 0.f;
        }
    }
    // L2-only load (peer slots: never serve a stale L1 line)
    static __device__ __forceinline__ void load_cg(const float *p, float v[4], int valid, bool vec) {
        if (vec && valid == 4) {
            float4 q = __ldcg(reinterpret_cast<const float4 *>(p));
            v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) v[i] = i < valid ? __ldcg(p + i) : 0.f;
        }
    }
    static __device__ __forceinline__ void store(float *p, const float v[4], int valid, bool vec) {
        if (vec && valid == 4) {
            *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (i < valid) p[i] = v[i];
        }
    }
    static __device__ __forceinline__ void store_hint(float *p, const float v[4], int valid, bool vec,
                                                      unsigned long long pol);
    static __device__ __forceinline__ void load_hint(const float *p, float v[4], int valid, bool vec,
                                                     unsigned long long pol) {
        if (vec && valid == 4) {
            float4 q = ld_hint_v4f(p, pol);
            v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
        } else {
            load(p, v, valid, vec);
        }
    }
    // value as it travels on a wire of this dtype
    static __device__ __forceinline__ float wire(float f) { return f; }
    // two-stage load: the raw 16 bytes first (so a thread can issue all of its
    // loads before the first use), converted to fp32 afterwards
    using Raw = float4;
    static __device__ __forceinline__ void load_raw_fast(const float *p, Raw &r, unsigned long long pol) {
        r = ld_hint_v4f(p, pol);
    }
    static __device__ __forceinline__ void load_raw(const float *p, Raw &r, int valid, bool vec,
                                                    unsigned long long pol) {
        if (vec && valid == 4) {
            r = ld_hint_v4f(p, pol);
        } else {
            r.x = valid > 0 ? p[0] : 0.f;
            r.y = valid > 1 ? p[1] : 0.f;
            r.z = valid > 2 ? p[2] : 0.f;
            r.w = valid > 3 ? p[3] : 0.f;
        }
    }
    static __device__ __forceinline__ void unpack(const Raw &r, float v[4]) {
        v[0] = r.x; v[1] = r.y; v[2] = r.z; v[3] = r.w;
    }
};

__device__ __forceinline__ unsigned short f2bf(float f) {
    __nv_bfloat16 h = __float2bfloat16_rn(f);
    return *reinterpret_cast<unsigned short *>(&h);
}
__device__ __forceinline__ float bf2f(unsigned short u) {
    return __uint_as_float(static_cast<unsigned int>(u) << 16);
}

template <>
struct Vec4<__nv_bfloat16> {
    static __device__ __forceinline__ void load(const __nv_bfloat16 *p, float v[4], int valid, bool vec) {
        const unsigned short *q = reinterpret_cast<const unsigned short *>(p);
        if (vec && valid == 4) {
            uint2 w = *reinterpret_cast<const uint2 *>(q);
            v[0] = __uint_as_float(w.x << 16); v[1] = __uint_as_float(w.x & 0xFFFF0000u);
            v[2] = __uint_as_float(w.y << 16); v[3] = __uint_as_float(w.y & 0xFFFF0000u);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) v[i] = i < valid ? bf2f(q[i]) : 0.f;
        }
    }
    static __device__ __forceinline__ void load_cg(const __nv_bfloat16 *p, float v[4], int valid, bool vec) {
        const unsigned short *q = reinterpret_cast<const unsigned short *>(p);
        if (vec && valid == 4) {
            uint2 w = __ldcg(reinterpret_cast<const uint2 *>(q));
            v[0] = __uint_as_float(w.x << 16); v[1] = __uint_as_float(w.x & 0xFFFF0000u);
            v[2] = __uint_as_float(w.y << 16); v[3] = __uint_as_float(w.y & 0xFFFF0000u);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) v[i] = i < valid ? bf2f(__ldcg(q + i)) : 0.f;
        }
    }
    static __device__ __forceinline__ void store(__nv_bfloat16 *p, const float v[4], int valid, bool vec) {
        unsigned short *q = reinterpret_cast<unsigned short *>(p);
        if (vec && valid == 4) {
            uint2 w;
            w.x = static_cast<unsigned int>(f2bf(v[0])) | (static_cast<unsigned int>(f2bf(v[1])) << 16);
            w.y = static_cast<unsigned int>(f2bf(v[2])) | (static_cast<unsigned int>(f2bf(v[3])) << 16);
            *reinterpret_cast<uint2 *>(q) = w;
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (i < valid) q[i] = f2bf(v[i]);
        }
    }
    static __device__ __forceinline__ void store_hint(__nv_bfloat16 *p, const float v[4], int valid, bool vec,
                                                      unsigned long long pol);
    static __device__ __forceinline__ void load_hint(const __nv_bfloat16 *p, float v[4], int valid, bool vec,
                                                     unsigned long long pol) {
        if (vec && valid == 4) {
            uint2 w = ld_hint_v2u(p, pol);
            v[0] = __uint_as_float(w.x << 16); v[1] = __uint_as_float(w.x & 0xFFFF0000u);
            v[2] = __uint_as_float(w.y << 16); v[3] = __uint_as_float(w.y & 0xFFFF0000u);
        } else {
            load(p, v, valid, vec);
        }
    }
    // value as it travels on a bf16 wire: round to nearest even (R17)
    static __device__ __forceinline__ float wire(float f) { return bf2f(f2bf(f)); }
    using Raw = uint2;
    static __device__ __forceinline__ void load_raw_fast(const __nv_bfloat16 *p, Raw &r, unsigned long long pol) {
        r = ld_hint_v2u(p, pol);
    }
    static __device__ __forceinline__ void load_raw(const __nv_bfloat16 *p, Raw &r, int valid, bool vec,
                                                    unsigned long long pol) {
        if (vec && valid == 4) {
            r = ld_hint_v2u(p, pol);
        } else {
            const unsigned short *q = reinterpret_cast<const unsigned short *>(p);
            const unsigned e0 = valid > 0 ? q[0] : 0u, e1 = valid > 1 ? q[1] : 0u;
            const unsigned e2 = valid > 2 ? q[2] : 0u, e3 = valid > 3 ? q[3] : 0u;
            r.x = e0 | (e1 << 16);
            r.y = e2 | (e3 << 16);
        }
    }
    static __device__ __forceinline__ void unpack(const Raw &r, float v[4]) {
        v[0] = __uint_as_float(r.x << 16); v[1] = __uint_as_float(r.x & 0xFFFF0000u);
        v[2] = __uint_as_float(r.y << 16); v[3] = __uint_as_float(r.y & 0xFFFF0000u);
    }
};

__device__ __forceinline__ void Vec4<float>::store_hint(float *p, const float v[4], int valid, bool vec,
                                                        unsigned long long pol) {
    if (vec && valid == 4)
        st_hint_v4f(p, v, pol);
    else
        store(p, v, valid, vec);
}
__device__ __forceinline__ void Vec4<__nv_bfloat16>::store_hint(__nv_bfloat16 *p, const float v[4], int valid,
                                                                bool vec, unsigned long long pol) {
    if (vec && valid == 4) {
        const unsigned a = static_cast<unsigned>(f2bf(v[0])) | (static_cast<unsigned>(f2bf(v[1])) << 16);
        const unsigned b = static_cast<unsigned>(f2bf(v[2])) | (static_cast<unsigned>(f2bf(v[3])) << 16);
        st_hint_v2u(p, a, b, pol);
    } else {
        store(p, v, valid, vec);
    }
}

// ---- V-element vectors (16-byte accesses for bf16: V = 8) -------------------
// VecN<T, 4> is Vec4<T>; VecN<bf16, 8> moves 8 bf16 values with one 16-byte
// access (the fused kernel uses V = 16 / sizeof(x dtype) elements per thread).
template <typename T, int V>
struct VecN;

template <typename T>
struct VecN<T, 4> {
    using Raw = typename Vec4<T>::Raw;
    static __device__ __forceinline__ void load_raw_fast(const T *p, Raw &r, unsigned long long pol) {
        Vec4<T>::load_raw_fast(p, r, pol);
    }
    static __device__ __forceinline__ void load_raw(const T *p, Raw &r, int valid, unsigned long long pol) {
        Vec4<T>::load_raw(p, r, valid, false, pol);
    }
    static __device__ __forceinline__ void unpack(const Raw &r, float v[4]) { Vec4<T>::unpack(r, v); }
    static __device__ __forceinline__ void load(const T *p, float v[4], int valid, bool vec) {
        Vec4<T>::load(p, v, valid, vec);
    }
    static __device__ __forceinline__ void load_hint(const T *p, float v[4], int valid, bool vec,
                                                     unsigned long long pol) {
        Vec4<T>::load_hint(p, v, valid, vec, pol);
    }
    static __device__ __forceinline__ void store_hint(T *p, const float v[4], int valid, bool vec,
                                                      unsigned long long pol) {
        Vec4<T>::store_hint(p, v, valid, vec, pol);
    }
    static __device__ __forceinline__ float wire(float f) { return Vec4<T>::wire(f); }
    static __device__ __forceinline__ void store(T *p, const float v[4], int valid, bool vec) {
        Vec4<T>::store(p, v, valid, vec);
    }
    static __device__ __forceinline__ void load_cg(const T *p, float v[4], int valid, bool vec) {
        Vec4<T>::load_cg(p, v, valid, vec);
    }
};

template <>
struct VecN<__nv_bfloat16, 8> {
    using Raw = uint4;
    static __device__ __forceinline__ void load_raw_fast(const __nv_bfloat16 *p, Raw &r, unsigned long long pol) {
        asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                     : "l"(p), "l"(pol));
    }
    static __device__ __forceinline__ void load_raw(const __nv_bfloat16 *p, Raw &r, int valid,
                                                    unsigned long long) {
        const unsigned short *q = reinterpret_cast<const unsigned short *>(p);
        unsigned e[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) e[i] = i < valid ? q[i] : 0u;
        r.x = e[0] | (e[1] << 16); r.y = e[2] | (e[3] << 16);
        r.z = e[4] | (e[5] << 16); r.w = e[6] | (e[7] << 16);
    }
    static __device__ __forceinline__ void unpack(const Raw &r, float v[8]) {
        const unsigned w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            v[2 * i] = __uint_as_float(w[i] << 16);
            v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
    }
    static __device__ __forceinline__ void load(const __nv_bfloat16 *p, float v[8], int valid, bool vec) {
        Raw r;
        if (vec && valid == 8) {
            r = *reinterpret_cast<const uint4 *>(p);
        } else {
            load_raw(p, r, valid, 0ull);
        }
        unpack(r, v);
    }
    static __device__ __forceinline__ void load_hint(const __nv_bfloat16 *p, float v[8], int valid, bool vec,
                                                     unsigned long long pol) {
        Raw r;
        if (vec && valid == 8)
            load_raw_fast(p, r, pol);
        else
            load_raw(p, r, valid, pol);
        unpack(r, v);
    }
    static __device__ __forceinline__ void store_hint(__nv_bfloat16 *p, const float v[8], int valid, bool vec,
                                                      unsigned long long pol) {
        unsigned short h[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) h[i] = f2bf(v[i]);
        if (vec && valid == 8) {
            const unsigned a = h[0] | (static_cast<unsigned>(h[1]) << 16), b = h[2] | (static_cast<unsigned>(h[3]) << 16);
            const unsigned c = h[4] | (static_cast<unsigned>(h[5]) << 16), d = h[6] | (static_cast<unsigned>(h[7]) << 16);
            asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(a), "r"(b),
                         "r"(c), "r"(d), "l"(pol)
                         : "memory");
        } else {
            unsigned short *q = reinterpret_cast<unsigned short *>(p);
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (i < valid) q[i] = h[i];
        }
    }
    static __device__ __forceinline__ float wire(float f) { return bf2f(f2bf(f)); }
    static __device__ __forceinline__ void store(__nv_bfloat16 *p, const float v[8], int valid, bool vec) {
        unsigned short h[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) h[i] = f2bf(v[i]);
        if (vec && valid == 8) {
            uint4 w;
            w.x = h[0] | (static_cast<unsigned>(h[1]) << 16); w.y = h[2] | (static_cast<unsigned>(h[3]) << 16);
            w.z = h[4] | (static_cast<unsigned>(h[5]) << 16); w.w = h[6] | (static_cast<unsigned>(h[7]) << 16);
            *reinterpret_cast<uint4 *>(p) = w;
        } else {
            unsigned short *q = reinterpret_cast<unsigned short *>(p);
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (i < valid) q[i] = h[i];
        }
    }
    static __device__ __forceinline__ void load_cg(const __nv_bfloat16 *p, float v[8], int valid, bool vec) {
        Raw r;
        if (vec && valid == 8) {
            r = __ldcg(reinterpret_cast<const uint4 *>(p));
        } else {
            const unsigned short *q = reinterpret_cast<const unsigned short *>(p);
            unsigned e[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) e[i] = i < valid ? __ldcg(q + i) : 0u;
            r.x = e[0] | (e[1] << 16); r.y = e[2] | (e[3] << 16);
            r.z = e[4] | (e[5] << 16); r.w = e[6] | (e[7] << 16);
        }
        unpack(r, v);
    }
};

// fp32 side buffers (window outboxes) next to 8-wide bf16 vectors: two float4
template <>
struct VecN<float, 8> {
    static __device__ __forceinline__ void load(const float *p, float v[8], int valid, bool vec) {
        Vec4<float>::load(p, v, valid < 4 ? valid : 4, vec);
        Vec4<float>::load(p + 4, v + 4, valid > 4 ? valid - 4 : 0, vec);
    }
    static __device__ __forceinline__ void store(float *p, const float v[8], int valid, bool vec) {
        Vec4<float>::store(p, v, valid < 4 ? valid : 4, vec);
        Vec4<float>::store(p + 4, v + 4, valid > 4 ? valid - 4 : 0, vec);
    }
    static __device__ __forceinline__ void load_hint(const float *p, float v[8], int valid, bool vec,
                                                     unsigned long long pol) {
        Vec4<float>::load_hint(p, v, valid < 4 ? valid : 4, vec, pol);
        Vec4<float>::load_hint(p + 4, v + 4, valid > 4 ? valid - 4 : 0, vec, pol);
    }
    static __device__ __forceinline__ void store_hint(float *p, const float v[8], int valid, bool vec,
                                                      unsigned long long pol) {
        Vec4<float>::store_hint(p, v, valid < 4 ? valid : 4, vec, pol);
        Vec4<float>::store_hint(p + 4, v + 4, valid > 4 ? valid - 4 : 0, vec, pol);
    }
};

// valid elements of the V-vector at offset e of a row with `rem` elements left
template <int V>
__device__ __forceinline__ int clamp_valid_v(long long rem, int e) {
    long long v = rem - e;
    return v >= V ? V : (v <= 0 ? 0 : static_cast<int>(v));
}

// Element index of vector j (0..kVecPerThread-1) of this thread inside a tile:
// consecutive threads touch consecutive 4-element vectors (coalesced).
__device__ __forceinline__ int tile_elem(int j) { return (j * kThreads + threadIdx.x) * kVec; }

__device__ __forceinline__ int clamp_valid(long long rem, int e) {
    long long v = rem - e;
    return v >= 4 ? 4 : (v <= 0 ? 0 : static_cast<int>(v));
}

// End-of-kernel protocol: the last CTA to finish runs `last()`.
template <typename F>
__device__ __forceinline__ void last_cta(Pad *pad, F last) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned int prev = atomicAdd(&pad->done_ctr, 1u);
        if (prev == gridDim.x - 1) {
            __threadfence();
            pad->done_ctr = 0;
            last();
        }
    }
}

}  // namespace bf
