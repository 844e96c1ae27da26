// nvlink_calib.cu -- calibration of the data movers the exchange kernels can use
// on a B200 box: local HBM copy, SM pull (128-bit peer
// loads), SM push (128-bit peer stores), TMA bulk copies from peer memory,
// copy-engine peer copies, all-pairs concurrent traffic, and the flag round-trip
// latency over NVLink.  One process drives every GPU (cudaDeviceEnablePeerAccess
// gives the same NVLink path as the CUDA-IPC mappings of the library).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlink_calib tools/nvlink_calib.cu
//   tools/nvlink_calib [MiB per buffer, default 1024]
//
// Output: one JSON object per line {"test", "gpus", "grid", "unroll", "gbs", ...};
// GB/s counts the bytes that cross the link (or, for local tests, read + write).
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

// dst[i] = src[i] with U independent 16-byte loads in flight per thread.
template <int U>
__global__ void __launch_bounds__(256) copy_v4(const float4 *__restrict__ src, float4 *__restrict__ dst, size_t n) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcg(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
    }
    for (; i < n; i += stride) dst[i] = __ldcg(src + i);
}

// y[i] = a*x[i] + b*p[i]: the combine shape (local read + peer read + local write)
template <int U>
__global__ void __launch_bounds__(256) axpy_v4(const float4 *__restrict__ x, const float4 *__restrict__ peer,
                                               float4 *__restrict__ y, size_t n) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        float4 a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            a[u] = __ldcg(x + i + u * stride);
            b[u] = __ldcg(peer + i + u * stride);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            y[i + u * stride] = make_float4(0.5f * a[u].x + 0.5f * b[u].x, 0.5f * a[u].y + 0.5f * b[u].y,
                                            0.5f * a[u].z + 0.5f * b[u].z, 0.5f * a[u].w + 0.5f * b[u].w);
    }
}

// TMA bulk copy: each CTA streams CHUNK-byte pieces src -> smem -> dst with a
// 2-stage ring (cp.async.bulk global->shared, then shared->global).
__device__ __forceinline__ unsigned su32(const void *p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(32) tma_copy(const char *src, char *dst, size_t bytes) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) unsigned long long bar[STAGES];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < STAGES; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const size_t nchunks = bytes / CHUNK;
    unsigned phase[STAGES] = {};
    size_t c = blockIdx.x;
    // prologue
    for (int s = 0; s < STAGES && c + s * gridDim.x < nchunks; ++s) {
        const size_t cc = c + s * gridDim.x;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(CHUNK)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(sm + s * CHUNK)),
                     "l"(src + cc * CHUNK), "r"(CHUNK), "r"(su32(&bar[s]))
                     : "memory");
    }
    int s = 0;
    for (size_t cc = c; cc < nchunks; cc += gridDim.x) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                su32(&bar[s])),
            "r"(phase[s])
            : "memory");
        phase[s] ^= 1;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + cc * CHUNK),
                     "r"(su32(sm + s * CHUNK)), "r"(CHUNK)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        const size_t nx = cc + static_cast<size_t>(STAGES) * gridDim.x;
        if (nx < nchunks) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // smem stage free again
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(CHUNK)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(sm + s * CHUNK)),
                "l"(src + nx * CHUNK), "r"(CHUNK), "r"(su32(&bar[s]))
                : "memory");
        }
        s = (s + 1) % STAGES;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Flag ping-pong: side 0 writes ping=i to the peer and waits for pong=i.
__global__ void pingpong(volatile unsigned long long *my_flag, unsigned long long *peer_flag, int iters, int side) {
    for (int i = 1; i <= iters; ++i) {
        if (side == 0) {
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer_flag), "l"((unsigned long long)i) : "memory");
            unsigned long long v;
            do {
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flag) : "memory");
            } while (v < (unsigned long long)i);
        } else {
            unsigned long long v;
            do {
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flag) : "memory");
            } while (v < (unsigned long long)i);
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer_flag), "l"((unsigned long long)i) : "memory");
        }
    }
}

// Fence cost under load: warps 0..7 stream (local HBM copy, or pull from a peer
// when `peer` != nullptr); warp 8 lane 0 times `iters` fences of kind `kind`
// (0 fence.acq_rel.sys, 1 fence.acq_rel.gpu, 2 st.release.sys of a flag, 3 none).
// Streaming warps with self_fence != 0 fence (same kind) after every 16 vectors
// and record their own fence time in out[2].
__global__ void __launch_bounds__(288) fence_cost(const float4 *src, float4 *dst, size_t n, int kind, int iters,
                                                  unsigned long long *out, unsigned long long *flag, int self_fence) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ volatile int stop;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    auto fence = [&](int k) {
        if (k == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
        else if (k == 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        else if (k == 2) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag + blockIdx.x), "l"(1ull) : "memory");
    };
    if (warp == 8) {
        if (lane == 0) {
            unsigned long long tot = 0;
            for (int i = 0; i < iters; ++i) {
                unsigned long long t0, t1;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
                fence(kind);
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
                tot += t1 - t0;
                __nanosleep(2000);
            }
            atomicAdd(&out[0], tot);
            atomicAdd(&out[1], (unsigned long long)iters);
            stop = 1;
        }
        return;
    }
    const size_t stride = static_cast<size_t>(gridDim.x) * 256;
    size_t i = static_cast<size_t>(blockIdx.x) * 256 + threadIdx.x;
    unsigned long long ft = 0, fc = 0;
    int cnt = 0;
    while (!stop) {
        for (int r = 0; r < 16 && i < n; ++r, i += stride) dst[i] = __ldcg(src + i);
        if (i >= n) i = static_cast<size_t>(blockIdx.x) * 256 + threadIdx.x;
        if (self_fence && ++cnt % 1 == 0) {
            unsigned long long t0, t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            fence(kind);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            ft += t1 - t0;
            ++fc;
        }
    }
    if (self_fence && lane == 0) {
        atomicAdd(&out[2], ft);
        atomicAdd(&out[3], fc);
    }
}

static int g_sms = 148;

struct Timer {
    std::vector<cudaEvent_t> a, b;
    explicit Timer(int n) : a(n), b(n) {
        for (int d = 0; d < n; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaEventCreate(&a[d]));
            CK(cudaEventCreate(&b[d]));
        }
    }
};

template <typename F>
static double time_on(int ndev, const int *devs, F launch, int reps = 5) {
    // launch(d) enqueues the work of device devs[d] on its default stream; returns max ms over devices
    std::vector<cudaEvent_t> e0(ndev), e1(ndev);
    for (int d = 0; d < ndev; ++d) {
        CK(cudaSetDevice(devs[d]));
        CK(cudaEventCreate(&e0[d]));
        CK(cudaEventCreate(&e1[d]));
    }
    double best = 1e30;
    for (int r = 0; r < reps + 1; ++r) {
        for (int d = 0; d < ndev; ++d) {
            CK(cudaSetDevice(devs[d]));
            CK(cudaDeviceSynchronize());
        }
        for (int d = 0; d < ndev; ++d) {
            CK(cudaSetDevice(devs[d]));
            CK(cudaEventRecord(e0[d]));
            launch(d);
            CK(cudaEventRecord(e1[d]));
        }
        double worst = 0;
        for (int d = 0; d < ndev; ++d) {
            CK(cudaSetDevice(devs[d]));
            CK(cudaEventSynchronize(e1[d]));
            CK(cudaGetLastError());
            float ms;
            CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
            worst = ms > worst ? ms : worst;
        }
        if (r > 0 && worst < best) best = worst;   // first rep is a warm-up
    }
    for (int d = 0; d < ndev; ++d) {
        CK(cudaSetDevice(devs[d]));
        cudaEventDestroy(e0[d]);
        cudaEventDestroy(e1[d]);
    }
    return best;
}

template <int U>
static void launch_copy(const void *s, void *d, size_t bytes, int grid) {
    copy_v4<U><<<grid, 256>>>(static_cast<const float4 *>(s), static_cast<float4 *>(d), bytes / 16);
}
static void launch_copy_u(int U, const void *s, void *d, size_t bytes, int grid) {
    switch (U) {
        case 1: launch_copy<1>(s, d, bytes, grid); break;
        case 2: launch_copy<2>(s, d, bytes, grid); break;
        case 4: launch_copy<4>(s, d, bytes, grid); break;
        default: launch_copy<8>(s, d, bytes, grid); break;
    }
}

int main(int argc, char **argv) {
    const size_t mib = argc > 1 ? strtoull(argv[1], nullptr, 10) : 1024;
    const size_t bytes = mib << 20;
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0));
    std::vector<char *> A(n), B(n), C(n);
    std::vector<unsigned long long *> F(n);
    for (int d = 0; d < n; ++d) {
        CK(cudaSetDevice(d));
        for (int q = 0; q < n; ++q)
            if (q != d) {
                int can = 0;
                CK(cudaDeviceCanAccessPeer(&can, d, q));
                if (can) CK(cudaDeviceEnablePeerAccess(q, 0));
            }
        CK(cudaMalloc(&A[d], bytes));
        CK(cudaMalloc(&B[d], bytes));
        CK(cudaMalloc(&C[d], bytes));
        CK(cudaMalloc(&F[d], 256));
        CK(cudaMemset(A[d], 1, bytes));
        CK(cudaMemset(B[d], 0, bytes));
        CK(cudaMemset(C[d], 0, bytes));
        CK(cudaMemset(F[d], 0, 256));
        CK(cudaFuncSetAttribute(tma_copy<4, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768));
        CK(cudaFuncSetAttribute(tma_copy<2, 65536>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 65536));
    }
    const double gb = static_cast<double>(bytes) / 1e9;
    auto emit = [&](const char *test, int gpus, int grid, int unroll, double ms, double link_bytes_gb) {
        printf("{\"test\": \"%s\", \"gpus\": %d, \"grid\": %d, \"unroll\": %d, \"mib\": %zu, \"ms\": %.4f, \"gbs\": %.1f}\n",
               test, gpus, grid, unroll, mib, ms, link_bytes_gb / (ms * 1e-3));
        fflush(stdout);
    };
    int d0[1] = {0};

    // ---- local HBM copy (read + write bytes) ----
    for (int U : {1, 4, 8})
        for (int gm : {1, 2, 4, 8}) {
            const int grid = g_sms * gm;
            double ms = time_on(1, d0, [&](int) { launch_copy_u(U, A[0], B[0], bytes, grid); });
            emit("hbm_copy", 1, grid, U, ms, 2 * gb);
        }
    if (n < 2) return 0;
    int d01[2] = {0, 1};

    // ---- pull: GPU0 loads GPU1's buffer (link bytes = buffer) ----
    for (int U : {1, 2, 4, 8})
        for (int gm : {1, 2, 4, 8}) {
            const int grid = g_sms * gm;
            double ms = time_on(1, d0, [&](int) { launch_copy_u(U, A[1], B[0], bytes, grid); });
            emit("pull_1to1", 1, grid, U, ms, gb);
        }
    // ---- push: GPU0 stores into GPU1's buffer ----
    for (int U : {1, 4, 8})
        for (int gm : {1, 2, 4, 8}) {
            const int grid = g_sms * gm;
            double ms = time_on(1, d0, [&](int) { launch_copy_u(U, A[0], B[1], bytes, grid); });
            emit("push_1to1", 1, grid, U, ms, gb);
        }
    // ---- combine shape: y0 = .5 x0 + .5 x1(peer) ----
    for (int gm : {2, 4, 8}) {
        const int grid = g_sms * gm;
        double ms = time_on(1, d0, [&](int) {
            axpy_v4<4><<<grid, 256>>>(reinterpret_cast<const float4 *>(A[0]), reinterpret_cast<const float4 *>(A[1]),
                                      reinterpret_cast<float4 *>(B[0]), bytes / 16);
        });
        emit("axpy_pull_1to1", 1, grid, 4, ms, gb);
    }
    // ---- TMA bulk from peer memory ----
    for (int gm : {1, 2, 4}) {
        const int grid = g_sms * gm;
        double ms = time_on(1, d0, [&](int) { tma_copy<4, 32768><<<grid, 32, 4 * 32768>>>(A[1], B[0], bytes); });
        emit("tma_pull_1to1_4x32K", 1, grid, 4, ms, gb);
        if (gm <= 1) {
            ms = time_on(1, d0, [&](int) { tma_copy<2, 65536><<<grid, 32, 2 * 65536>>>(A[1], B[0], bytes); });
            emit("tma_pull_1to1_2x64K", 1, grid, 2, ms, gb);
        }
        ms = time_on(1, d0, [&](int) { tma_copy<4, 32768><<<grid, 32, 4 * 32768>>>(A[0], B[1], bytes); });
        emit("tma_push_1to1_4x32K", 1, grid, 4, ms, gb);
    }
    // ---- TMA chunk size sweep, both directions busy (the exchange case) ----
    CK(cudaSetDevice(1));
    CK(cudaFuncSetAttribute(tma_copy<16, 4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 4096));
    CK(cudaFuncSetAttribute(tma_copy<8, 8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8192));
    CK(cudaFuncSetAttribute(tma_copy<4, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384));
    CK(cudaSetDevice(0));
    CK(cudaFuncSetAttribute(tma_copy<16, 4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 4096));
    CK(cudaFuncSetAttribute(tma_copy<8, 8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8192));
    CK(cudaFuncSetAttribute(tma_copy<4, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384));
    for (int gm : {1, 2}) {
        const int grid = g_sms * gm;
        double ms = time_on(2, d01, [&](int d) { tma_copy<16, 4096><<<grid, 32, 16 * 4096>>>(A[1 - d], B[d], bytes); });
        emit("tma_pull_bidir_16x4K", 2, grid, 16, ms, gb);
        ms = time_on(2, d01, [&](int d) { tma_copy<8, 8192><<<grid, 32, 8 * 8192>>>(A[1 - d], B[d], bytes); });
        emit("tma_pull_bidir_8x8K", 2, grid, 8, ms, gb);
        ms = time_on(2, d01, [&](int d) { tma_copy<4, 16384><<<grid, 32, 4 * 16384>>>(A[1 - d], B[d], bytes); });
        emit("tma_pull_bidir_4x16K", 2, grid, 4, ms, gb);
        ms = time_on(2, d01, [&](int d) { tma_copy<4, 32768><<<grid, 32, 4 * 32768>>>(A[1 - d], B[d], bytes); });
        emit("tma_pull_bidir_4x32K", 2, grid, 4, ms, gb);
        ms = time_on(1, d0, [&](int) { tma_copy<16, 4096><<<grid, 32, 16 * 4096>>>(A[1], B[0], bytes); });
        emit("tma_pull_1to1_16x4K", 1, grid, 16, ms, gb);
    }
    // ---- copy engine ----
    {
        double ms = time_on(1, d0, [&](int) { CK(cudaMemcpyPeerAsync(B[0], 0, A[1], 1, bytes, 0)); });
        emit("ce_pull_1to1", 1, 0, 0, ms, gb);
        ms = time_on(1, d0, [&](int) { CK(cudaMemcpyPeerAsync(B[1], 1, A[0], 0, bytes, 0)); });
        emit("ce_push_1to1", 1, 0, 0, ms, gb);
    }
    // ---- bidirectional pull: both GPUs pull from each other at once ----
    for (int gm : {2, 4, 8}) {
        const int grid = g_sms * gm;
        double ms = time_on(2, d01, [&](int d) { launch_copy_u(4, A[1 - d], B[d], bytes, grid); });
        emit("pull_bidir_per_gpu", 2, grid, 4, ms, gb);
        ms = time_on(2, d01, [&](int d) { launch_copy_u(4, A[d], B[1 - d], bytes, grid); });
        emit("push_bidir_per_gpu", 2, grid, 4, ms, gb);
    }
    // ---- all GPUs pull from all others at once (each GPU: (n-1) x bytes/(n-1) in) ----
    if (n > 2) {
        std::vector<int> all(n);
        for (int d = 0; d < n; ++d) all[d] = d;
        const size_t part = (bytes / (n - 1)) & ~static_cast<size_t>(4095);
        for (int gm : {2, 4, 8}) {
            const int grid = g_sms * gm / (n - 1);
            double ms = time_on(n, all.data(), [&](int d) {
                for (int q = 1; q < n; ++q) {
                    const int src = (d + q) % n;
                    launch_copy_u(4, A[src] + (q - 1) * part, B[d] + (q - 1) * part, part, grid);
                }
            });
            emit("pull_all2all_per_gpu", n, grid, 4, ms, static_cast<double>(part) * (n - 1) / 1e9);
        }
        // ring pattern: every GPU pulls from d-1 only (one-peer shift)
        for (int gm : {2, 4}) {
            const int grid = g_sms * gm;
            double ms = time_on(n, all.data(), [&](int d) { launch_copy_u(4, A[(d + n - 1) % n], B[d], bytes, grid); });
            emit("pull_shift1_per_gpu", n, grid, 4, ms, gb);
        }
    }
    // ---- fence cost under load ----
    {
        unsigned long long *out;
        CK(cudaSetDevice(0));
        CK(cudaMalloc(&out, 64));
        const char *kn[] = {"fence.acq_rel.sys", "fence.acq_rel.gpu", "st.release.sys", "none"};
        const char *ld[] = {"idle", "hbm_copy", "nvlink_pull"};
        for (int load = 0; load < 3; ++load)
            for (int kind = 0; kind < 3; ++kind)
                for (int self = 0; self < 2; ++self) {
                    if (load == 0 && self) continue;
                    CK(cudaMemset(out, 0, 64));
                    const float4 *src = reinterpret_cast<const float4 *>(load == 2 ? A[1] : A[0]);
                    size_t nvec = load == 0 ? 0 : bytes / 16;
                    fence_cost<<<g_sms * 2, 288>>>(src, reinterpret_cast<float4 *>(B[0]), nvec, kind, 50, out,
                                                   reinterpret_cast<unsigned long long *>(C[0]), self);
                    CK(cudaDeviceSynchronize());
                    unsigned long long h[4];
                    CK(cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost));
                    printf("{\"test\": \"fence_cost\", \"fence\": \"%s\", \"load\": \"%s\", \"streamers_fence\": %d, "
                           "\"signal_warp_us\": %.3f, \"streamer_us\": %.3f}\n",
                           kn[kind], ld[load], self, h[1] ? h[0] / 1e3 / h[1] : 0.0, h[3] ? h[2] / 1e3 / h[3] : 0.0);
                    fflush(stdout);
                }
        CK(cudaFree(out));
    }
    // ---- flag round trip (GPU0 <-> GPU1) ----
    {
        const int iters = 10000;
        cudaStream_t s1;
        CK(cudaSetDevice(1));
        CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
        for (int rep = 0; rep < 2; ++rep) {
            for (int d = 0; d < 2; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaMemset(F[d], 0, 256));
                CK(cudaDeviceSynchronize());
            }
            cudaEvent_t e0, e1;
            CK(cudaSetDevice(1));
            pingpong<<<1, 1, 0, s1>>>(F[1], F[0], iters, 1);
            CK(cudaSetDevice(0));
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            CK(cudaEventRecord(e0));
            pingpong<<<1, 1>>>(F[0], F[1], iters, 0);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            CK(cudaSetDevice(1));
            CK(cudaStreamSynchronize(s1));
            if (rep == 1)
                printf("{\"test\": \"flag_round_trip\", \"gpus\": 2, \"us\": %.3f}\n", ms * 1e3 / iters);
        }
    }
    return 0;
}
