// runtime.cu -- host runtime behind the C ABI (include/bluefog_b200.h):
// context and symmetric heap, CUDA-IPC bootstrap, topology / weight manager
// (P:334-382), argument validation (P:381 footnote), schedules,
// window registry, and the launchers of the sm_100a kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstddef>
#include <map>
#include <string>
#include <vector>

#include "bf_internal.h"

using namespace bf;

namespace {

thread_local std::string g_last_error;

bf_status fail(bf_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

#define CU(call)                                                                               \
    do {                                                                                       \
        cudaError_t _e = (call);                                                               \
        if (_e != cudaSuccess)                                                                 \
            return fail(BF_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e), \
                        __FILE__, __LINE__);                                                   \
    } while (0)

constexpr uint32_t kBlobMagic = 0xBF0B200u;

struct Blob {
    uint32_t magic;
    int proc, nprocs, k;
    uint64_t heap_bytes;
    cudaIpcMemHandle_t handle;
};

struct WinSide {
    std::vector<int> in, out;   // ascending global ranks
};

struct Window {
    std::string name;
    void *x = nullptr;
    size_t count = 0;
    int dtype = 0, with_p = 0, zero_init = 0;
    int ef = 0;                 // error feedback of the bf16 wire rounding (R24)
    int maxdin = 1, maxdout = 1;
    std::vector<WinSide> side;  // per global agent
    WinParams base{};           // offsets filled at creation
    size_t alloc_begin = 0, alloc_end = 0;
};

}  // namespace

struct bf_ctx {
    int proc = 0, nprocs = 1, k = 1, n = 1, device = 0;
    size_t heap_bytes = 0, heap_used = 0;
    char *heap = nullptr;
    unsigned long long peer_base[kMaxP] = {};
    char *peer_opened[kMaxP] = {};
    bool connected = false;
    bool poisoned = false;
    bf_status fault = BF_OK;
    volatile unsigned int *h_err = nullptr;   // host view
    unsigned int *d_err = nullptr;            // device view of the same word
    unsigned long long timeout_ns = 10ull * 1000 * 1000 * 1000;
    std::vector<double> W;                    // n*n
    int machine_L = 0, n_machines = 0;
    std::vector<double> WM;
    int sched_kind = 0, sched_L = 1;
    int topo_check = 1;
    int exch_kernel = 3;                      // BF_EXCH: chunk | fused (default)
    int chunk_tiles = 0;                      // BF_CHUNK_TILES; 0 = 256 on one GPU, 1024 across GPUs
    unsigned long long ccnt_off = 0, cflag_off = 0, prog_off = 0;
    // exchange region
    size_t exch_cap = 0;                      // bytes per agent per parity
    size_t exch_begin = 0, exch_top = 0;      // heap range of exchange (+ hierarchical) regions
    unsigned long long slot_off = 0, ready_off = 0;
    int ready_stride = 0;
    // hierarchical region
    bool hier_ready = false;
    int hier_L = 0;
    size_t hier_begin = 0, hier_top = 0;
    unsigned long long b_off = 0, c_off = 0, fb_off = 0, fc_off = 0, bc_agent_stride = 0, bc_parity_stride = 0;
    // staging for host pointers
    void *stage_x = nullptr, *stage_g = nullptr;
    size_t stage_x_bytes = 0, stage_g_bytes = 0;
    std::map<std::string, Window> windows;
    unsigned long long bar_epoch = 0;
    unsigned long long launches = 0;
    unsigned long long *stats = nullptr;      // BF_STATS=1: per-CTA diagnostics of the fused kernel
    int hier_mode = 0;                        // BF_HIER: 0 auto, 1 staged (always), 2 fused (also across GPUs)
    int xfer = 1;                             // BF_XFER: 1 push (default across GPUs), 0 pull, 2 push_all (tuning)
    unsigned long long inbox_off = 0, pflag_off = 0;   // push inboxes [n][2][cap] + progress words (0: none)
    unsigned long long ll_off = 0;            // tagged-word inboxes [n][2][ll_cap] u64 (small messages; 0: none)
    // elements per agent up to which tagged words are used: BF_LL_CAP, default 262144 (1 MB
    // fp32; measured crossover at N = 2: 1 MB 16.9 vs 19.9 us pushed, 4 MB 30.4 vs 27.7 us)
    long long ll_cap_req = 262144, ll_cap = 0;
    // NVLS (bf_hier_set_multicast): this process's copy of a multicast-backed fp32 buffer
    // [2][nvls_cap] of its machine's group, the multicast address, and machine flags
    float *nvls_uc = nullptr;
    unsigned long long nvls_mc = 0, nflag_off = 0;
    long long nvls_cap = 0;
    int nvls_L = 0;
    // NVLS only pays when a machine spans enough processes: measured at N = 4, one machine of
    // 4 GPUs 0.399 ms (NVLS) vs 0.522 ms (per-process partials pushed); machines of 2 GPUs
    // 0.527 / 0.564 vs 0.516 / 0.533 ms.  BF_NVLS_MIN_P overrides.
    int nvls_min_p = 4;
    int ll = 1;                               // BF_LL=0 turns the small-message path off
    int max_ctas = 0;                         // bf_set_max_ctas: grid cap of the exchange kernels (0 = all SMs)
    // host copy of the schedule round (advanced with every schedule-mode exchange call):
    // only picks the kernel of a K = 4 round; the device counter drives the schedule
    unsigned long long host_round = 0;
    bool win_ef = false;                      // BF_WIN_EF=1: new windows start with error feedback on
    // stream order across calls: every call of a context reads and advances the same
    // device state (epoch, round, slots, progress words), so a call issued on another
    // stream than the previous one first waits for the previous stream's work
    cudaStream_t last_stream = nullptr;
    bool have_last = false;
    cudaEvent_t order_ev = nullptr;
};

bf_status bf_barrier_internal(bf_ctx *c);

namespace {

bf_status check_ctx(bf_ctx *c, bool need_connected = true) {
    if (!c) return fail(BF_ERR_ARG, "null context");
    if (c->poisoned) return fail(BF_ERR_STATE, "context poisoned by an earlier device fault (%d)", c->fault);
    if (c->h_err && *c->h_err) {
        c->poisoned = true;
        c->fault = static_cast<bf_status>(*c->h_err);
        return fail(BF_ERR_STATE, "device fault %d latched (timeout or topology mismatch)", c->fault);
    }
    if (need_connected && !c->connected) return fail(BF_ERR_STATE, "bf_connect_peers has not been called");
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != c->device) cudaSetDevice(c->device);
    return BF_OK;
}

// Serialise this call after the context's previous call when they are issued on
// different streams (a non-blocking call on a side stream followed by any other
// call).  Same stream: nothing to do (stream order).  Inside a CUDA
// graph capture the captured dependencies fix the order, so nothing is recorded.
void order_stream(bf_ctx *c, cudaStream_t st) {
    if (c->have_last && st != c->last_stream && c->order_ev) {
        cudaStreamCaptureStatus a = cudaStreamCaptureStatusNone, b = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &a) == cudaSuccess && cudaStreamIsCapturing(c->last_stream, &b) == cudaSuccess &&
            a == cudaStreamCaptureStatusNone && b == cudaStreamCaptureStatusNone) {
            if (cudaEventRecord(c->order_ev, c->last_stream) == cudaSuccess) cudaStreamWaitEvent(st, c->order_ev, 0);
        }
        cudaGetLastError();   // a stream the caller destroyed since: nothing left to wait for
    }
    c->last_stream = st;
    c->have_last = true;
}

bf_status heap_alloc(bf_ctx *c, size_t bytes, unsigned long long *off) {
    size_t start = (c->heap_used + kAlign - 1) / kAlign * kAlign;
    bytes = (bytes + kAlign - 1) / kAlign * kAlign;
    if (start + bytes > c->heap_bytes)
        return fail(BF_ERR_NOMEM, "symmetric heap exhausted: need %zu more bytes (heap %zu, used %zu)", bytes,
                    c->heap_bytes, c->heap_used);
    CU(cudaMemset(c->heap + start, 0, bytes));
    c->heap_used = start + bytes;
    *off = start;
    return BF_OK;
}

Geometry make_geo(bf_ctx *c, size_t count) {
    Geometry g{};
    g.k = c->k;
    g.n = c->n;
    g.me = c->proc;
    g.nprocs = c->nprocs;
    g.count = static_cast<long long>(count);
    g.T = static_cast<int>((count + kTile - 1) / kTile);
    g.vec_ok = 0;
    g.timeout_ns = c->timeout_ns;
    for (int q = 0; q < kMaxP; ++q) g.peer_base[q] = c->peer_base[q];
    g.host_err = reinterpret_cast<volatile unsigned int *>(c->d_err);
    return g;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// A newly allocated (and zeroed) symmetric region becomes visible to the peers
// only after every process has zeroed its copy: peers read our progress words and
// flags, and an unzeroed reused region holds stale data that would read as
// "published".  Zeroing finished on this device, then a barrier (collective: the
// callers make the same allocation on every process).
bf_status publish_region(bf_ctx *c) {
    if (c->nprocs == 1) return BF_OK;
    CU(cudaDeviceSynchronize());
    bf_status s = bf_barrier_internal(c);
    if (s) return s;
    CU(cudaDeviceSynchronize());
    return BF_OK;
}

// Exchange region: double-buffered slots + per-tile ready flags of every local
// agent.  Grows on demand (collective: every process makes the same call):
// quiesce all processes first, then release the old region if it is on top of
// the heap (otherwise it is abandoned) and allocate the new one.
bf_status ensure_exchange(bf_ctx *c, size_t bytes_per_agent) {
    if (c->exch_cap >= bytes_per_agent && c->exch_cap) return BF_OK;
    size_t tile_bytes = static_cast<size_t>(kTile) * 4;
    size_t cap = (bytes_per_agent + tile_bytes - 1) / tile_bytes * tile_bytes;
    if (cap == 0) cap = tile_bytes;
    if (c->exch_cap) {
        CU(cudaDeviceSynchronize());
        bf_status s = bf_barrier_internal(c);
        if (s) return s;
        CU(cudaDeviceSynchronize());
        if (c->heap_used == c->exch_top) c->heap_used = c->exch_begin;
        c->hier_ready = false;
        cap = std::max(cap, 2 * c->exch_cap);
    }
    const size_t begin = c->heap_used;
    unsigned long long slot_off, ready_off;
    bf_status s = heap_alloc(c, static_cast<size_t>(c->k) * 2 * cap, &slot_off);
    if (s) return s;
    const int tmax = static_cast<int>(cap / (static_cast<size_t>(kTile) * 2));
    s = heap_alloc(c, static_cast<size_t>(c->k) * tmax * 8, &ready_off);
    if (s) return s;
    unsigned long long ccnt_off, cflag_off;
    if ((s = heap_alloc(c, static_cast<size_t>(tmax) * 4, &ccnt_off))) return s;
    if ((s = heap_alloc(c, static_cast<size_t>(tmax) * 8, &cflag_off))) return s;
    c->ccnt_off = ccnt_off;
    c->cflag_off = cflag_off;
    if ((s = heap_alloc(c, static_cast<size_t>(kMaxGrid) * 8, &c->prog_off))) return s;
    // push inboxes (cross-GPU fused kernel at K = 1, 2): one double-buffered inbox per
    // source agent in every reader's heap.  Optional: without room the pull kernel runs.
    c->inbox_off = c->pflag_off = c->ll_off = c->nflag_off = 0;
    if (c->nprocs > 1) {   // NVLS machine flags (hier_nvls.cu), small
        unsigned long long off;
        if (c->heap_used + static_cast<size_t>(kMaxP) * kMaxGrid * 8 + kAlign <= c->heap_bytes) {
            if ((s = heap_alloc(c, static_cast<size_t>(kMaxP) * kMaxGrid * 8, &off))) return s;
            c->nflag_off = off;
        }
    }
    if (c->nprocs > 1 && c->ll && (c->k == 1 || c->k == 2 || c->k == 4)) {   // small-message tagged inboxes
        // (the threshold shrinks to 32768 elements when the heap has no room for the default)
        for (long long cap_try : {c->ll_cap_req, std::min(c->ll_cap_req, kLLCap)}) {
            const size_t llb = static_cast<size_t>(c->n) * 2 * static_cast<size_t>(cap_try) * 8;
            if (c->heap_used + llb + kAlign > c->heap_bytes) continue;
            unsigned long long off;
            if ((s = heap_alloc(c, llb, &off))) return s;
            c->ll_off = off;
            c->ll_cap = cap_try;
            break;
        }
    }
    if (c->nprocs > 1 && c->xfer && (c->k == 1 || c->k == 2 || c->k == 4)) {
        const size_t need = static_cast<size_t>(c->n) * 2 * cap + static_cast<size_t>(kMaxP) * kMaxGrid * 8 + 2 * kAlign;
        if (c->heap_used + need <= c->heap_bytes) {
            unsigned long long ib, pf;
            if ((s = heap_alloc(c, static_cast<size_t>(c->n) * 2 * cap, &ib))) return s;
            if ((s = heap_alloc(c, static_cast<size_t>(kMaxP) * kMaxGrid * 8, &pf))) return s;
            c->inbox_off = ib;
            c->pflag_off = pf;
        }
    }
    c->exch_cap = cap;
    c->slot_off = slot_off;
    c->ready_off = ready_off;
    c->ready_stride = tmax;
    c->exch_begin = begin;
    c->exch_top = c->heap_used;
    return publish_region(c);
}

bool is_finite_w(double v) { return std::isfinite(v); }

// Validate one local view against P:381's four configurations.
bf_status validate_view(const bf_ctx *c, int gid, const bf_weights &w, bool allow_src, bool allow_dst,
                        int n_ranks) {
    const bool has_self = !std::isnan(w.self_weight);
    const bool has_src = w.n_src >= 0, has_dst = w.n_dst >= 0;
    if (!has_self)
        return fail(BF_ERR_ARG, "agent %d: self_weight is required with src/dst weights (P:381 footnote)", gid);
    if (!has_src && !has_dst)
        return fail(BF_ERR_ARG, "agent %d: self_weight alone is not one of the four valid configurations (P:381)",
                    gid);
    if (has_src && !allow_src) return fail(BF_ERR_ARG, "agent %d: src_weights not accepted here", gid);
    if (has_dst && !allow_dst) return fail(BF_ERR_ARG, "agent %d: dst_weights not accepted here", gid);
    if (!is_finite_w(w.self_weight)) return fail(BF_ERR_ARG, "agent %d: non-finite self_weight", gid);
    if (w.n_src > kMaxS || w.n_dst > kMaxS)
        return fail(BF_ERR_UNSUPPORTED, "agent %d: more than %d declared neighbours", gid, kMaxS);
    for (int pass = 0; pass < 2; ++pass) {
        const int nn = pass ? w.n_dst : w.n_src;
        const int *r = pass ? w.dst_ranks : w.src_ranks;
        const double *v = pass ? w.dst_weights : w.src_weights;
        if (nn > 0 && (!r || !v)) return fail(BF_ERR_ARG, "agent %d: null rank/weight array", gid);
        for (int q = 0; q < nn; ++q) {
            if (r[q] < 0 || r[q] >= n_ranks) return fail(BF_ERR_ARG, "agent %d: rank %d out of range", gid, r[q]);
            if (r[q] == gid) return fail(BF_ERR_ARG, "agent %d: self rank in %s list", gid, pass ? "dst" : "src");
            if (!is_finite_w(v[q])) return fail(BF_ERR_ARG, "agent %d: non-finite weight for rank %d", gid, r[q]);
            for (int q2 = 0; q2 < q; ++q2)
                if (r[q2] == r[q]) return fail(BF_ERR_ARG, "agent %d: duplicate rank %d", gid, r[q]);
        }
    }
    (void)c;
    return BF_OK;
}

// Static coefficients of local agent a from the global W (Eq. 5), sources in
// (i - j) mod n order.
bf_status static_row(const bf_ctx *c, int a, SrcTab &tab) {
    const int gid = c->proc * c->k + a, n = c->n;
    tab.self_w[a] = static_cast<float>(c->W[static_cast<size_t>(gid) * n + gid]);
    int cnt = 0;
    for (int d = 1; d < n; ++d) {
        const int j = ((gid - d) % n + n) % n;
        const double w = c->W[static_cast<size_t>(gid) * n + j];
        if (w == 0.0) continue;
        if (cnt >= kMaxS)
            return fail(BF_ERR_UNSUPPORTED, "agent %d has more than %d in-neighbours in the static topology", gid,
                        kMaxS);
        tab.src[a][cnt] = static_cast<unsigned char>(j);
        tab.coef[a][cnt] = static_cast<float>(w);
        ++cnt;
    }
    tab.nsrc[a] = static_cast<unsigned char>(cnt);
    return BF_OK;
}

bf_status fill_weights(bf_ctx *c, const bf_weights *weights, ExchParams &p) {
    memset(&p.tab, 0, sizeof(p.tab));
    memset(&p.dyn, 0, sizeof(p.dyn));
    p.check = c->topo_check;
    if (!weights) {
        if (c->sched_kind) {
            p.wmode = kWSchedule;
            p.sched_kind = c->sched_kind;
            p.sched_L = c->sched_L;
            return BF_OK;
        }
        p.wmode = kWStatic;
        for (int a = 0; a < c->k; ++a) {
            bf_status s = static_row(c, a, p.tab);
            if (s) return s;
        }
        return BF_OK;
    }
    p.wmode = kWDynamic;
    for (int a = 0; a < c->k; ++a) {
        const int gid = c->proc * c->k + a;
        const bf_weights &w = weights[a];
        bf_status s = validate_view(c, gid, w, true, true, c->n);
        if (s) return s;
        p.tab.self_w[a] = static_cast<float>(w.self_weight);
        p.dyn.has_src[a] = w.n_src >= 0;
        p.dyn.has_dst[a] = w.n_dst >= 0;
        if (w.n_src > 0) {
            for (int q = 0; q < w.n_src; ++q) {
                p.tab.src[a][q] = static_cast<unsigned char>(w.src_ranks[q]);
                p.tab.coef[a][q] = static_cast<float>(w.src_weights[q]);
            }
            p.tab.nsrc[a] = static_cast<unsigned char>(w.n_src);
        }
        if (w.n_dst > 0) {
            for (int q = 0; q < w.n_dst; ++q) {
                p.dyn.dst[a][q] = static_cast<unsigned char>(w.dst_ranks[q]);
                p.dyn.s[a][q] = static_cast<float>(w.dst_weights[q]);
            }
            p.dyn.ndst[a] = static_cast<unsigned char>(w.n_dst);
        }
    }
    return BF_OK;
}

bool is_host_ptr(const void *p) {
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return attr.type == cudaMemoryTypeHost || attr.type == cudaMemoryTypeUnregistered;
}

bf_status ensure_stage(void **buf, size_t *have, size_t need) {
    if (*have >= need) return BF_OK;
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    *have = 0;
    CU(cudaMalloc(buf, need));
    *have = need;
    return BF_OK;
}

std::vector<int> in_list(const bf_ctx *c, int i) {
    std::vector<int> v;
    for (int j = 0; j < c->n; ++j)
        if (j != i && c->W[static_cast<size_t>(i) * c->n + j] != 0.0) v.push_back(j);
    return v;
}
std::vector<int> out_list(const bf_ctx *c, int i) {
    std::vector<int> v;
    for (int j = 0; j < c->n; ++j)
        if (j != i && c->W[static_cast<size_t>(j) * c->n + i] != 0.0) v.push_back(j);
    return v;
}

int ceil_log2(int n) {
    int t = 0;
    while ((1 << t) < n) ++t;
    return t;
}

void topology_fill(int kind, int n, uint64_t k, double *W) {
    std::fill(W, W + static_cast<size_t>(n) * n, 0.0);
    if (n == 1) {
        W[0] = 1.0;
        return;
    }
    if (kind == 0) {                       // ring
        if (n == 2) {
            for (int q = 0; q < 4; ++q) W[q] = 0.5;
            return;
        }
        for (int i = 0; i < n; ++i)
            for (int d : {-1, 0, 1}) W[static_cast<size_t>(i) * n + ((i + d) % n + n) % n] = 1.0 / 3.0;
    } else if (kind == 1) {                // exponential-2 (R4)
        int deg = 0;
        for (int off = 1; off <= n - 1; off *= 2) ++deg;
        for (int i = 0; i < n; ++i) {
            W[static_cast<size_t>(i) * n + i] = 1.0 / (deg + 1);
            for (int off = 1; off <= n - 1; off *= 2)
                W[static_cast<size_t>(i) * n + ((i - off) % n + n) % n] += 1.0 / (deg + 1);
        }
    } else if (kind == 2) {                // fully connected
        for (size_t q = 0; q < static_cast<size_t>(n) * n; ++q) W[q] = 1.0 / n;
    } else {                               // one-peer exp-2 at round k (R5)
        const int off = 1 << static_cast<int>(k % static_cast<uint64_t>(ceil_log2(n)));
        for (int i = 0; i < n; ++i) {
            W[static_cast<size_t>(i) * n + i] = 0.5;
            W[static_cast<size_t>(i) * n + ((i - off) % n + n) % n] += 0.5;
        }
    }
}

}  // namespace

// ============================================================================
extern "C" {

const char *bf_last_error(void) { return g_last_error.c_str(); }

const char *bf_status_string(bf_status s) {
    switch (s) {
        case BF_OK: return "BF_OK";
        case BF_ERR_ARG: return "BF_ERR_ARG";
        case BF_ERR_STATE: return "BF_ERR_STATE";
        case BF_ERR_TOPOLOGY: return "BF_ERR_TOPOLOGY";
        case BF_ERR_CUDA: return "BF_ERR_CUDA";
        case BF_ERR_TIMEOUT: return "BF_ERR_TIMEOUT";
        case BF_ERR_NOMEM: return "BF_ERR_NOMEM";
        case BF_ERR_UNSUPPORTED: return "BF_ERR_UNSUPPORTED";
        case BF_ERR_WINDOW: return "BF_ERR_WINDOW";
    }
    return "BF_ERR_UNKNOWN";
}

size_t bf_ipc_blob_size(void) { return sizeof(Blob); }

bf_status bf_init(int proc_rank, int n_procs, int agents_per_proc, int cuda_device, size_t heap_bytes,
                  bf_ctx **out) {
    if (!out) return fail(BF_ERR_ARG, "null out");
    *out = nullptr;
    if (n_procs < 1 || n_procs > kMaxP) return fail(BF_ERR_UNSUPPORTED, "n_procs must be in [1, %d]", kMaxP);
    if (proc_rank < 0 || proc_rank >= n_procs) return fail(BF_ERR_ARG, "proc_rank out of range");
    if (agents_per_proc < 1 || agents_per_proc > kMaxK)
        return fail(BF_ERR_UNSUPPORTED, "agents_per_proc must be in [1, %d]", kMaxK);
    if (static_cast<long long>(n_procs) * agents_per_proc > kMaxN)
        return fail(BF_ERR_UNSUPPORTED, "at most %d agents", kMaxN);
    if (heap_bytes < kPadBytes + (1u << 20)) return fail(BF_ERR_ARG, "heap_bytes too small");
    CU(cudaSetDevice(cuda_device));
    int coop = 0;
    CU(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, cuda_device));
    if (!coop) return fail(BF_ERR_UNSUPPORTED, "device does not support cooperative launch");
    bf_ctx *c = new bf_ctx();
    c->proc = proc_rank;
    c->nprocs = n_procs;
    c->k = agents_per_proc;
    c->n = n_procs * agents_per_proc;
    c->device = cuda_device;
    c->heap_bytes = heap_bytes;
    if (const char *t = getenv("BF_TIMEOUT_MS")) c->timeout_ns = strtoull(t, nullptr, 10) * 1000000ull;
    if (const char *x = getenv("BF_EXCH"))
        c->exch_kernel = strcmp(x, "chunk") == 0 ? 2 : 3;
    if (const char *x = getenv("BF_CHUNK_TILES")) c->chunk_tiles = std::max(1, atoi(x));
    if (const char *x = getenv("BF_HIER")) c->hier_mode = strcmp(x, "staged") == 0 ? 1 : strcmp(x, "fused") == 0 ? 2 : 0;
    if (const char *x = getenv("BF_WIN_EF")) c->win_ef = atoi(x) != 0;
    if (const char *x = getenv("BF_LL")) c->ll = atoi(x) != 0;
    if (const char *x = getenv("BF_NVLS_MIN_P")) c->nvls_min_p = std::max(2, atoi(x));
    if (const char *x = getenv("BF_LL_CAP")) c->ll_cap_req = std::max(4LL, std::min(atoll(x), 1LL << 26)) / 4 * 4;
    if (const char *x = getenv("BF_XFER")) c->xfer = strcmp(x, "pull") == 0 ? 0 : (strcmp(x, "push_all") == 0 ? 2 : 1);
    if (const char *x = getenv("BF_STATS"))
        if (atoi(x) && cudaMalloc(&c->stats, static_cast<size_t>(kMaxGrid) * 8 * 8) == cudaSuccess)
            cudaMemset(c->stats, 0, static_cast<size_t>(kMaxGrid) * 8 * 8);
    cudaError_t e = cudaMalloc(&c->heap, heap_bytes);
    if (e != cudaSuccess) {
        delete c;
        return fail(BF_ERR_NOMEM, "cudaMalloc(%zu) failed: %s", heap_bytes, cudaGetErrorString(e));
    }
    cudaMemset(c->heap, 0, kPadBytes);
    c->heap_used = kPadBytes;
    void *h = nullptr;
    e = cudaHostAlloc(&h, 64, cudaHostAllocMapped);
    if (e != cudaSuccess) {
        cudaFree(c->heap);
        delete c;
        return fail(BF_ERR_CUDA, "cudaHostAlloc: %s", cudaGetErrorString(e));
    }
    memset(h, 0, 64);
    c->h_err = static_cast<volatile unsigned int *>(h);
    cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->d_err), h, 0);
    c->W.assign(static_cast<size_t>(c->n) * c->n, 1.0 / c->n);   // default: fully connected (R15)
    c->peer_base[proc_rank] = reinterpret_cast<unsigned long long>(c->heap);
    cudaEventCreateWithFlags(&c->order_ev, cudaEventDisableTiming);
    cudaDeviceSynchronize();
    *out = c;
    return BF_OK;
}

bf_status bf_get_ipc_blob(bf_ctx *c, void *blob, size_t *len) {
    bf_status s = check_ctx(c, false);
    if (s) return s;
    if (!blob || !len || *len < sizeof(Blob)) return fail(BF_ERR_ARG, "blob buffer too small");
    Blob b{};
    b.magic = kBlobMagic;
    b.proc = c->proc;
    b.nprocs = c->nprocs;
    b.k = c->k;
    b.heap_bytes = c->heap_bytes;
    if (c->nprocs > 1) CU(cudaIpcGetMemHandle(&b.handle, c->heap));
    memcpy(blob, &b, sizeof(Blob));
    *len = sizeof(Blob);
    return BF_OK;
}

bf_status bf_connect_peers(bf_ctx *c, const void *blobs, size_t blob_len) {
    bf_status s = check_ctx(c, false);
    if (s) return s;
    if (c->connected) return fail(BF_ERR_STATE, "already connected");
    if (c->nprocs > 1) {
        if (!blobs || blob_len < sizeof(Blob)) return fail(BF_ERR_ARG, "blobs required for n_procs > 1");
        for (int q = 0; q < c->nprocs; ++q) {
            Blob b;
            memcpy(&b, static_cast<const char *>(blobs) + q * blob_len, sizeof(Blob));
            if (b.magic != kBlobMagic || b.proc != q || b.nprocs != c->nprocs || b.k != c->k ||
                b.heap_bytes != c->heap_bytes)
                return fail(BF_ERR_ARG, "blob %d inconsistent (magic/proc/nprocs/agents/heap mismatch)", q);
            if (q == c->proc) continue;
            void *ptr = nullptr;
            CU(cudaIpcOpenMemHandle(&ptr, b.handle, cudaIpcMemLazyEnablePeerAccess));
            c->peer_opened[q] = static_cast<char *>(ptr);
            c->peer_base[q] = reinterpret_cast<unsigned long long>(ptr);
        }
    }
    c->connected = true;
    return bf_barrier(c, nullptr) == BF_OK ? (cudaDeviceSynchronize() == cudaSuccess ? BF_OK
                                                                                      : fail(BF_ERR_CUDA, "sync"))
                                           : BF_ERR_TIMEOUT;
}

bf_status bf_finalize(bf_ctx *c) {
    if (!c) return BF_OK;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (int q = 0; q < kMaxP; ++q)
        if (c->peer_opened[q]) cudaIpcCloseMemHandle(c->peer_opened[q]);
    if (c->heap) cudaFree(c->heap);
    if (c->stage_x) cudaFree(c->stage_x);
    if (c->stage_g) cudaFree(c->stage_g);
    if (c->stats) cudaFree(c->stats);
    if (c->h_err) cudaFreeHost(const_cast<unsigned int *>(c->h_err));
    if (c->order_ev) cudaEventDestroy(c->order_ev);
    delete c;
    return BF_OK;
}

int bf_size(const bf_ctx *c) { return c ? c->n : 0; }
int bf_rank(const bf_ctx *c) { return c ? c->proc * c->k : -1; }
int bf_local_agents(const bf_ctx *c) { return c ? c->k : 0; }
uint64_t bf_kernel_launches(const bf_ctx *c) { return c ? c->launches : 0; }

bf_status bf_exchange_stats(bf_ctx *c, uint64_t *out, size_t cap, int reset) {
    if (!c || !out) return fail(BF_ERR_ARG, "null argument");
    if (!c->stats) return fail(BF_ERR_STATE, "context was not created with BF_STATS=1");
    const size_t n = std::min(cap, static_cast<size_t>(kMaxGrid) * 8);
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(out, c->stats, n * 8, cudaMemcpyDeviceToHost));
    if (reset) CU(cudaMemset(c->stats, 0, static_cast<size_t>(kMaxGrid) * 8 * 8));
    return BF_OK;
}

// ---- topology ------------------------------------------------------------------
bf_status bf_topology_matrix(int kind, int n, uint64_t k, double *W) {
    if (!W || n < 1 || n > kMaxN || kind < 0 || kind > 3) return fail(BF_ERR_ARG, "bad topology request");
    topology_fill(kind, n, k, W);
    return BF_OK;
}

bf_status bf_schedule_one_peer_exp2(int n, int rank, uint64_t round, int *src, int *dst) {
    if (n < 1 || rank < 0 || rank >= n || !src || !dst) return fail(BF_ERR_ARG, "bad schedule request");
    const int tau = ceil_log2(n);
    if (tau == 0) {
        *src = *dst = -1;
        return BF_OK;
    }
    const int off = 1 << static_cast<int>(round % static_cast<uint64_t>(tau));
    *src = ((rank - off) % n + n) % n;
    *dst = (rank + off) % n;
    return BF_OK;
}

bf_status bf_schedule_inner_outer_exp2(int n, int local_size, int rank, uint64_t round, int *src, int *dst) {
    if (n < 1 || local_size < 1 || n % local_size || rank < 0 || rank >= n || !src || !dst)
        return fail(BF_ERR_ARG, "bad schedule request");
    sched_peers(2, n, local_size, round, rank, *src, *dst);
    return BF_OK;
}

bf_status bf_set_topology(bf_ctx *c, int n, const double *W) {
    bf_status s = check_ctx(c, false);
    if (s) return s;
    if (n != c->n || !W) return fail(BF_ERR_ARG, "topology size %d != %d agents", n, c->n);
    for (size_t q = 0; q < static_cast<size_t>(n) * n; ++q)
        if (!is_finite_w(W[q])) return fail(BF_ERR_ARG, "non-finite weight in W");
    for (int i = 0; i < n; ++i) {
        int d = 0;
        for (int j = 0; j < n; ++j) d += (j != i && W[static_cast<size_t>(i) * n + j] != 0.0);
        if (d > kMaxS) return fail(BF_ERR_UNSUPPORTED, "agent %d has %d > %d in-neighbours", i, d, kMaxS);
    }
    c->W.assign(W, W + static_cast<size_t>(n) * n);
    c->sched_kind = 0;
    return BF_OK;
}

// Static topology from local views (P:378-381 self/src/dst; Eq. 9):
// every process publishes its agents' views in its pad, a barrier, then every
// process reads all pads and assembles the same global W:
//   w_ii = self_weight_i;
//   j in src_i:            w_ij = r_ij * (s_ij if j lists i as destination, else 1)   (R1)
//   i gives no src list:   w_ij = s_ij for every j that lists i as destination        (push, R16)
// With the topology check on, a receiver with a src list must list exactly the
// senders that name it: else BF_ERR_TOPOLOGY on every process.
bf_status bf_set_topology_local(bf_ctx *c, const bf_weights *weights) {
    bf_status s = check_ctx(c);
    if (s) return s;
    if (!weights) return fail(BF_ERR_ARG, "null local views");
    std::vector<LocalView> mine(c->k);
    for (int a = 0; a < c->k; ++a) {
        const int gid = c->proc * c->k + a;
        const bf_weights &w = weights[a];
        if ((s = validate_view(c, gid, w, true, true, c->n))) return s;
        LocalView &v = mine[a];
        memset(&v, 0, sizeof(v));
        v.self_w = w.self_weight;
        v.nsrc = w.n_src;
        v.ndst = w.n_dst;
        for (int q = 0; q < w.n_src; ++q) {
            v.src[q] = static_cast<unsigned char>(w.src_ranks[q]);
            v.r[q] = w.src_weights[q];
        }
        for (int q = 0; q < w.n_dst; ++q) {
            v.dst[q] = static_cast<unsigned char>(w.dst_ranks[q]);
            v.s[q] = w.dst_weights[q];
        }
    }
    Pad *pad = reinterpret_cast<Pad *>(c->heap);
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(pad->lview, mine.data(), sizeof(LocalView) * c->k, cudaMemcpyHostToDevice));
    if ((s = publish_region(c))) return s;   // every pad written before anyone reads
    std::vector<LocalView> all(c->n);
    for (int q = 0; q < c->nprocs; ++q) {
        const Pad *pq = reinterpret_cast<const Pad *>(c->peer_base[q]);
        CU(cudaMemcpy(&all[static_cast<size_t>(q) * c->k], pq->lview, sizeof(LocalView) * c->k,
                      cudaMemcpyDeviceToHost));
    }
    if ((s = publish_region(c))) return s;   // nobody overwrites a pad another process still reads
    const int n = c->n;
    std::vector<double> W(static_cast<size_t>(n) * n, 0.0);
    auto sends = [&](int j, int i, double *sw) {   // does j list i as destination, with which s
        const LocalView &v = all[j];
        for (int q = 0; q < std::max(v.ndst, 0); ++q)
            if (v.dst[q] == i) {
                *sw = v.s[q];
                return true;
            }
        return false;
    };
    for (int i = 0; i < n; ++i) {
        const LocalView &v = all[i];
        W[static_cast<size_t>(i) * n + i] = v.self_w;
        if (v.nsrc >= 0) {
            for (int q = 0; q < v.nsrc; ++q) {
                double sw = 1.0;
                const int j = v.src[q];
                const bool pushed = sends(j, i, &sw);
                if (c->topo_check && all[j].ndst >= 0 && !pushed)
                    return fail(BF_ERR_TOPOLOGY, "agent %d lists %d as source, but %d does not send to %d (P:382)", i,
                                j, j, i);
                W[static_cast<size_t>(i) * n + j] = v.r[q] * (pushed ? sw : 1.0);
            }
            if (c->topo_check)
                for (int j = 0; j < n; ++j) {
                    double sw;
                    if (j == i || !sends(j, i, &sw)) continue;
                    bool listed = false;
                    for (int q = 0; q < v.nsrc; ++q) listed |= v.src[q] == j;
                    if (!listed)
                        return fail(BF_ERR_TOPOLOGY, "agent %d sends to %d, which does not list it as source (P:382)",
                                    j, i);
                }
        } else {
            for (int j = 0; j < n; ++j) {
                double sw;
                if (j != i && sends(j, i, &sw)) W[static_cast<size_t>(i) * n + j] = sw;
            }
        }
    }
    return bf_set_topology(c, n, W.data());
}

bf_status bf_set_machine_topology(bf_ctx *c, int local_size, int n_machines, const double *WM) {
    bf_status s = check_ctx(c, false);
    if (s) return s;
    if (local_size < 1 || n_machines < 1 || local_size * n_machines != c->n || !WM)
        return fail(BF_ERR_ARG, "machines (%d x %d) must tile the %d agents homogeneously (P:668)", n_machines,
                    local_size, c->n);
    for (int m = 0; m < n_machines; ++m) {
        int d = 0;
        for (int q = 0; q < n_machines; ++q) {
            if (!is_finite_w(WM[m * n_machines + q])) return fail(BF_ERR_ARG, "non-finite machine weight");
            d += (q != m && WM[m * n_machines + q] != 0.0);
        }
        if (d > kMaxS) return fail(BF_ERR_UNSUPPORTED, "machine %d has too many neighbours", m);
    }
    c->machine_L = local_size;
    c->n_machines = n_machines;
    c->WM.assign(WM, WM + static_cast<size_t>(n_machines) * n_machines);
    return BF_OK;
}

bf_status bf_in_neighbors(bf_ctx *c, int agent, int *ranks, int cap, int *n_out) {
    if (!c || agent < 0 || agent >= c->n || !n_out) return fail(BF_ERR_ARG, "bad agent");
    auto v = in_list(c, agent);
    *n_out = static_cast<int>(v.size());
    for (int q = 0; q < cap && q < *n_out; ++q) ranks[q] = v[q];
    return BF_OK;
}

bf_status bf_out_neighbors(bf_ctx *c, int agent, int *ranks, int cap, int *n_out) {
    if (!c || agent < 0 || agent >= c->n || !n_out) return fail(BF_ERR_ARG, "bad agent");
    auto v = out_list(c, agent);
    *n_out = static_cast<int>(v.size());
    for (int q = 0; q < cap && q < *n_out; ++q) ranks[q] = v[q];
    return BF_OK;
}

bf_status bf_set_dynamic_schedule(bf_ctx *c, int kind, uint64_t round0) {
    bf_status s = check_ctx(c);
    if (s) return s;
    if (kind < 0 || kind > 2) return fail(BF_ERR_ARG, "unknown schedule kind %d", kind);
    if (kind == 2 && !c->machine_L)
        return fail(BF_ERR_STATE, "inner-outer schedule needs bf_set_machine_topology (machine size)");
    c->sched_kind = kind;
    c->sched_L = kind == 2 ? c->machine_L : 1;
    c->host_round = round0;
    if (kind) {
        Pad *pad = reinterpret_cast<Pad *>(c->heap);
        order_stream(c, nullptr);
        CU(launch_set_u64(&pad->round, round0, nullptr));
        c->launches++;
        CU(cudaDeviceSynchronize());
    }
    return BF_OK;
}

bf_status bf_set_topology_check(bf_ctx *c, int enable) {
    if (!c) return fail(BF_ERR_ARG, "null context");
    c->topo_check = enable ? 1 : 0;
    return BF_OK;
}

bf_status bf_reserve(bf_ctx *c, size_t bytes_per_agent) {
    bf_status s = check_ctx(c);
    if (s) return s;
    return ensure_exchange(c, bytes_per_agent);
}

// ---- hot path ---------------------------------------------------------------
// K = 4 schedule rounds: push when every local agent's source sits on another process
// (measured at N = 2, one-peer: that round 0.69 ms pushed vs 0.75 pulled; rounds with 1-2
// remote sources of 4 run faster pulled).  Decided from the host copy of the round; in a
// captured CUDA graph the capture-time choice is replayed -- either kernel is correct for
// any round, the device counter drives the schedule.
static bool all_remote_round(const bf_ctx *c) {
    for (int a = 0; a < c->k; ++a) {
        int src, dst;
        sched_peers(c->sched_kind, c->n, c->sched_L, c->host_round, c->proc * c->k + a, src, dst);
        if (src < 0 || src / c->k == c->proc) return false;
    }
    return true;
}

struct GtArgs {                     // push-sum gradient tracking steps (MODE 4 / 5)
    int mode = 0;
    const float *g2 = nullptr;
    float *v = nullptr;
    float *x_out = nullptr;
};

static bf_status exchange_common(bf_ctx *c, const void *x, const void *g, void *y, void *shadow, size_t count,
                                 int x_kind, int g_kind, int wire_kind, int y_kind, float lr,
                                 const bf_weights *weights, cudaStream_t st, const void *awc_g = nullptr,
                                 const SrcTab *static_tab = nullptr, float *psi = nullptr,
                                 unsigned static_pub = 0, const GtArgs *gt = nullptr) {
    if (count == 0) return BF_OK;
    if (count > (1ull << 40)) return fail(BF_ERR_ARG, "count too large");
    ExchParams p;
    memset(&p, 0, sizeof(p));
    bf_status s = BF_OK;
    if (static_tab) {   // a W assembled by the caller (hierarchical: W_M (x) J_L/L)
        p.wmode = kWStatic;
        p.tab = *static_tab;
    } else {
        s = fill_weights(c, weights, p);
        if (s) return s;
    }
    const size_t wire_es = wire_kind == 0 ? 4 : 2;
    s = ensure_exchange(c, count * wire_es);
    if (s) return s;
    if ((count + kTile - 1) / kTile > static_cast<size_t>(c->ready_stride))
        return fail(BF_ERR_NOMEM, "too many tiles for the reserved exchange region");
    p.geo = make_geo(c, count);
    // rows of agent a start at a * count elements: 16-byte vectors need count to be a
    // multiple of the vector width (4 fp32, 8 bf16 elements per 16 bytes)
    const size_t vwidth = (x_kind == 1 || y_kind == 1) ? 8 : 4;
    p.geo.vec_ok = (count % vwidth == 0) && aligned16(x) && aligned16(y) && (!g || aligned16(g)) &&
                   (!shadow || aligned16(shadow));
    p.x_kind = x_kind;
    p.wire_kind = wire_kind;
    p.y_kind = y_kind;
    p.x = x;
    p.g = g;
    p.y = y;
    p.shadow = shadow;
    p.lr = lr;
    p.slot_off = c->slot_off;
    p.slot_agent_stride = 2 * c->exch_cap;
    p.slot_parity_stride = c->exch_cap;
    p.ready_off = c->ready_off;
    p.ready_stride = c->ready_stride;
    // kernel 3 (local-agent fused) is instantiated for k = 1, 2, 4, 8; other k use the chunked kernel
    p.kernel = c->exch_kernel == 3 && !fused_supported(c->k, c->nprocs) ? 2 : c->exch_kernel;
    if (static_tab) {
        p.pub_mask = c->nprocs > 1 ? static_pub : 0u;   // the caller knows who reads its agents
    } else if (p.wmode == kWStatic && c->nprocs > 1) {   // local agents whose x_half another process reads
        for (int a = 0; a < c->k; ++a) {
            const int gid = c->proc * c->k + a;
            for (int j = 0; j < c->n; ++j)
                if (j / c->k != c->proc && c->W[static_cast<size_t>(j) * c->n + gid] != 0.0) p.pub_mask |= 1u << a;
        }
    }
    if (awc_g) {
        p.awc = 1;
        p.g = awc_g;
        p.g_bf16 = g_kind == 1;
        p.lr = lr;
        p.geo.vec_ok = p.geo.vec_ok && aligned16(awc_g);
    }
    p.chunk_tiles = c->chunk_tiles ? c->chunk_tiles : (c->nprocs > 1 ? 1024 : 256);
    p.ccnt_off = c->ccnt_off;
    p.prog_off = c->prog_off;
    p.stats = c->stats;
    if (psi) {   // Exact-Diffusion: only the fused kernel implements MODE 3
        if (p.kernel != 3)
            return fail(BF_ERR_UNSUPPORTED, "Exact-Diffusion needs the fused exchange kernel (agents_per_proc 1, 2, 4 "
                                            "or 8 on one GPU)");
        if (!aligned16(psi)) p.geo.vec_ok = 0;
        p.psi = psi;
    }
    p.cflag_off = c->cflag_off;
    if (gt) {   // gradient tracking: only the fused kernel implements MODE 4 / 5
        if (p.kernel != 3)
            return fail(BF_ERR_UNSUPPORTED, "gradient tracking needs the fused exchange kernel (agents_per_proc 1, 2, "
                                            "4 or 8 on one GPU)");
        p.gt = gt->mode;
        p.g2 = gt->g2;
        p.gt_v = gt->v;
        p.x_out = gt->x_out;
        if (gt->g2 && !aligned16(gt->g2)) p.geo.vec_ok = 0;
        if (gt->x_out && !aligned16(gt->x_out)) p.geo.vec_ok = 0;
    }
    // cross-GPU push variant (exchange_push.cuh): static topologies and schedules at
    // K = 1, 2, when the inboxes fit in the heap; per-call views and the caller-assembled
    // hierarchical W keep the pull kernel
    // small messages across GPUs: tagged words, no fence, no progress word (exchange_ll.cuh)
    if (p.kernel == 3 && c->nprocs > 1 && c->ll_off && !static_tab && p.wmode != kWDynamic && !psi && !gt &&
        static_cast<long long>(count) <= c->ll_cap && (c->k == 1 || c->k == 2 || c->k == 4)) {
        p.ll = 1;
        p.ll_off = c->ll_off;
        p.ll_stride = static_cast<unsigned long long>(c->ll_cap) * 8;
        if (p.wmode == kWStatic)
            for (int a = 0; a < c->k; ++a) {
                const int gid = c->proc * c->k + a;
                for (int i = 0; i < c->n; ++i)
                    if (i / c->k != c->proc && c->W[static_cast<size_t>(i) * c->n + gid] != 0.0)
                        p.pushq[a] |= 1u << (i / c->k);
            }
    }
        // K = 4: push only for static W (measured at N = 2, 8 agents: exp-2 0.77 ms push vs
    // 1.18 pull; one-peer rounds with 1-2 remote sources of 4 run faster pulled, 0.50 vs 0.60)
    if (!p.ll && p.kernel == 3 && c->nprocs > 1 && c->inbox_off && !static_tab && p.wmode != kWDynamic &&
        (c->k == 1 || c->k == 2 ||
         (c->k == 4 && (p.wmode == kWStatic || c->xfer == 2 || (p.wmode == kWSchedule && all_remote_round(c)))))) {
        p.push = 1;
        p.inbox_off = c->inbox_off;
        p.inbox_agent_stride = 2 * c->exch_cap;
        p.inbox_parity_stride = c->exch_cap;
        p.pflag_off = c->pflag_off;
        if (p.wmode == kWStatic)
            for (int a = 0; a < c->k; ++a) {
                const int gid = c->proc * c->k + a;
                for (int i = 0; i < c->n; ++i)
                    if (i / c->k != c->proc && c->W[static_cast<size_t>(i) * c->n + gid] != 0.0)
                        p.pushq[a] |= 1u << (i / c->k);
            }
    }
    order_stream(c, st);
    CU(launch_exchange(p, x_kind, awc_g ? x_kind : g_kind, wire_kind, y_kind, g != nullptr, c->max_ctas, st));
    if (p.wmode == kWSchedule) c->host_round++;
    c->launches++;
    return BF_OK;
}

bf_status bf_neighbor_allreduce(bf_ctx *c, const void *x, void *y, size_t count, bf_dtype dtype,
                                const bf_weights *weights, void *stream) {
    bf_status s = check_ctx(c);
    if (s) return s;
    if (count == 0) return BF_OK;   // empty input: nothing to exchange, no kernel
    if (!x || !y) return fail(BF_ERR_ARG, "null tensor");
    if (dtype != BF_FLOAT32 && dtype != BF_BFLOAT16) return fail(BF_ERR_UNSUPPORTED, "dtype");
    return exchange_common(c, x, nullptr, y, nullptr, count, dtype, dtype, dtype, dtype, 0.f, weights,
                           static_cast<cudaStream_t>(stream));
}

bf_status bf_atc_step(bf_ctx *c, float *x, const void *g, bf_dtype g_dtype, size_t count, float lr, bf_dtype wire,
                      void *x_bf16_shadow, const bf_weights *weights, void *stream) {
    bf_status s = check_ctx(c);
    if (s) return s;
    if (count == 0) return BF_OK;   // empty input: nothing to exchange, no kernel
    if (!x || !g) return fail(BF_ERR_ARG, "null tensor");
    if ((g_dtype != BF_FLOAT32 && g_dtype != BF_BFLOAT16) || (wire != BF_FLOAT32 && wire != BF_BFLOAT16))
        return fail(BF_ERR_UNSUPPORTED, "dtype");
    if (!std::isfinite(lr)) return fail(BF_ERR_ARG, "non-finite lr");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t rows = static_cast<size_t>(c->k) * count;
    float *xd = x;
    const void *gd = g;
    const bool x_host = is_host_ptr(x), g_host = is_host_ptr(g);
    if (x_host || g_host) order_stream(c, st);
    if (x_host) {   // end-to-end path: stage the host tensors through device memory
        s = ensure_stage(&c->stage_x, &c->stage_x_bytes, rows * 4);
        if (s) return s;
        CU(cudaMemcpyAsync(c->stage_x, x, rows * 4, cudaMemcpyHostToDevice, st));
        xd = static_cast<float *>(c->stage_x);
    }
    if (g_host) {
        const size_t gb = rows * (g_dtype == BF_FLOAT32 ? 4 : 2);
        s = ensure_stage(&c->stage_g, &c->stage_g_bytes, gb);
        if (s) return s;
        CU(cudaMemcpyAsync(c->stage_g, g, gb, cudaMemcpyHostToDevice, st));
        gd = c->stage_g;
    }
    s = exchange_common(c, xd, gd, xd, x_bf16_shadow, count, 0, g_dtype, wire, 0, lr, weights, st);
    if (s) return s;
    if (x_host) CU(cudaMemcpyAsync(x, c->stage_x, rows * 4, cudaMemcpyDeviceToHost, st));
    return BF_OK;
}

bf_status bf_awc_step(bf_ctx *c, float *x, const void *g, bf_dtype g_dtype, size_t count, float lr,
                      const bf_weights *weights, void *stream) {
    bf_status s = check_ctx(c);
    if (s) return s;
    if (count == 0) return BF_OK;   // empty input: nothing to exchange, no kernel
    if (!x || !g) return fail(BF_ERR_ARG, "null tensor");
    if (g_dtype != BF_FLOAT32 && g_dtype != BF_BFLOAT16) return fail(BF_ERR_UNSUPPORTED, "dtype");
    if (!std::isfinite(lr)) return fail(BF_ERR_ARG, "non-finite lr");
    if (is_host_ptr(x) || is_host_ptr(g)) return fail(BF_ERR_ARG, "bf_awc_step takes device tensors");
    return exchange_common(c, x, nullptr, x, nullptr, count, 0, g_dtype, 0, 0, lr, weights,
                           static_cast<cudaStream_t>(stream), g);
}

bf_status bf_exact_diffusion_step(bf_ctx *c, float *x, const void *g, bf_dtype g_dtype, float *psi, size_t count,
                                  float lr, bf_dtype wire, const bf_weights *weights, void *stream) {
    bf_status s = check_ctx(c);
    if (s) return s;
    if (count == 0) return BF_OK;   // empty input: nothing to exchange, no kernel
    if (!x || !g || !psi) return fail(BF_ERR_ARG, "null tensor");
    if ((g_dtype != BF_FLOAT32 && g_dtype != BF_BFLOAT16) || (wire != BF_FLOAT32 && wire != BF_BFLOAT16))
        return fail(BF_ERR_UNSUPPORTED, "dtype");
    if (!std::isfinite(lr)) return fail(BF_ERR_ARG, "non-finite lr");
    if (is_host_ptr(x) || is_host_ptr(g) || is_host_ptr(psi))
        return fail(BF_ERR_ARG, "bf_exact_diffusion_step takes device tensors");
    return exchange_common(c, x, g, x, nullptr, count, 0, g_dtype, wire, 0, lr, weights,
                           static_cast<cudaStream_t>(stream), nullptr, nullptr, psi);
}

// Push-sum gradient tracking (appendix), one fused launch
// per partial averaging.
bf_status bf_gt_uv_step(bf_ctx *c, float *u, float *v, const float *y, float *x_out, size_t count, float lr,
                        bf_dtype wire, const bf_weights *weights, void *stream) {
    bf_status s = check_ctx(c);
    if (s) return s;
    if (count == 0) return BF_OK;
    if (!u || !v || !y || !x_out) return fail(BF_ERR_ARG, "null tensor");
    if (wire != BF_FLOAT32 && wire != BF_BFLOAT16) return fail(BF_ERR_UNSUPPORTED, "dtype");
    if (!std::isfinite(lr)) return fail(BF_ERR_ARG, "non-finite lr");
    if (is_host_ptr(u) || is_host_ptr(v) || is_host_ptr(y) || is_host_ptr(x_out))
        return fail(BF_ERR_ARG, "bf_gt_uv_step takes device tensors");
    GtArgs gt;
    gt.mode = 5;
    gt.v = v;
    gt.x_out = x_out;
    return exchange_common(c, u, y, u, nullptr, count, 0, 0, wire, 0, lr, weights, static_cast<cudaStream_t>(stream),
                           nullptr, nullptr, nullptr, 0, &gt);
}

bf_status bf_gt_y_step(bf_ctx *c, float *y, const float *g, const float *g_prev, size_t count, bf_dtype wire,
                       const bf_weights *weights, void *stream) {
    bf_status s = check_ctx(c);
    if (s) return s;
    if (count == 0) return BF_OK;
    if (!y || !g || !g_prev) return fail(BF_ERR_ARG, "null tensor");
    if (wire != BF_FLOAT32 && wire != BF_BFLOAT16) return fail(BF_ERR_UNSUPPORTED, "dtype");
    if (is_host_ptr(y) || is_host_ptr(g) || is_host_ptr(g_prev))
        return fail(BF_ERR_ARG, "bf_gt_y_step takes device tensors");
    GtArgs gt;
    gt.mode = 4;
    gt.g2 = g_prev;
    return exchange_common(c, y, g, y, nullptr, count, 0, 0, wire, 0, 0.f, weights, static_cast<cudaStream_t>(stream),
                           nullptr, nullptr, nullptr, 0, &gt);
}

// hmode 0: y = (W_M (x) J_L/L) x; 1 (H-ATC): x <- (W_M (x) J_L/L)(x - lr g);
// 2 (H-AWC): x <- (W_M (x) J_L/L) x - lr g.
static bf_status hier_common(bf_ctx *c, const void *x, void *y, size_t count, bf_dtype dtype, int hmode,
                             const void *g, bf_dtype g_dtype, float lr, const bf_weights *machine_weights,
                             void *stream) {
    bf_status s = check_ctx(c);
    if (s) return s;
    if (count == 0) return BF_OK;   // empty input: nothing to exchange, no kernel
    if (!x || !y || (hmode && !g)) return fail(BF_ERR_ARG, "null tensor");
    if (dtype != BF_FLOAT32 && dtype != BF_BFLOAT16) return fail(BF_ERR_UNSUPPORTED, "dtype");
    if (hmode && (g_dtype != BF_FLOAT32 && g_dtype != BF_BFLOAT16)) return fail(BF_ERR_UNSUPPORTED, "dtype");
    if (hmode && !std::isfinite(lr)) return fail(BF_ERR_ARG, "non-finite lr");
    if (hmode && (is_host_ptr(x) || is_host_ptr(g))) return fail(BF_ERR_ARG, "hierarchical steps take device tensors");
    if (!c->machine_L) return fail(BF_ERR_STATE, "bf_set_machine_topology has not been called");
    const int L = c->machine_L, NM = c->n_machines;
    HierParams p;
    memset(&p, 0, sizeof(p));
    // The hierarchical average is the plain mix with W = W_M (x) J_L / L (P:660,
    // R12).  When that W fits the fused exchange kernel (in-degree <= kMaxS,
    // agents_per_proc it is instantiated for) it is applied there: in registers
    // on one GPU (read x, write y), and across GPUs with the same pull pipeline
    // as any static W.  Otherwise (or BF_HIER=staged) the staged sliced kernel.
    int kron_deg = 0;
    if (!machine_weights) {
        for (int m = 0; m < NM; ++m) {
            int d = 0;
            for (int q = 0; q < NM; ++q) d += (q != m && c->WM[static_cast<size_t>(m) * NM + q] != 0.0);
            kron_deg = std::max(kron_deg, L - 1 + d * L);
        }
    } else {
        for (int a = 0; a < c->k; ++a) kron_deg = std::max(kron_deg, L - 1 + std::max(machine_weights[a].n_src, 0) * L);
    }
    // Across GPUs the Kronecker W pulls every remote agent of the machine
    // neighbourhood in full (L rows per machine instead of one slice average):
    // measured slower than the staged kernel at N = 2, so it
    // is used there only when forced (BF_HIER=fused).
    const bool as_mix = c->hier_mode != 1 && (c->nprocs == 1 || c->hier_mode == 2) && c->exch_kernel == 3 &&
                        fused_supported(c->k, c->nprocs) && kron_deg <= kMaxS;
    for (int a = 0; a < c->k; ++a) {
        const int gid = c->proc * c->k + a, m = gid / L;
        if (!machine_weights) {
            p.mtab.self_w[a] = static_cast<float>(c->WM[static_cast<size_t>(m) * NM + m]);
            int cnt = 0;
            for (int d = 1; d < NM; ++d) {
                const int q = ((m - d) % NM + NM) % NM;
                const double w = c->WM[static_cast<size_t>(m) * NM + q];
                if (w == 0.0) continue;
                p.mtab.src[a][cnt] = static_cast<unsigned char>(q);
                p.mtab.coef[a][cnt] = static_cast<float>(w);
                ++cnt;
            }
            p.mtab.nsrc[a] = static_cast<unsigned char>(cnt);
        } else {
            const bf_weights &w = machine_weights[a];
            s = validate_view(c, m, w, true, false, NM);
            if (s) return s;
            p.mtab.self_w[a] = static_cast<float>(w.self_weight);
            for (int q = 0; q < w.n_src; ++q) {
                p.mtab.src[a][q] = static_cast<unsigned char>(w.src_ranks[q]);
                p.mtab.coef[a][q] = static_cast<float>(w.src_weights[q]);
            }
            p.mtab.nsrc[a] = static_cast<unsigned char>(w.n_src > 0 ? w.n_src : 0);
        }
    }
    if (as_mix) {
        SrcTab tab;
        memset(&tab, 0, sizeof(tab));
        for (int a = 0; a < c->k; ++a) {
            const int gid = c->proc * c->k + a, m = gid / L;
            tab.self_w[a] = p.mtab.self_w[a] / static_cast<float>(L);
            int cnt = 0;
            auto add = [&](int mm, float w) {
                for (int l = 0; l < L; ++l) {
                    const int j = mm * L + l;
                    if (j == gid) continue;
                    tab.src[a][cnt] = static_cast<unsigned char>(j);
                    tab.coef[a][cnt] = w / static_cast<float>(L);
                    ++cnt;
                }
            };
            add(m, p.mtab.self_w[a]);   // the rest of the own machine
            for (int q = 0; q < p.mtab.nsrc[a]; ++q) add(p.mtab.src[a][q], p.mtab.coef[a][q]);
            tab.nsrc[a] = static_cast<unsigned char>(cnt);
        }
        // local agents another process reads: static machine topology -> from W_M;
        // per-call machine views -> every agent (the readers are not known here)
        unsigned pub = 0;
        for (int a = 0; a < c->k; ++a) {
            const int gid = c->proc * c->k + a, m = gid / L;
            bool read = machine_weights != nullptr;
            for (int i = 0; i < c->n && !read; ++i) {
                if (i / c->k == c->proc) continue;
                const int mi = i / L;
                read = mi == m || c->WM[static_cast<size_t>(mi) * NM + m] != 0.0;
            }
            if (read) pub |= 1u << a;
        }
        const int gk = hmode ? static_cast<int>(g_dtype) : static_cast<int>(dtype);
        return exchange_common(c, x, hmode == 1 ? g : nullptr, y, nullptr, count, dtype, gk, dtype, dtype,
                               hmode ? lr : 0.f, nullptr, static_cast<cudaStream_t>(stream),
                               hmode == 2 ? g : nullptr, &tab, nullptr, pub);
    }
    const size_t es = dtype == BF_FLOAT32 ? 4 : 2;
    s = ensure_exchange(c, count * es);
    if (s) return s;
    // Across GPUs with every machine inside one process (L divides agents_per_proc) and a
    // static machine topology: the push kernel's hierarchical modes (exchange_push.cuh
    // MODE 6-8) -- each machine's average is formed in registers from its L rows, crosses
    // NVLink once per reader process, and the combine is stored to the L rows.
    // A machine spanning P processes with a multicast buffer registered for this machine
    // size (bf_hier_set_multicast): NVLS machine average (hier_nvls.cu), then the push
    // kernel's hierarchical mode over the average row (machine-level exchange between the
    // processes of the same local index, broadcast to the K rows).
    if (c->hier_mode != 1 && c->nprocs > 1 && c->inbox_off && c->nvls_mc && c->nvls_L == L && !machine_weights &&
        dtype == BF_FLOAT32 && L > c->k && L % c->k == 0 && L / c->k >= c->nvls_min_p &&
        static_cast<long long>(count) <= c->nvls_cap &&
        count * 4 <= c->exch_cap) {
        const int P = L / c->k, me = c->proc, m = me / P, l = me % P;
        if (!c->nflag_off) return fail(BF_ERR_STATE, "NVLS flags not allocated");
        NvlsParams v;
        memset(&v, 0, sizeof(v));
        v.geo = make_geo(c, count);
        v.geo.vec_ok = (count % 4 == 0) && aligned16(x) && (!hmode || aligned16(g));
        v.x = static_cast<const float *>(x);
        v.g = g;
        v.hmode = hmode;
        v.lr = hmode ? lr : 0.f;
        v.invL = 1.0f / static_cast<float>(L);
        v.uc = c->nvls_uc;
        v.mc = c->nvls_mc;
        v.cap = c->nvls_cap;
        v.avg = nullptr;   // the average lands in the local copy of the buffer's average half
        v.nflag_off = c->nflag_off;
        v.proc0 = m * P;
        v.P = P;
        order_stream(c, static_cast<cudaStream_t>(stream));
        CU(launch_hier_nvls(v, hmode && g_dtype == BF_BFLOAT16 ? 1 : 0, static_cast<cudaStream_t>(stream)));
        c->launches++;
        // machine-level combine over the processes of local index l: (m', l) for m' with W_M[m][m'] != 0
        ExchParams q;
        memset(&q, 0, sizeof(q));
        q.geo = make_geo(c, count);
        q.geo.k = 1;
        q.geo.n = c->nprocs;
        q.geo.vec_ok = (count % 4 == 0) && aligned16(y) && (hmode != 2 || aligned16(g));
        q.wmode = kWStatic;
        q.tab.self_w[0] = static_cast<float>(c->WM[static_cast<size_t>(m) * NM + m]);
        int cnt = 0;
        for (int d = 1; d < NM; ++d) {
            const int mm = ((m - d) % NM + NM) % NM;
            const double w = c->WM[static_cast<size_t>(m) * NM + mm];
            if (w == 0.0) continue;
            q.tab.src[0][cnt] = static_cast<unsigned char>(mm * P + l);
            q.tab.coef[0][cnt] = static_cast<float>(w);
            ++cnt;
        }
        q.tab.nsrc[0] = static_cast<unsigned char>(cnt);
        for (int i = 0; i < NM; ++i)   // the process of local index l in every machine that reads machine m
            if (i != m && c->WM[static_cast<size_t>(i) * NM + m] != 0.0) q.pushq[0] |= 1u << (i * P + l);
        // the machine exchange reads the average half of the NVLS launch's parity: that launch
        // is the epoch before this one, so the push kernel picks x / x_alt by its epoch - 1
        q.x = c->nvls_uc + 2 * c->nvls_cap;
        q.x_alt = c->nvls_uc + 3 * c->nvls_cap;
        q.y = y;
        q.g = hmode == 2 ? g : nullptr;
        q.lr = hmode == 2 ? lr : 0.f;
        q.kernel = 3;
        q.push = 1;
        q.hier_L = c->k;
        q.hier_in = 1;
        q.hier_mode = hmode == 2 ? 8 : 6;
        q.slot_off = c->slot_off;
        q.slot_agent_stride = 2 * c->exch_cap;
        q.slot_parity_stride = c->exch_cap;
        q.inbox_off = c->inbox_off;
        q.inbox_agent_stride = 2 * c->exch_cap;
        q.inbox_parity_stride = c->exch_cap;
        q.pflag_off = c->pflag_off;
        q.prog_off = c->prog_off;
        q.stats = c->stats;
        q.max_ctas = c->max_ctas;
        CU(launch_hier_push(q, 0, hmode == 2 ? static_cast<int>(g_dtype) : 0, static_cast<cudaStream_t>(stream)));
        c->launches++;
        return BF_OK;
    }
    // Machines inside processes (L divides K): K / L machine agents per process.  A
    // machine spanning P = L / K processes: one "partial" agent per process -- the
    // average of its K rows -- and machine m's average is the mean of its P partials,
    // so partial q' enters with weight W_M[m][m(q')] / P (the same push kernel).
    const int Km = L <= c->k && c->k % L == 0 ? c->k / L : (L % c->k == 0 ? 1 : 0);
    const int P = L > c->k ? L / c->k : 1;   // processes per machine
    if (c->hier_mode != 1 && c->nprocs > 1 && c->inbox_off && !machine_weights && (Km == 1 || Km == 2 || Km == 4) &&
        count <= c->exch_cap / es && (P == 1 || P <= kMaxS)) {
        ExchParams q;
        memset(&q, 0, sizeof(q));
        q.geo = make_geo(c, count);
        q.geo.k = Km;
        q.geo.n = P == 1 ? NM : c->nprocs;
        const size_t vw = dtype == BF_BFLOAT16 ? 8 : 4;
        q.geo.vec_ok = (count % vw == 0) && aligned16(x) && aligned16(y) && (!hmode || aligned16(g));
        q.wmode = kWStatic;
        if (P == 1) {
            for (int a = 0; a < Km; ++a) {   // machine-level rows of W_M, sources in (m - d) mod M order
                const int m = c->proc * Km + a;
                q.tab.self_w[a] = static_cast<float>(c->WM[static_cast<size_t>(m) * NM + m]);
                int cnt = 0;
                for (int d = 1; d < NM; ++d) {
                    const int mm = ((m - d) % NM + NM) % NM;
                    const double w = c->WM[static_cast<size_t>(m) * NM + mm];
                    if (w == 0.0) continue;
                    q.tab.src[a][cnt] = static_cast<unsigned char>(mm);
                    q.tab.coef[a][cnt] = static_cast<float>(w);
                    ++cnt;
                }
                q.tab.nsrc[a] = static_cast<unsigned char>(cnt);
                for (int i = 0; i < NM; ++i)   // processes hosting a machine that reads machine m
                    if (i / Km != c->proc && c->WM[static_cast<size_t>(i) * NM + m] != 0.0)
                        q.pushq[a] |= 1u << (i / Km);
            }
        } else {   // one partial agent per process; processes in (me - d) mod nprocs order
            const int np = c->nprocs, me = c->proc, m = me / P;
            q.tab.self_w[0] = static_cast<float>(c->WM[static_cast<size_t>(m) * NM + m] / P);
            int cnt = 0;
            for (int d = 1; d < np; ++d) {
                const int qq = ((me - d) % np + np) % np;
                const double w = c->WM[static_cast<size_t>(m) * NM + qq / P];
                if (w == 0.0) continue;
                if (cnt >= kMaxS) return fail(BF_ERR_UNSUPPORTED, "hierarchical: too many source processes");
                q.tab.src[0][cnt] = static_cast<unsigned char>(qq);
                q.tab.coef[0][cnt] = static_cast<float>(w / P);
                ++cnt;
            }
            q.tab.nsrc[0] = static_cast<unsigned char>(cnt);
            for (int i = 0; i < np; ++i)   // processes whose machine reads machine m
                if (i != me && c->WM[static_cast<size_t>(i / P) * NM + m] != 0.0) q.pushq[0] |= 1u << i;
        }
        q.x = x;
        q.y = y;
        q.g = g;
        q.lr = hmode ? lr : 0.f;
        q.kernel = 3;
        q.push = 1;
        q.hier_L = P == 1 ? L : c->k;   // rows per (machine / partial) agent
        q.hier_mode = hmode == 0 ? 6 : (hmode == 1 ? 7 : 8);
        q.slot_off = c->slot_off;
        q.slot_agent_stride = 2 * c->exch_cap;
        q.slot_parity_stride = c->exch_cap;
        q.inbox_off = c->inbox_off;
        q.inbox_agent_stride = 2 * c->exch_cap;
        q.inbox_parity_stride = c->exch_cap;
        q.pflag_off = c->pflag_off;
        q.prog_off = c->prog_off;
        q.stats = c->stats;
        order_stream(c, static_cast<cudaStream_t>(stream));
        q.max_ctas = c->max_ctas;
        CU(launch_hier_push(q, dtype, hmode ? static_cast<int>(g_dtype) : 0, static_cast<cudaStream_t>(stream)));
        c->launches++;
        return BF_OK;
    }
    if (c->hier_ready && c->hier_L != L) {   // slices are sized per machine size: reallocate
        CU(cudaDeviceSynchronize());
        if ((s = bf_barrier_internal(c))) return s;
        CU(cudaDeviceSynchronize());
        if (c->heap_used == c->hier_top) c->heap_used = c->hier_begin;
        c->hier_ready = false;
    }
    if (!c->hier_ready) {
        // fp32 slice buffers: each agent averages / combines ceil(tiles / L) tiles
        const bool on_top = c->heap_used == c->exch_top;
        c->hier_begin = c->heap_used;
        const size_t slice_tiles = (static_cast<size_t>(c->ready_stride) + L - 1) / L;
        const size_t bytes = slice_tiles * kTile * 4;
        unsigned long long off;
        if ((s = heap_alloc(c, static_cast<size_t>(c->k) * 2 * bytes, &off))) return s;
        c->b_off = off;
        if ((s = heap_alloc(c, static_cast<size_t>(c->k) * 2 * bytes, &off))) return s;
        c->c_off = off;
        if ((s = heap_alloc(c, static_cast<size_t>(c->k) * c->ready_stride * 8, &off))) return s;
        c->fb_off = off;
        if ((s = heap_alloc(c, static_cast<size_t>(c->k) * c->ready_stride * 8, &off))) return s;
        c->fc_off = off;
        if (on_top) c->exch_top = c->heap_used;   // released together with the exchange region
        c->hier_top = c->heap_used;
        c->hier_L = L;
        c->bc_agent_stride = 2 * bytes;
        c->bc_parity_stride = bytes;
        c->hier_ready = true;
        if ((s = publish_region(c))) return s;
    }
    p.geo = make_geo(c, count);
    p.geo.vec_ok = (count % 4 == 0) && aligned16(x) && aligned16(y) && (!hmode || aligned16(g));
    p.x = x;
    p.y = y;
    p.L = L;
    p.hmode = hmode;
    for (int a = 0; a < c->k; ++a) {   // stage A: only agents whose machine spans other processes
        const int m = (c->proc * c->k + a) / L;
        if ((m * L) / c->k != c->proc || (m * L + L - 1) / c->k != c->proc) p.pubA |= 1u << a;
    }
    p.g = g;
    p.g_bf16 = hmode && g_dtype == BF_BFLOAT16;
    p.lr = lr;
    p.TS = (p.geo.T + L - 1) / L;
    p.slot_off = c->slot_off;
    p.slot_agent_stride = 2 * c->exch_cap;
    p.slot_parity_stride = c->exch_cap;
    p.ready_off = c->ready_off;
    p.ready_stride = c->ready_stride;
    p.b_off = c->b_off;
    p.c_off = c->c_off;
    p.fb_off = c->fb_off;
    p.fc_off = c->fc_off;
    p.bc_agent_stride = c->bc_agent_stride;
    p.bc_parity_stride = c->bc_parity_stride;
    order_stream(c, static_cast<cudaStream_t>(stream));
    CU(launch_hier(p, dtype, 0, static_cast<cudaStream_t>(stream)));
    c->launches++;
    return BF_OK;
}

bf_status bf_set_max_ctas(bf_ctx *c, int ctas) {
    bf_status s = check_ctx(c, false);
    if (s) return s;
    if (ctas < 0 || ctas > kMaxGrid) return fail(BF_ERR_ARG, "max_ctas must be in [0, %d]", kMaxGrid);
    c->max_ctas = ctas;
    return BF_OK;
}

bf_status bf_hier_set_multicast(bf_ctx *c, int local_size, void *uc, unsigned long long mc, size_t bytes) {
    bf_status s = check_ctx(c);
    if (s) return s;
    if (!uc && !mc) {   // unregister
        c->nvls_uc = nullptr;
        c->nvls_mc = 0;
        c->nvls_cap = 0;
        c->nvls_L = 0;
        return BF_OK;
    }
    if (!uc || !mc || bytes < 2 * 16 || (reinterpret_cast<uintptr_t>(uc) & 15u) || (mc & 15u))
        return fail(BF_ERR_ARG, "multicast buffer: unicast and multicast addresses (16-byte aligned) and its size");
    if (local_size <= c->k || local_size % c->k)
        return fail(BF_ERR_ARG, "NVLS averages machines that span processes: local_size must be a multiple of "
                                "agents_per_proc larger than it");
    c->nvls_uc = static_cast<float *>(uc);
    c->nvls_mc = mc;
    c->nvls_cap = static_cast<long long>(bytes / 16) / 4 * 4;   // fp32 elements per half (partials and averages x 2)
    c->nvls_L = local_size;
    return BF_OK;
}

bf_status bf_hierarchical_neighbor_allreduce(bf_ctx *c, const void *x, void *y, size_t count, bf_dtype dtype,
                                             const bf_weights *machine_weights, void *stream) {
    return hier_common(c, x, y, count, dtype, 0, nullptr, BF_FLOAT32, 0.f, machine_weights, stream);
}

bf_status bf_hierarchical_atc_step(bf_ctx *c, float *x, const void *g, bf_dtype g_dtype, size_t count, float lr,
                                   const bf_weights *machine_weights, void *stream) {
    return hier_common(c, x, x, count, BF_FLOAT32, 1, g, g_dtype, lr, machine_weights, stream);
}

bf_status bf_hierarchical_awc_step(bf_ctx *c, float *x, const void *g, bf_dtype g_dtype, size_t count, float lr,
                                   const bf_weights *machine_weights, void *stream) {
    return hier_common(c, x, x, count, BF_FLOAT32, 2, g, g_dtype, lr, machine_weights, stream);
}

// ---- windows ----------------------------------------------------------------
static Window *find_win(bf_ctx *c, const char *name) {
    if (!name) return nullptr;
    auto it = c->windows.find(name);
    return it == c->windows.end() ? nullptr : &it->second;
}

bf_status bf_win_create(bf_ctx *c, const char *name, void *x, size_t count, bf_dtype dtype, int zero_init,
                        int with_p) {
    bf_status s = check_ctx(c);
    if (s) return s;
    if (!name || !*name) return fail(BF_ERR_ARG, "window name required");
    if (find_win(c, name)) return fail(BF_ERR_WINDOW, "window '%s' already exists", name);
    if (!x || count == 0) return fail(BF_ERR_ARG, "window tensor must be non-empty");
    if (dtype != BF_FLOAT32 && dtype != BF_BFLOAT16) return fail(BF_ERR_UNSUPPORTED, "dtype");
    Window w;
    w.name = name;
    w.x = x;
    w.count = count;
    w.dtype = dtype;
    w.with_p = with_p ? 1 : 0;
    w.ef = c->win_ef ? 1 : 0;
    w.zero_init = zero_init ? 1 : 0;
    w.side.resize(c->n);
    for (int i = 0; i < c->n; ++i) {
        w.side[i].in = in_list(c, i);
        w.side[i].out = out_list(c, i);
        w.maxdin = std::max<int>(w.maxdin, static_cast<int>(w.side[i].in.size()));
        w.maxdout = std::max<int>(w.maxdout, static_cast<int>(w.side[i].out.size()));
    }
    if (w.maxdin > kMaxS || w.maxdout > kMaxS) return fail(BF_ERR_UNSUPPORTED, "window degree > %d", kMaxS);
    const size_t es = dtype == BF_FLOAT32 ? 4 : 2;
    const size_t K = c->k, DI = w.maxdin, DO = w.maxdout;
    WinParams &b = w.base;
    memset(&b, 0, sizeof(b));
    w.alloc_begin = c->heap_used;
    unsigned long long off;
#define WALLOC(field, bytes)                           \
    do {                                               \
        if ((s = heap_alloc(c, (bytes), &off))) {      \
            c->heap_used = w.alloc_begin;              \
            return s;                                  \
        }                                              \
        b.field = off;                                 \
    } while (0)
    const size_t cpad = (count + 7) / 8 * 8;   // 16-byte rows for 8-wide bf16 / 4-wide fp32 vectors
    WALLOC(slot_off, K * DI * 2 * cpad * es);
    WALLOC(pslot_off, K * DI * 2 * 8);
    WALLOC(version_off, K * DI * 8);
    WALLOC(consumed_off, K * DO * 8);
    WALLOC(outbox_off, K * DO * cpad * 4);
    WALLOC(pout_off, K * DO * 8);
    WALLOC(delivered_off, K * DO * 8);
    WALLOC(obvalid_off, K * DO * 4);
    WALLOC(conslocal_off, K * DI * 8);
    WALLOC(p_off, K * 8);
    WALLOC(dec_off, K * DO * 8);
    WALLOC(snap_off, K * DI * 16);
    WALLOC(ctl_off, 4 * 8);
#undef WALLOC
    w.alloc_end = c->heap_used;
    b.maxdin = w.maxdin;
    b.maxdout = w.maxdout;
    b.cpad = static_cast<long long>(cpad);
    b.x = x;
    b.out = x;
    b.dtype = dtype;
    b.with_p = w.with_p;
    std::vector<double> ones(K, 1.0);
    CU(cudaMemcpy(c->heap + b.p_off, ones.data(), K * 8, cudaMemcpyHostToDevice));
    if (!zero_init) {
        // slots start as a copy of the local tensor, in half 1 (R10)
        for (int a = 0; a < c->k; ++a) {
            const int gid = c->proc * c->k + a;
            for (size_t q = 0; q < w.side[gid].in.size(); ++q)
                CU(cudaMemcpy(c->heap + b.slot_off + ((a * DI + q) * 2 + 1) * cpad * es,
                              static_cast<char *>(x) + a * count * es, count * es, cudaMemcpyDeviceToDevice));
        }
    }
    CU(cudaDeviceSynchronize());
    c->windows[name] = w;
    s = bf_barrier(c, nullptr);
    if (s) return s;
    CU(cudaDeviceSynchronize());
    return BF_OK;
}

bf_status bf_win_set_error_feedback(bf_ctx *c, const char *name, int enable) {
    bf_status s = check_ctx(c);
    if (s) return s;
    Window *w = find_win(c, name);
    if (!w) return fail(BF_ERR_WINDOW, "unknown window '%s'", name ? name : "(null)");
    w->ef = enable ? 1 : 0;
    return BF_OK;
}

bf_status bf_win_free(bf_ctx *c, const char *name) {
    bf_status s = check_ctx(c);
    if (s) return s;
    Window *w = find_win(c, name);
    if (!w) return fail(BF_ERR_WINDOW, "unknown window '%s'", name ? name : "(null)");
    CU(cudaDeviceSynchronize());
    s = bf_barrier(c, nullptr);
    if (s) return s;
    CU(cudaDeviceSynchronize());
    if (w->alloc_end == c->heap_used) c->heap_used = w->alloc_begin;   // LIFO release
    c->windows.erase(name);
    return BF_OK;
}

static bf_status win_setup(bf_ctx *c, Window *w, uint64_t agent_mask, WinParams &p) {
    p = w->base;
    p.geo = make_geo(c, w->count);
    // 16-byte vectors: 4 fp32 or 8 bf16 elements per access (WinVec)
    p.geo.vec_ok = (w->count % (w->dtype == BF_BFLOAT16 ? 8 : 4) == 0) && aligned16(w->x);
    const uint64_t all = c->k >= 64 ? ~0ull : ((1ull << c->k) - 1);
    p.agent_mask = agent_mask ? (agent_mask & all) : all;
    return BF_OK;
}

static bf_status win_push(bf_ctx *c, const char *name, const bf_weights *weights, uint64_t agent_mask,
                          int overwrite, void *stream, const void *grad = nullptr, float lr = 0.f) {
    bf_status s = check_ctx(c);
    if (s) return s;
    Window *w = find_win(c, name);
    if (!w) return fail(BF_ERR_WINDOW, "unknown window '%s'", name ? name : "(null)");
    WinParams p;
    win_setup(c, w, agent_mask, p);
    p.overwrite = overwrite;
    p.ef = (w->dtype == BF_BFLOAT16 && !overwrite && w->ef) ? 1 : 0;
    p.g = grad;
    p.lr = lr;
    if (grad && !aligned16(grad)) p.geo.vec_ok = 0;
    for (int a = 0; a < c->k; ++a) {
        const int gid = c->proc * c->k + a;
        const auto &outs = w->side[gid].out;
        if (!weights) {   // Listing 3: 1/(outdegree+1) to every out-neighbour
            const double wt = 1.0 / (outs.size() + 1.0);
            p.self_w[a] = static_cast<float>(wt);
            p.self_wd[a] = wt;
            for (size_t q = 0; q < outs.size(); ++q) {
                const int j = outs[q];
                const auto &ins = w->side[j].in;
                p.out_q[a][q] = static_cast<unsigned char>(q);
                p.out_dst[a][q] = static_cast<unsigned char>(j);
                p.out_qin[a][q] = static_cast<unsigned char>(std::find(ins.begin(), ins.end(), gid) - ins.begin());
                p.out_s[a][q] = static_cast<float>(wt);
                p.out_sd[a][q] = wt;
            }
            p.nout[a] = static_cast<unsigned char>(outs.size());
            continue;
        }
        const bf_weights &v = weights[a];
        s = validate_view(c, gid, v, false, true, c->n);
        if (s) return s;
        p.self_w[a] = static_cast<float>(v.self_weight);
        p.self_wd[a] = v.self_weight;
        for (int q = 0; q < v.n_dst; ++q) {
            const int j = v.dst_ranks[q];
            auto it = std::find(outs.begin(), outs.end(), j);
            if (it == outs.end())
                return fail(BF_ERR_WINDOW, "agent %d: dst %d is not an out-neighbour at window creation (P:398)",
                            gid, j);
            const auto &ins = w->side[j].in;
            p.out_q[a][q] = static_cast<unsigned char>(it - outs.begin());
            p.out_dst[a][q] = static_cast<unsigned char>(j);
            p.out_qin[a][q] = static_cast<unsigned char>(std::find(ins.begin(), ins.end(), gid) - ins.begin());
            p.out_s[a][q] = static_cast<float>(v.dst_weights[q]);
            p.out_sd[a][q] = v.dst_weights[q];
        }
        p.nout[a] = static_cast<unsigned char>(v.n_dst > 0 ? v.n_dst : 0);
    }
    order_stream(c, static_cast<cudaStream_t>(stream));
    CU(launch_win_push(p, 0, static_cast<cudaStream_t>(stream)));
    c->launches += 1;
    return BF_OK;
}

bf_status bf_win_put(bf_ctx *c, const char *name, const bf_weights *weights, uint64_t agent_mask, void *stream) {
    return win_push(c, name, weights, agent_mask, 1, stream);
}

bf_status bf_win_accumulate(bf_ctx *c, const char *name, const bf_weights *weights, int require_mutex,
                            uint64_t agent_mask, void *stream) {
    (void)require_mutex;   // the versioned SPSC slot protocol is the mutex
    return win_push(c, name, weights, agent_mask, 0, stream);
}

bf_status bf_win_accumulate_grad(bf_ctx *c, const char *name, const void *g, float lr, const bf_weights *weights,
                                 uint64_t agent_mask, void *stream) {
    bf_status s = check_ctx(c);
    if (s) return s;
    if (!g) return fail(BF_ERR_ARG, "null gradient");
    if (!std::isfinite(lr)) return fail(BF_ERR_ARG, "non-finite lr");
    if (is_host_ptr(g)) return fail(BF_ERR_ARG, "bf_win_accumulate_grad takes a device gradient");
    return win_push(c, name, weights, agent_mask, 0, stream, g, lr);
}

static bf_status win_pull(bf_ctx *c, const char *name, const bf_weights *weights, void *out, uint64_t agent_mask,
                          int update, void *stream) {
    bf_status s = check_ctx(c);
    if (s) return s;
    Window *w = find_win(c, name);
    if (!w) return fail(BF_ERR_WINDOW, "unknown window '%s'", name ? name : "(null)");
    WinParams p;
    win_setup(c, w, agent_mask, p);
    if (out) {
        p.out = out;
        p.geo.vec_ok = p.geo.vec_ok && aligned16(out);
    }
    for (int b = 0; b < c->k; ++b) {
        const int gid = c->proc * c->k + b;
        const auto &ins = w->side[gid].in;
        p.nin[b] = static_cast<unsigned char>(ins.size());
        for (size_t q = 0; q < ins.size(); ++q) {
            const int src = ins[q];
            const auto &outs = w->side[src].out;
            p.in_src[b][q] = static_cast<unsigned char>(src);
            p.in_qout[b][q] = static_cast<unsigned char>(std::find(outs.begin(), outs.end(), gid) - outs.begin());
            p.in_r[b][q] = static_cast<float>(1.0 / (ins.size() + 1.0));
        }
        p.self_w[b] = static_cast<float>(1.0 / (ins.size() + 1.0));
        if (update && weights) {
            const bf_weights &v = weights[b];
            s = validate_view(c, gid, v, true, false, c->n);
            if (s) return s;
            p.self_w[b] = static_cast<float>(v.self_weight);
            for (size_t q = 0; q < ins.size(); ++q) p.in_r[b][q] = 0.f;
            for (int q = 0; q < v.n_src; ++q) {
                auto it = std::find(ins.begin(), ins.end(), v.src_ranks[q]);
                if (it == ins.end())
                    return fail(BF_ERR_WINDOW, "agent %d: src %d is not an in-neighbour at window creation", gid,
                                v.src_ranks[q]);
                p.in_r[b][it - ins.begin()] = static_cast<float>(v.src_weights[q]);
            }
        }
    }
    order_stream(c, static_cast<cudaStream_t>(stream));
    CU(launch_win_collect(p, update, 0, static_cast<cudaStream_t>(stream)));
    c->launches += 1;
    return BF_OK;
}

bf_status bf_alloc(bf_ctx *c, size_t bytes, void **ptr) {
    bf_status s = check_ctx(c);
    if (s) return s;
    if (!ptr || bytes == 0) return fail(BF_ERR_ARG, "bad allocation request");
    unsigned long long off;
    if ((s = heap_alloc(c, bytes, &off))) return s;
    *ptr = c->heap + off;
    return BF_OK;
}

bf_status bf_win_get(bf_ctx *c, const char *name, const bf_weights *weights, uint64_t agent_mask, void *stream) {
    bf_status s = check_ctx(c);
    if (s) return s;
    Window *w = find_win(c, name);
    if (!w) return fail(BF_ERR_WINDOW, "unknown window '%s'", name ? name : "(null)");
    const char *xp = static_cast<const char *>(w->x);
    if (xp < c->heap || xp + w->count * c->k * (w->dtype == BF_BFLOAT16 ? 2 : 4) > c->heap + c->heap_bytes)
        return fail(BF_ERR_UNSUPPORTED, "win_get reads the neighbours' window tensors: create the window on a "
                                        "tensor allocated with bf_alloc (symmetric heap)");
    WinParams p;
    win_setup(c, w, agent_mask, p);
    for (int b = 0; b < c->k; ++b) {
        const int gid = c->proc * c->k + b;
        const auto &ins = w->side[gid].in;
        p.nin[b] = static_cast<unsigned char>(ins.size());
        for (size_t q = 0; q < ins.size(); ++q) {
            p.in_src[b][q] = static_cast<unsigned char>(ins[q]);
            p.in_r[b][q] = weights ? 0.f : 1.f;   // default: every in-neighbour, weight 1
        }
        if (weights) {
            const bf_weights &v = weights[b];
            s = validate_view(c, gid, v, true, false, c->n);
            if (s) return s;
            for (int q = 0; q < v.n_src; ++q) {
                auto it = std::find(ins.begin(), ins.end(), v.src_ranks[q]);
                if (it == ins.end())
                    return fail(BF_ERR_WINDOW, "agent %d: src %d is not an in-neighbour at window creation", gid,
                                v.src_ranks[q]);
                p.in_r[b][it - ins.begin()] = static_cast<float>(v.src_weights[q]);
            }
        }
    }
    order_stream(c, static_cast<cudaStream_t>(stream));
    CU(launch_win_get(p, static_cast<unsigned long long>(xp - c->heap), static_cast<cudaStream_t>(stream)));
    c->launches += 2;
    return BF_OK;
}

bf_status bf_win_update(bf_ctx *c, const char *name, const bf_weights *weights, void *out, uint64_t agent_mask,
                        void *stream) {
    return win_pull(c, name, weights, out, agent_mask, 1, stream);
}

bf_status bf_win_update_then_collect(bf_ctx *c, const char *name, uint64_t agent_mask, void *stream) {
    return win_pull(c, name, nullptr, nullptr, agent_mask, 0, stream);
}

bf_status bf_win_get_p(bf_ctx *c, const char *name, double *p_host, void *stream) {
    bf_status s = check_ctx(c);
    if (s) return s;
    Window *w = find_win(c, name);
    if (!w) return fail(BF_ERR_WINDOW, "unknown window '%s'", name ? name : "(null)");
    if (!p_host) return fail(BF_ERR_ARG, "null p_host");
    CU(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    CU(cudaMemcpy(p_host, c->heap + w->base.p_off, c->k * 8, cudaMemcpyDeviceToHost));
    return BF_OK;
}

bf_status bf_win_counters(bf_ctx *c, const char *name, int dst_local, int src_rank, uint64_t *version,
                          uint64_t *consumed) {
    bf_status s = check_ctx(c);
    if (s) return s;
    Window *w = find_win(c, name);
    if (!w) return fail(BF_ERR_WINDOW, "unknown window '%s'", name ? name : "(null)");
    if (dst_local < 0 || dst_local >= c->k || !version || !consumed) return fail(BF_ERR_ARG, "bad agent");
    const auto &ins = w->side[c->proc * c->k + dst_local].in;
    auto it = std::find(ins.begin(), ins.end(), src_rank);
    if (it == ins.end()) return fail(BF_ERR_WINDOW, "rank %d is not an in-neighbour", src_rank);
    const size_t ci = static_cast<size_t>(dst_local) * w->maxdin + (it - ins.begin());
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(version, c->heap + w->base.version_off + ci * 8, 8, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(consumed, c->heap + w->base.conslocal_off + ci * 8, 8, cudaMemcpyDeviceToHost));
    return BF_OK;
}

bf_status bf_win_version(bf_ctx *c, const char *name, int src_rank, uint64_t *version) {
    bf_status s = check_ctx(c);
    if (s) return s;
    Window *w = find_win(c, name);
    if (!w) return fail(BF_ERR_WINDOW, "unknown window '%s'", name ? name : "(null)");
    if (!version) return fail(BF_ERR_ARG, "null version");
    for (int a = 0; a < c->k; ++a) {   // the first local agent that has src_rank as an in-neighbour
        const auto &ins = w->side[c->proc * c->k + a].in;
        if (std::find(ins.begin(), ins.end(), src_rank) == ins.end()) continue;
        uint64_t consumed;
        return bf_win_counters(c, name, a, src_rank, version, &consumed);
    }
    return fail(BF_ERR_WINDOW, "rank %d is not an in-neighbour of a local agent", src_rank);
}

long long bf_win_slot_offset(bf_ctx *c, const char *name, int agent, int src_rank) {
    if (!c) return -1;
    Window *w = find_win(c, name);
    if (!w || agent < 0 || agent >= c->n) return -1;
    const auto &ins = w->side[agent].in;
    auto it = std::find(ins.begin(), ins.end(), src_rank);
    if (it == ins.end()) return -1;
    return static_cast<long long>(it - ins.begin()) * static_cast<long long>(w->count);
}

// ---- misc ---------------------------------------------------------------------
bf_status bf_barrier(bf_ctx *c, void *stream) {
    bf_status s = check_ctx(c);
    if (s) return s;
    if (c->nprocs == 1) return BF_OK;
    Geometry g = make_geo(c, 0);
    order_stream(c, static_cast<cudaStream_t>(stream));
    CU(launch_barrier(g, ++c->bar_epoch, static_cast<cudaStream_t>(stream)));
    c->launches++;
    return BF_OK;
}

}  // extern "C"

bf_status bf_barrier_internal(bf_ctx *c) { return bf_barrier(c, nullptr); }

extern "C" {

bf_status bf_poll_error(bf_ctx *c) {
    if (!c) return fail(BF_ERR_ARG, "null context");
    if (c->h_err && !*c->h_err && c->heap) {
        // a peer may have raised an abort in this process's pad after our last kernel
        unsigned int code = 0;
        cudaSetDevice(c->device);
        if (cudaMemcpy(&code, c->heap + offsetof(Pad, abort), 4, cudaMemcpyDeviceToHost) == cudaSuccess && code)
            *const_cast<unsigned int *>(c->h_err) = code;
    }
    if (c->h_err && *c->h_err) {
        c->poisoned = true;
        c->fault = static_cast<bf_status>(*c->h_err);
    }
    if (c->fault) return fail(c->fault, "latched device fault: %s", bf_status_string(c->fault));
    return BF_OK;
}

bf_status bf_fill_uniform(void *dst, bf_dtype dtype, size_t count, uint64_t seed, uint64_t offset, float scale,
                          void *stream) {
    if (!dst && count) return fail(BF_ERR_ARG, "null dst");
    if (dtype != BF_FLOAT32 && dtype != BF_BFLOAT16) return fail(BF_ERR_UNSUPPORTED, "dtype");
    CU(launch_fill_uniform(dst, dtype, count, seed, offset, scale, static_cast<cudaStream_t>(stream)));
    return BF_OK;
}

}  // extern "C"
