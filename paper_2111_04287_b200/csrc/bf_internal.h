// bf_internal.h -- internal structures shared by the runtime (runtime.cu) and
// the sm_100a kernels (exchange.cu, window.cu, generate.cu).
//
// Symmetric heap.  Every process cudaMalloc's one heap of the same size and
// exports it through CUDA IPC.  All collective allocations are made in the
// same order on every process, so a region has the same OFFSET in every heap:
// the address of process q's copy is peer_base[q] + offset.  Byte 0 of the
// heap is the process's signal pad (struct Pad).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bluefog_b200.h"

namespace bf {

#ifndef BF_TILE
#define BF_TILE 4096
#endif
#ifndef BF_THREADS
#define BF_THREADS 256
#endif
#ifndef BF_MINB
#define BF_MINB 3
#endif
constexpr int kTile = BF_TILE;         // elements per tile (the unit of one flag)
constexpr int kThreads = BF_THREADS;   // threads per CTA of the streaming kernels
constexpr int kVec = 4;                // elements per vector access
constexpr int kVecPerThread = kTile / (kThreads * kVec);   // 4
constexpr int kMaxK = BF_MAX_LOCAL_AGENTS;
constexpr int kMaxS = BF_MAX_DEGREE;
constexpr int kMaxN = BF_MAX_AGENTS;
constexpr int kMaxP = BF_MAX_PROCS;
constexpr size_t kPadBytes = 64 * 1024;
constexpr size_t kAlign = 4096;
constexpr int kMaxGrid = 4096;         // CTAs of one exchange launch (progress counters per process)
constexpr long long kLLCap = 32768;    // elements per agent up to which the cross-GPU exchange uses tagged words

// Per-agent, per-parity descriptor of a dynamic call (push side of Eq. 9):
// which agents this agent pushes to and with which s (sender-side weight).
struct Desc {
    unsigned long long epoch;      // epoch this descriptor belongs to
    unsigned long long dstmask;    // bit j: this agent declared j as destination
    unsigned long long has_dst;    // 1 if the agent declared destinations at all (push / push-pull)
    unsigned long long pad_;
    float s[kMaxN];                // s_j: weight for destination j
};

// Static local view of one agent (bf_set_topology_local): published in
// the agent's pad so every process can assemble the same global W.
struct LocalView {
    double self_w;
    int nsrc, ndst;                // -1: not given
    unsigned char src[kMaxS], dst[kMaxS];
    double r[kMaxS], s[kMaxS];
};

struct Pad {
    unsigned long long epoch;      // last completed exchange epoch of this process
    unsigned long long round;      // device-resident one-peer schedule round
    unsigned int done_ctr;         // CTA completion counter of the running kernel
    unsigned int abort;            // nonzero: abort code (bf_status) -- set locally or by a peer
    unsigned long long resv[13];
    unsigned long long done_from[kMaxP];   // done_from[q] = last epoch process q finished reading
    unsigned long long bar_from[kMaxP];    // device barrier arrivals
    Desc desc[kMaxK][2];
    LocalView lview[kMaxK];
    // push-sum gradient tracking (MODE 5): the scalar push-sum weight v of each local
    // agent for this epoch, published for the readers; tag = epoch
    unsigned long long gtv_tag[kMaxK][2];
    float gtv[kMaxK][2];
};
static_assert(sizeof(Pad) <= kPadBytes, "pad too large");

// Source table of one local agent for one call.
struct SrcTab {
    float self_w[kMaxK];
    float coef[kMaxK][kMaxS];
    unsigned char src[kMaxK][kMaxS];
    unsigned char nsrc[kMaxK];
};

// Dynamic-call declarations of the local agents (kernel-side copy of bf_weights).
struct DynDecl {
    unsigned char has_src[kMaxK];
    unsigned char has_dst[kMaxK];
    unsigned char ndst[kMaxK];
    unsigned char dst[kMaxK][kMaxS];
    float s[kMaxK][kMaxS];
};

enum WMode : int { kWStatic = 0, kWSchedule = 1, kWDynamic = 2 };

// Dynamic one-peer schedules, evaluated from a round counter on the host
// (bf_schedule_*) and inside the kernels (device-resident counter):
//   kind 1: one-peer exp-2 (R5): t = k mod ceil(log2 n), pull i - 2^t, push i + 2^t
//   kind 2: inner-outer exp-2 (R27): machines of L agents; local
//           rank o = k mod L pulls from machine m - 2^t, t = (k div L) mod
//           ceil(log2 M), same local rank; the other L - 1 agents of the machine,
//           relabelled r = (l - o - 1) mod L, run kind 1 over a group of L - 1
//           with t' = k mod ceil(log2(L - 1)).
// src = dst = -1: no peer this round (self weight 1).  Every agent with a peer
// mixes 1/2 self + 1/2 source, so each round's W is doubly stochastic.
__host__ __device__ inline void sched_peers(int kind, int n, int L, unsigned long long k, int i, int &src, int &dst) {
    src = dst = -1;
    int grp = n, base = 0, r = i, stride = 1;
    unsigned long long kk = k;
    if (kind == 2) {
        const int M = n / L, m = i / L, l = i % L;
        const int o = static_cast<int>(k % static_cast<unsigned long long>(L));
        if (l == o) {              // outer: one-peer exp-2 over the machines, slot o
            grp = M; base = o; r = m; stride = L; kk = k / static_cast<unsigned long long>(L);
        } else {                   // inner: one-peer exp-2 over the other L - 1 slots
            grp = L - 1; r = ((l - o - 1) % L + L) % L;
            int tau = 0;
            while ((1 << tau) < grp) ++tau;
            if (tau == 0) return;
            const int off = 1 << static_cast<int>(k % static_cast<unsigned long long>(tau));
            src = m * L + ((r - off + grp) % grp + o + 1) % L;
            dst = m * L + ((r + off) % grp + o + 1) % L;
            return;
        }
    }
    int tau = 0;
    while ((1 << tau) < grp) ++tau;
    if (tau == 0) return;
    const int off = 1 << static_cast<int>(kk % static_cast<unsigned long long>(tau));
    src = base + ((r - off) % grp + grp) % grp * stride;
    dst = base + (r + off) % grp * stride;
}

struct Geometry {
    int k;               // local agents
    int n;               // total agents
    int me;              // process rank
    int nprocs;
    long long count;     // elements per agent
    int T;               // tiles per agent
    int vec_ok;          // all rows 16B aligned and count % 4 == 0
    unsigned long long timeout_ns;
    unsigned long long peer_base[kMaxP];   // heap base of every process, valid in this process
    volatile unsigned int *host_err;       // mapped pinned word
};

struct ExchParams {
    Geometry geo;
    int x_kind, wire_kind, y_kind;         // 0 fp32, 1 bf16 (the template also fixes them)
    const void *x;
    const void *g;
    void *y;
    void *shadow;                           // bf16 copy of y (nullable)
    float lr;
    int awc;                                // AWC (Eq. 16): combine x, then subtract lr * g_self
    int g_bf16;                             // AWC: dtype of g
    // exchange region (offsets into every heap)
    unsigned long long slot_off, slot_agent_stride, slot_parity_stride;
    unsigned long long ready_off;           // u64 [k][ready_stride]
    int ready_stride;
    int wmode;
    int check;
    int kernel;                             // 2: chunked (any k); 3: local-agent fused (default, fused_supported)
    int chunk_tiles;                        // kernels 2, 3: tiles per chunk
    unsigned long long ccnt_off;            // kernels 2, 3: u32 [tmax] per-chunk CTA counters (local)
    unsigned long long cflag_off;           // kernels 2, 3: u64 [tmax] per-chunk release flags
    unsigned pub_mask;                      // kernel 3, kWStatic: local agents read by another process
    int sched_kind, sched_L;                // kWSchedule: schedule kind (1, 2) and machine size
    unsigned long long prog_off;            // kernel 3: u64 [kMaxGrid] per-CTA publish progress
    unsigned long long *stats;              // kernel 3 built with BF_STATS=1: u64 [grid][8] (diagnostics)
    float *psi;                             // kernel 3 MODE 3 (Exact-Diffusion): psi state [k][count], in place
    int gt;                                 // kernel 3: 4 = GT y-step (MODE 4), 5 = GT u/v-step (MODE 5), else 0
    int hier_L;                             // push MODE 6-8 (hierarchical): rows per machine agent (machine size)
    int hier_in;                            // rows averaged per machine agent (0: hier_L; 1: x is a machine average)
    const void *x_alt;                      // non-null: read x_alt instead of x when (epoch - 1) is odd (NVLS averages)
    int hier_mode;                          // 0: not hierarchical; 6, 7, 8: MODE of the hierarchical push
    int max_ctas;                           // hierarchical push launches: grid cap (0 = all SMs)
    const float *g2;                        // kernel 3 MODE 4 (GT y-step): g_prev [k][count] (fp32)
    float *gt_v;                            // kernel 3 MODE 5 (GT u/v-step): scalar weight v [k], updated in place
    float *x_out;                           // kernel 3 MODE 5: x = u / v [k][count]
    int ll;                                 // kernel 3 across GPUs, small messages: tagged 64-bit words (exchange_ll.cuh)
    unsigned long long ll_off, ll_stride;   // ll: u64 [n source agents][2 parities][ll cap] in every heap; row bytes
    int push;                               // kernel 3 across GPUs: writers push into the readers' inboxes
    unsigned long long inbox_off;           // push: wire dtype [n source agents][2 parities][cap] in every heap
    unsigned long long inbox_agent_stride, inbox_parity_stride;   // bytes
    unsigned long long pflag_off;           // push: u64 [kMaxP writer processes][kMaxGrid] in every heap
    unsigned pushq[kMaxK];                  // push, kWStatic: bit q = process q reads local agent a
    SrcTab tab;                             // kWStatic: final coefficients; kWDynamic: declared r
    DynDecl dyn;
};

// Hierarchical neighbour allreduce: stages A (publish), B (intra-
// machine average of one slice), C (machine-level combine of the slice),
// D (gather the slices).
struct HierParams {
    Geometry geo;
    const void *x;
    void *y;
    int L;                                  // agents per machine
    int hmode;                              // 0 plain, 1 H-ATC, 2 H-AWC (Eqs. 16-17)
    unsigned pubA;                          // local agents stage A publishes (machine spans processes)
    const void *g;                          // hmode 1, 2: gradient [k][count]
    int g_bf16;
    float lr;
    int TS;                                 // tiles per slice
    unsigned long long slot_off, slot_agent_stride, slot_parity_stride;   // stage A (x dtype)
    unsigned long long ready_off;
    int ready_stride;
    unsigned long long b_off, c_off, bc_agent_stride, bc_parity_stride;   // fp32 slices
    unsigned long long fb_off, fc_off;      // u64 flags [k][ready_stride]
    SrcTab mtab;                            // machine-level: src = machine ids
};

// NVLS intra-machine average (hier_nvls.cu): machines spanning P processes.
struct NvlsParams {
    Geometry geo;                           // k = rows of this process, count
    const float *x;                         // [k][count]
    const void *g;                          // H-ATC: gradient [k][count]
    int hmode;                              // 1: average x - lr g (H-ATC), else x
    float lr;
    float invL;                             // 1 / machine size
    float *uc;                              // this process's copy of the multicast buffer: fp32 [4][cap]
                                            // (partials [2 parities], averages [2 parities])
    unsigned long long mc;                  // multicast address of the same buffer
    long long cap;                          // elements per parity half
    float *avg;                             // (unused: the average stays in the buffer's average half)
    unsigned long long nflag_off;           // u64 [kMaxP][kMaxGrid] in every heap
    int proc0, P;                           // processes proc0 .. proc0 + P - 1 form this machine
};

// One-sided windows.
struct WinParams {
    Geometry geo;
    void *x;                                // registered stacked tensor
    void *out;                              // win_update output (or == x)
    int dtype;                              // 0 fp32, 1 bf16 (slot dtype = x dtype)
    int overwrite;                          // put
    int ef;                                 // error feedback of the bf16 wire rounding into the outbox
    const void *g;                          // gradient-in-window push (window dtype, [k][count]) or null
    float lr;
    int with_p;
    unsigned long long agent_mask;
    int maxdin, maxdout;
    long long cpad;                         // row stride of slots / outboxes: count rounded up to 8
    // heap offsets (symmetric)
    unsigned long long slot_off;            // [k][maxdin][2][count]
    unsigned long long pslot_off;           // double [k][maxdin][2]
    unsigned long long version_off;         // u64 [k][maxdin]   (written by producers)
    unsigned long long consumed_off;        // u64 [k][maxdout]  (written by consumers)
    unsigned long long outbox_off;          // float [k][maxdout][count]
    unsigned long long pout_off;            // double [k][maxdout]
    unsigned long long delivered_off;       // u64 [k][maxdout]  (local control)
    unsigned long long obvalid_off;         // u32 [k][maxdout]
    unsigned long long conslocal_off;       // u64 [k][maxdin]
    unsigned long long p_off;               // double [k]
    unsigned long long dec_off;             // u64 [k][maxdout] push decisions
    unsigned long long snap_off;            // u64 [k][maxdin][2] collect snapshot (c, v)
    unsigned long long ctl_off;             // u64 [4]: push gate (snapshot, done), collect gate (snapshot, done)
    // per-call tables
    float self_w[kMaxK];
    unsigned char nout[kMaxK];              // selected destinations of local agent a
    unsigned char out_q[kMaxK][kMaxS];      // out-index (position in the creation out-list)
    unsigned char out_dst[kMaxK][kMaxS];    // destination agent id
    unsigned char out_qin[kMaxK][kMaxS];    // its in-index at the destination
    float out_s[kMaxK][kMaxS];
    double out_sd[kMaxK][kMaxS];            // the same weights in fp64 for the p lane
    double self_wd[kMaxK];
    unsigned char nin[kMaxK];               // all creation in-neighbours of local agent a
    unsigned char in_src[kMaxK][kMaxS];
    unsigned char in_qout[kMaxK][kMaxS];    // position of a in the source's out-list
    float in_r[kMaxK][kMaxS];               // win_update weights
};

// ---- launchers (exchange.cu / window.cu / generate.cu) --------------------
cudaError_t launch_exchange(const ExchParams &p, int x_kind, int g_kind, int wire_kind, int y_kind,
                            int has_g, int grid, cudaStream_t s);
cudaError_t launch_hier(const HierParams &p, int x_kind, int grid, cudaStream_t s);
cudaError_t launch_hier_push(const ExchParams &p, int x_kind, int g_kind, cudaStream_t s);
cudaError_t launch_hier_nvls(const NvlsParams &p, int g_kind, cudaStream_t s);
cudaError_t launch_barrier(const Geometry &geo, unsigned long long epoch, cudaStream_t s);
cudaError_t launch_win_push(const WinParams &p, int grid, cudaStream_t s);
cudaError_t launch_win_collect(const WinParams &p, int update, int grid, cudaStream_t s);
cudaError_t launch_win_get(const WinParams &p, unsigned long long x_off, cudaStream_t s);
cudaError_t launch_fill_uniform(void *dst, int kind, size_t count, unsigned long long seed,
                                unsigned long long offset, float scale, cudaStream_t s);
cudaError_t launch_set_u64(unsigned long long *dst, unsigned long long v, cudaStream_t s);
int max_coresident(const void *func, int threads, size_t smem);
bool fused_supported(int k, int nprocs);   // kernel 3 is instantiated for this configuration

}  // namespace bf
