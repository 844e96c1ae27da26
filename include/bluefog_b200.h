/*
 * bluefog_b200.h -- C ABI of the B200-native decentralized partial-averaging
 * hot path (BlueFog, arXiv 2111.04287).
 *
 * Citations: P:NNN = line of the paper text (reference PAPER.md), with the
 * equation / section it belongs to.  "R<k>" = numbered reading of the paper
 * in DESIGN.md where the paper is silent or garbled.
 *
 * Model.  n agents ("nodes") run one process per GPU.  A process
 * hosts `agents_per_proc` consecutive agents (1 on an 8-GPU box; > 1 to
 * emulate n agents on fewer GPUs -- "virtual agents").  Global agent id
 * (the paper's rank) = proc_rank * agents_per_proc + local index.
 *
 * Data layout.  Every data call takes STACKED per-process buffers: the
 * vector of local agent a starts at element a*count (row-major
 * [agents_per_proc][count]).  All pointers are DEVICE pointers unless a
 * function says otherwise; `stream` is a cudaStream_t passed as void*
 * (NULL = legacy default stream).  Calls are stream-ordered and return
 * before the GPU work completes (that is the non-blocking form of P:635;
 * "wait" = synchronize the stream).  Caller-owned buffers must stay valid
 * until the stream work completes; the library never frees them.
 *
 * Empty inputs.  A data call with count == 0 returns BF_OK without checking its
 * pointers and without enqueueing anything (the epoch does not advance).
 *
 * Errors.  Every function returns a bf_status.  Host-side validation is
 * synchronous and enqueues nothing on failure.  Device-side faults (a spin
 * that exceeded BF_TIMEOUT_MS, a topology-check mismatch) are latched in the
 * context: bf_poll_error() returns them and the context is then poisoned
 * (later calls return BF_ERR_STATE).  bf_last_error() gives a message
 * (thread-local).  No call ever blocks forever: every device wait is bounded.
 *
 * Collectives: bf_connect_peers, bf_set_topology, bf_set_topology_local,
 * bf_set_machine_topology, bf_reserve, bf_alloc, bf_neighbor_allreduce,
 * bf_atc_step, bf_awc_step, bf_exact_diffusion_step, bf_gt_uv_step,
 * bf_gt_y_step, bf_hierarchical_neighbor_allreduce (and its ATC / AWC steps),
 * bf_win_create, bf_win_free and bf_barrier must be called by every process in
 * the same order (bf_set_max_ctas and bf_hier_set_multicast with the same
 * arguments on every process).  Window data calls (put / accumulate / update /
 * collect / get) are one-sided and need no matching call.
 *
 * Transfer across GPUs (internal, chosen per call): messages up to 262144
 * elements per agent (BF_LL_CAP; 32768 when the heap has no room for that
 * region) travel as epoch-tagged 64-bit words (no fence on the data path); larger ones are pushed into the readers' inboxes (static topologies and
 * schedules) or pulled by the readers (per-call pull-only views).  BF_XFER=pull
 * and BF_LL=0 (read at bf_init) force the pull path / turn the tagged words off.
 */
#ifndef BLUEFOG_B200_H
#define BLUEFOG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bf_ctx bf_ctx;

typedef enum {
    BF_OK = 0,
    BF_ERR_ARG = 1,          /* invalid argument (rank range, duplicate, NaN weight, bad config) */
    BF_ERR_STATE = 2,        /* context not connected / poisoned by an earlier device fault */
    BF_ERR_TOPOLOGY = 3,     /* send/receive declarations do not match */
    BF_ERR_CUDA = 4,         /* a CUDA runtime call failed */
    BF_ERR_TIMEOUT = 5,      /* a device wait exceeded BF_TIMEOUT_MS (peer missing / stalled) */
    BF_ERR_NOMEM = 6,        /* symmetric heap exhausted */
    BF_ERR_UNSUPPORTED = 7,  /* limits below exceeded, or unsupported dtype combination */
    BF_ERR_WINDOW = 8        /* unknown / duplicate window name, dst outside creation topology */
} bf_status;

typedef enum { BF_FLOAT32 = 0, BF_BFLOAT16 = 1 } bf_dtype;

/* Limits of this build. */
#define BF_MAX_AGENTS 64          /* n */
#define BF_MAX_PROCS 16           /* processes (GPUs) */
#define BF_MAX_LOCAL_AGENTS 16    /* agents_per_proc */
#define BF_MAX_DEGREE 16          /* declared sources / destinations per agent per call */

/* Local view of Eq. 9 for ONE agent and ONE call:
 *   x_i <- self_weight * x_i + sum_j r_ij * s_ij * x_j.
 * src_weights are r_ij for j in N(i) (receiver side, Eq. 11); dst_weights are
 * s_ji for j in M(i) (sender side, Eq. 10).  n_src < 0 / n_dst < 0 means "not
 * given".  Valid configurations (P:381 footnote): self+dst (push), self+src
 * (pull), self+src+dst (push-pull).  The static form is a NULL bf_weights
 * pointer.  Ranks are global agent ids; self or duplicate ranks -> BF_ERR_ARG.
 * Weights may be any finite real (Eq. 8 allows w_ij in R; reading R3). */
typedef struct {
    double self_weight;
    int n_src;
    const int *src_ranks;
    const double *src_weights;
    int n_dst;
    const int *dst_ranks;
    const double *dst_weights;
} bf_weights;

/* ---- context ------------------------------------------------------------------
 * bf_init: create the context of process `proc_rank` of `n_procs`, hosting
 * `agents_per_proc` agents on CUDA device `cuda_device`, with a symmetric
 * (SURVEY 8(b) names the fourth argument local_size, the paper's agents per
 * machine.  Here one process hosts agents_per_proc agents on one GPU --
 * 1 on an 8-GPU box, as in the paper; the machine size of the hierarchical
 * calls is set separately by bf_set_machine_topology.)  With a symmetric
 * heap of `heap_bytes` device bytes (exchange slots, windows, hierarchical
 * buffers and signal pads all live there; it is exported through CUDA IPC).
 * Env: BF_TIMEOUT_MS (default 10000) bounds every device wait.  Tuning /
 * diagnostics (read at bf_init): BF_EXCH=chunk forces the chunked exchange
 * kernel (default: the local-agent fused kernel where instantiated,
 * agents_per_proc 1, 2, 4, or 8 on one GPU), BF_FUSED_GRID (CTAs of the fused
 * kernel), BF_HIER=staged (sliced hierarchical kernel also on one GPU) or
 * BF_HIER=fused (Kronecker mix in the fused kernel also across GPUs),
 * BF_WIN_EF=1 (error feedback on for new bf16 windows), BF_STATS=1 (per-CTA
 * timings, bf_exchange_stats, with a -DBF_STATS=1 build). */
bf_status bf_init(int proc_rank, int n_procs, int agents_per_proc, int cuda_device,
                  size_t heap_bytes, bf_ctx **out);
/* Bootstrap: each process writes its blob (<= bf_ipc_blob_size() bytes) and the
 * caller all-gathers them (e.g. torch.distributed) in proc order, then every
 * process calls bf_connect_peers(ctx, all_blobs, blob_len) (collective).
 * With n_procs == 1 call bf_connect_peers(ctx, NULL, 0). */
size_t bf_ipc_blob_size(void);
bf_status bf_get_ipc_blob(bf_ctx *ctx, void *blob, size_t *len);
bf_status bf_connect_peers(bf_ctx *ctx, const void *blobs, size_t blob_len);
bf_status bf_finalize(bf_ctx *ctx);
int bf_size(const bf_ctx *ctx);                /* n, total agents ("size") */
int bf_rank(const bf_ctx *ctx);                /* global id of local agent 0 */
int bf_local_agents(const bf_ctx *ctx);
const char *bf_last_error(void);
const char *bf_status_string(bf_status s);

/* ---- topology (global view; P:199-206 neighbour sets) ---------------
 * W[i*n + j] = w_ij, the weight agent i applies to x_j (Eq. 8).  Every process
 * passes the same W.  Default before any call: fully connected 1/n (R15). */
bf_status bf_set_topology(bf_ctx *ctx, int n, const double *W);
/* Static topology from LOCAL views (Eq. 9; SURVEY 8(b)
 * "bf_set_topology_local"): weights[a] is the view of local agent a
 * (self_weight required; src ranks / r_ij and / or dst ranks / s_ji, the same
 * four configurations as the per-call views).  Collective: every process passes
 * its agents' views; the library exchanges them through the peers' signal pads
 * and every process assembles the same global W:
 *   w_ii = self_weight;  j in src_i: w_ij = r_ij * (s_ij if j lists i as a
 *   destination, else 1) (R1);  no src list (push only): w_ij = s_ij for every
 *   j that lists i (R16).
 * With the topology check on (default), a receiver's src list must name exactly
 * the senders that list it: else BF_ERR_TOPOLOGY (on every process, nothing
 * changed).  On success it replaces the topology like bf_set_topology (and
 * turns a dynamic schedule off). */
bf_status bf_set_topology_local(bf_ctx *ctx, const bf_weights *weights);
/* Hierarchical machine topology: machines of `local_size` consecutive
 * agents (machine_rank = rank // local_size); WM is n_machines^2. */
bf_status bf_set_machine_topology(bf_ctx *ctx, int local_size, int n_machines, const double *WM);
bf_status bf_in_neighbors(bf_ctx *ctx, int agent, int *ranks, int cap, int *n_out);
bf_status bf_out_neighbors(bf_ctx *ctx, int agent, int *ranks, int cap, int *n_out);
/* Built-in topologies into W (n*n, caller-owned host array): 0 ring,
 * 1 exponential-2 (R4), 2 fully connected, 3 one-peer exp-2 at round k. */
bf_status bf_topology_matrix(int kind, int n, uint64_t k, double *W);
/* One-peer dynamic exponential-2 schedule (R5): at round k, t = k mod
 * ceil(log2 n); agent `rank` pulls from rank - 2^t and pushes to rank + 2^t. */
bf_status bf_schedule_one_peer_exp2(int n, int rank, uint64_t round, int *src, int *dst);
/* Inner-outer dynamic exponential-2 schedule (named at P:828 and P:869; the
 * paper gives no formula -- DESIGN.md reading R27): machines of local_size
 * consecutive agents.  At round k local rank o = k mod local_size
 * pulls from machine m - 2^t (same local rank), t = (k div local_size) mod
 * ceil(log2 M); the other local_size - 1 agents of the machine run the
 * one-peer exp-2 rule among themselves (relabelled r = (l - o - 1) mod L,
 * t' = k mod ceil(log2(L - 1))).  *src = *dst = -1: no peer this round.
 * BF_ERR_ARG if local_size does not divide n. */
bf_status bf_schedule_inner_outer_exp2(int n, int local_size, int rank, uint64_t round, int *src, int *dst);
/* kind 0: none (static W); 1: one-peer exp-2; 2: inner-outer exp-2 over the
 * machine size of the last bf_set_machine_topology (BF_ERR_STATE if none).
 * Kinds 1 and 2 are evaluated ON DEVICE from a device-resident round counter
 * starting at round0, advanced by every schedule-mode call (graph-capturable);
 * every agent with a peer mixes 1/2 self + 1/2 its source. */
bf_status bf_set_dynamic_schedule(bf_ctx *ctx, int kind, uint64_t round0);
bf_status bf_set_topology_check(bf_ctx *ctx, int enable);   /* P:613; default on */
/* Cap the CTAs of the exchange kernels (0 = as many as the SMs hold, the default).
 * CTA b of every process pairs with CTA b of its peers, so every process must set
 * the same cap before its next exchange (collective by convention).  Use it when
 * exchanges overlap other GPU work (the optimizer's per-layer steps during
 * backward): the exchange then leaves SMs to the concurrent kernels. */
bf_status bf_set_max_ctas(bf_ctx *ctx, int ctas);

/* ---- the hot path ------------------------------------------------------------
 * bf_neighbor_allreduce (Eq. 5 P:183 static; Eq. 9-11 P:355-362 dynamic):
 * y_i = w_ii x_i + sum_j w_ij x_j for every local agent i.  x, y: stacked
 * [agents_per_proc][count] of `dtype`; y may alias x.  weights: NULL (static /
 * schedule) or an array of agents_per_proc local views.  fp32 accumulation;
 * bf16 output rounded RNE. */
bf_status bf_neighbor_allreduce(bf_ctx *ctx, const void *x, void *y, size_t count, bf_dtype dtype,
                                const bf_weights *weights, void *stream);
/* bf_atc_step: fused adapt-then-combine DSGD step (Eq. 4-5, Eq. 17
 * P:711, R6): x_i <- sum_j w_ij (x_j - lr*g_j), in place on the fp32 master x.
 * g: `g_dtype` gradients; x or g may be HOST pointers (pinned or pageable):
 * they are then staged through device memory inside the call (end-to-end
 * path).  wire: dtype of the copy neighbours read (R18: the agent's own term
 * uses the fp32 x_half).  x_bf16_shadow (nullable): also write RNE(x). */
bf_status bf_atc_step(bf_ctx *ctx, float *x, const void *g, bf_dtype g_dtype, size_t count,
                      float lr, bf_dtype wire, void *x_bf16_shadow,
                      const bf_weights *weights, void *stream);
/* bf_awc_step: fused adapt-while-communicate DSGD step (Eq. 16; R6):
 * x_i <- sum_j w_ij x_j - lr * g_i, in place on the fp32 master x (device
 * tensors).  The neighbours exchange x itself, so in a training loop the
 * exchange does not depend on this step's gradient. */
bf_status bf_awc_step(bf_ctx *ctx, float *x, const void *g, bf_dtype g_dtype, size_t count, float lr,
                      const bf_weights *weights, void *stream);
/* Exact-Diffusion step (appendix of the paper, Eqs. ed-1..ed-3, Listing ED-static;
 * SURVEY 8(f) rank 4), fused like bf_atc_step:
 *   psi_i = x_i - lr * g_i            (local update; written over psi, the state)
 *   phi_i = psi_i + x_i - psi_prev_i  (bias correction; psi_prev = psi on entry)
 *   x_i  <- sum_j w_ij phi_j          (partial averaging: static topology, schedule
 *                                      or per-call views as in bf_neighbor_allreduce)
 * x and psi: fp32 device tensors [agents_per_proc][count], updated in place; g:
 * fp32 or bf16.  Initialise psi = x^(0) so the first step is an ATC step.  The
 * neighbours' phi travel in `wire` (bf16: RNE, R18/R25).  Needs the fused
 * exchange kernel (agents_per_proc 1, 2, 4, or 8 on one GPU): else
 * BF_ERR_UNSUPPORTED.  Errors as bf_atc_step; host pointers are rejected. */
bf_status bf_exact_diffusion_step(bf_ctx *ctx, float *x, const void *g, bf_dtype g_dtype, float *psi,
                                  size_t count, float lr, bf_dtype wire, const bf_weights *weights,
                                  void *stream);

/* Push-sum gradient tracking (appendix "Push-sum gradient tracking", PAPER.md lines
 * 1000-1006, listing GT-varying), one fused launch per partial
 * averaging of a round (the gradient at the new x is the caller's, in between):
 *   bf_gt_uv_step:  u_i <- sum_j w_ij (u_j - lr y_j)            (line 1002)
 *                   v_i <- sum_j w_ij v_j                         (line 1003)
 *                   x_out_i = u_i / v_i                           (line 1004)
 *   bf_gt_y_step:   y_i <- sum_j w_ij (y_j + g_j - g_prev_j)     (line 1006)
 * u, y, x_out, g, g_prev: fp32 device tensors [agents_per_proc][count]; u and y are
 * updated in place.  v: fp32 device array [agents_per_proc], ONE push-sum weight per
 * agent (v^0 = 1 keeps every entry of the paper's vector v equal -- reading R28),
 * updated in place; the neighbours' weights travel through the signal pads.  W:
 * static topology, schedule or per-call views, as bf_neighbor_allreduce (the
 * listing uses push views: self 1/(d_out+1), dst 1/(d_out+1), src 1).  wire: dtype
 * of the neighbours' copies.  Needs the fused exchange kernel (agents_per_proc 1,
 * 2, 4 or 8 on one GPU): else BF_ERR_UNSUPPORTED.  Collective like
 * bf_neighbor_allreduce. */
bf_status bf_gt_uv_step(bf_ctx *ctx, float *u, float *v, const float *y, float *x_out, size_t count, float lr,
                        bf_dtype wire, const bf_weights *weights, void *stream);
bf_status bf_gt_y_step(bf_ctx *ctx, float *y, const float *g, const float *g_prev, size_t count, bf_dtype wire,
                       const bf_weights *weights, void *stream);

/* bf_hierarchical_neighbor_allreduce (R12): y = (W_M kron J_L/L) x:
 * intra-machine average, machine-level neighbour averaging, broadcast.
 * machine_weights: NULL (static machine topology) or an array of
 * agents_per_proc views whose ranks are MACHINE ranks (self + src, pull form;
 * every agent of a machine must pass the same view). */
bf_status bf_hierarchical_neighbor_allreduce(bf_ctx *ctx, const void *x, void *y, size_t count,
                                             bf_dtype dtype, const bf_weights *machine_weights,
                                             void *stream);
/* NVLS for the hierarchical calls when a machine spans processes ("intra-
 * machine allreduce"): register this process's copy `uc` of a
 * multicast-backed buffer of `bytes` bytes shared by the processes of its machine,
 * and the buffer's multicast address `mc` (the caller allocates it -- e.g. torch
 * symmetric memory rendezvous over the machine's process group, api.py
 * Context.enable_nvls).  Then fp32 hierarchical calls with machines of local_size
 * agents (> agents_per_proc) and a static machine topology average each machine
 * with one multimem.ld_reduce per 16 bytes through the switch, before the
 * machine-level exchange.  The buffer holds 4 x count fp32 (partial sums and
 * machine averages, each double-buffered).
 * uc = NULL and mc = 0 unregister.  Local (not collective); every process of the
 * context must register for the path to be used consistently. */
bf_status bf_hier_set_multicast(bf_ctx *ctx, int local_size, void *uc, unsigned long long mc, size_t bytes);
/* Hierarchical ATC / AWC steps (H-ATC, H-AWC: caption P:869, Table):
 *   H-ATC (Eq. 17 with the hierarchical combine):  x <- (W_M kron J_L/L)(x - lr g)
 *   H-AWC (Eq. 16 with the hierarchical combine):  x <- (W_M kron J_L/L) x - lr g
 * x: fp32 [agents_per_proc][count], updated in place; g: fp32 or bf16, same
 * layout.  One kernel per call: the adapt is fused into the publish (H-ATC)
 * or the final write (H-AWC).  Device tensors only; machine_weights and errors
 * as bf_hierarchical_neighbor_allreduce; collective like it. */
bf_status bf_hierarchical_atc_step(bf_ctx *ctx, float *x, const void *g, bf_dtype g_dtype, size_t count, float lr,
                                   const bf_weights *machine_weights, void *stream);
bf_status bf_hierarchical_awc_step(bf_ctx *ctx, float *x, const void *g, bf_dtype g_dtype, size_t count, float lr,
                                   const bf_weights *machine_weights, void *stream);

/* ---- one-sided windows (async push-sum P:551-585) -------------------
 * bf_win_create (collective): registers the stacked tensor x (borrowed until
 * bf_win_free) and allocates, for every local agent and every in-neighbour of
 * the CURRENT static topology (ascending rank), a double-buffered slot
 * (R11).  zero_init != 0: slots start at 0; else at a copy of the
 * local tensor (R10).  with_p != 0 adds the push-sum weight p (fp64, starts at
 * 1) that travels with every payload. */
bf_status bf_win_create(bf_ctx *ctx, const char *name, void *x, size_t count, bf_dtype dtype,
                        int zero_init, int with_p);
bf_status bf_win_free(bf_ctx *ctx, const char *name);
/* Symmetric-heap allocation (collective: same sizes in the same order on every
 * process, so the block has the same offset in every heap).  *ptr receives a
 * device pointer that stays valid until bf_finalize; never freed separately.
 * BF_ERR_NOMEM when the heap is exhausted. */
bf_status bf_alloc(bf_ctx *ctx, size_t bytes, void **ptr);
/* neighbor_win_get (reading R26): for every local agent in agent_mask
 * (0 = all) and every in-neighbour j at window creation selected by weights[a]
 * (src ranks + weights; self_weight required by the view rules but ignored;
 * NULL = every in-neighbour with weight 1), copy weight * x_j -- j's window
 * tensor as it is in memory now -- into this agent's slot for j and release a
 * new version, so bf_win_update sees it as the latest payload.  The window
 * tensor must live in the symmetric heap (bf_alloc), because other processes
 * read it; else BF_ERR_UNSUPPORTED.  Stream-ordered, one-sided (no call on the
 * owners).  Mixing get with put / accumulate on the same window is a race (as
 * with MPI windows without a mutex). */
bf_status bf_win_get(bf_ctx *ctx, const char *name, const bf_weights *weights, uint64_t agent_mask,
                     void *stream);
/* Error feedback for a bf16 window (reading R24 in DESIGN.md; not in the
 * paper).  Payloads travel in the window dtype, so a bf16 payload is rounded
 * (RNE) like BlueFog's MPI window in the tensor dtype; with enable != 0 the
 * sender keeps the rounding residual in its fp32 outbox and adds it to the next
 * payload to that destination, so the total mass sum_i x_i + in-flight is
 * conserved exactly at the cost of 8 B of outbox traffic per element
 * and round.  Off by default (BF_WIN_EF=1 at bf_init turns it on for new
 * windows).  Local, not collective; BF_ERR_WINDOW for an unknown name. */
bf_status bf_win_set_error_feedback(bf_ctx *ctx, const char *name, int enable);
/* put / accumulate of the REGISTERED window tensor (the paper's win_put(tensor,
 * name) passes the tensor given to win_create, Listing 3; SURVEY
 * 8(b)'s optional x argument is therefore not taken) by the local agents
 * selected in agent_mask (bit a = local
 * agent a; 0 = all): for each dst j in weights[a] (self + dst only; dst must
 * be out-neighbours at creation) deliver s_ja * x_a into j's slot for a
 * (put: overwrite, accumulate: add), then x_a <- self_weight * x_a
 * (R8).  A payload whose destination half is still unconsumed waits in a
 * sender-side outbox and is delivered by a later call (no remote
 * read-modify-write, no lock; require_mutex is accepted, the versioned
 * single-producer/single-consumer slot IS the mutex). weights == NULL:
 * all out-neighbours with 1/(outdegree+1) (Listing 3). */
bf_status bf_win_put(bf_ctx *ctx, const char *name, const bf_weights *weights,
                     uint64_t agent_mask, void *stream);
bf_status bf_win_accumulate(bf_ctx *ctx, const char *name, const bf_weights *weights,
                            int require_mutex, uint64_t agent_mask, void *stream);
/* Gradient-in-window push (SGP-style push-sum SGD): one kernel
 * does the local step x_a <- x_a - lr g_a (Eq. 4) and then exactly what
 * bf_win_accumulate does with the updated x_a (payloads s_ja x_a to the
 * destinations, x_a <- self_weight x_a).  g: device tensor of the
 * window's dtype and layout [agents_per_proc][count].  The push-sum weight p is
 * not touched by the step (it scales only the numerator).  Errors as
 * bf_win_accumulate; BF_ERR_ARG for a null / host gradient or non-finite lr. */
bf_status bf_win_accumulate_grad(bf_ctx *ctx, const char *name, const void *g, float lr, const bf_weights *weights,
                                 uint64_t agent_mask, void *stream);
/* bf_win_update: out_a = self_w * x_a + sum_j r_aj * (latest
 * complete payload from j); weights NULL = uniform 1/(d_in+1) (R10); out NULL =
 * in place.  Marks the read payloads consumed; slots are not reset. */
bf_status bf_win_update(bf_ctx *ctx, const char *name, const bf_weights *weights, void *out,
                        uint64_t agent_mask, void *stream);
/* bf_win_update_then_collect (R9): x_a += every delivered, not yet
 * consumed payload (and p += its p), then release the halves.  In place. */
bf_status bf_win_update_then_collect(bf_ctx *ctx, const char *name, uint64_t agent_mask,
                                     void *stream);
/* Host reads (synchronize `stream` first): p of every local agent (fp64
 * [agents_per_proc]), and the slot counters of (dst local agent, src rank). */
bf_status bf_win_get_p(bf_ctx *ctx, const char *name, double *p_host, void *stream);
bf_status bf_win_counters(bf_ctx *ctx, const char *name, int dst_local, int src_rank,
                          uint64_t *version, uint64_t *consumed);
/* SURVEY 8(b) bf_win_version: the version counter (payloads delivered so far) of
 * the slot that receives from src_rank, for the first local agent (ascending)
 * that has src_rank as an in-neighbour at window creation -- with one agent per
 * process (the paper's model) that is the process's agent.  bf_win_counters
 * gives both counters of any (local agent, source) pair. */
bf_status bf_win_version(bf_ctx *ctx, const char *name, int src_rank, uint64_t *version);
/* Slot layout of agent `agent` (P:388 pin): element offset of the slot that
 * receives from `src_rank` in the paper's logical numel*d_in layout, or -1. */
long long bf_win_slot_offset(bf_ctx *ctx, const char *name, int agent, int src_rank);

/* ---- misc ----------------------------------------------------------------------- */
bf_status bf_barrier(bf_ctx *ctx, void *stream);      /* device barrier over all processes */
bf_status bf_poll_error(bf_ctx *ctx);                 /* latched device fault, non-blocking */
/* Reserve exchange capacity (collective; optional -- the first call reserves
 * what it needs): bytes per agent of the largest message. */
bf_status bf_reserve(bf_ctx *ctx, size_t bytes_per_agent);
/* Synthetic input generator (same counter-based
 * generator as synthetic/__init__.py): dst[i] = u(seed, offset+i) * scale. */
bf_status bf_fill_uniform(void *dst, bf_dtype dtype, size_t count, uint64_t seed,
                          uint64_t offset, float scale, void *stream);
/* Number of kernels the library launched so far on this context (bench accounting). */
uint64_t bf_kernel_launches(const bf_ctx *ctx);

/* Diagnostics (not part of the paper's API).  With the environment variable
 * BF_STATS=1 at bf_init and a library built with -DBF_STATS=1, the fused
 * exchange kernel accumulates per-CTA timings into a device buffer of
 * 4096 x 8 u64: [0] kernel ns, [1] consumer ns waiting for remote tiles,
 * [2] communication-warp ns blocked on peers' progress, [3] ns blocked on ring
 * slots, [4] release-fence ns, [5] fences, [6] progress polls, [7] prologue ns.
 * Copies min(cap, 4096 * 8) values to the host buffer `out` (synchronises the
 * device) and zeroes the buffer if `reset`.  BF_ERR_STATE if BF_STATS was not
 * set at bf_init; BF_ERR_ARG on null arguments. */
bf_status bf_exchange_stats(bf_ctx *ctx, uint64_t *out, size_t cap, int reset);

#ifdef __cplusplus
}
#endif
#endif /* BLUEFOG_B200_H */
