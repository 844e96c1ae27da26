/*
 * bf_oracle.c -- CPU reference ("oracle") for the BlueFog hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see bf_oracle.h).  Plain single-threaded fp64 C,
 * each function written in the order of the paper passage it cites.
 * Compiled with -O2 -ffp-contract=off (no fused multiply-add, no fast-math).
 *
 * Readings of the paper where it is silent or garbled are the numbered rows
 * "R<k>" of DESIGN.md "Readings of the paper".
 */
#include "bf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ========================================================================
 * Topologies (global view).  P:334-339 "set_topology(graph_object)"; the
 * built-ins are named at P:339 and P:447.
 * ====================================================================== */

/* Undirected ring, uniform weights over {i-1, i, i+1} (P:986 ring
 * graph used for Exact-Diffusion).  n = 2 has a single neighbour: 1/2. */
void ora_ring(int n, double *W) {
    memset(W, 0, sizeof(double) * (size_t)n * n);
    if (n == 1) { W[0] = 1.0; return; }
    if (n == 2) { W[0] = W[1] = W[2] = W[3] = 0.5; return; }
    for (int i = 0; i < n; ++i) {
        W[i * n + i] = 1.0 / 3.0;
        W[i * n + (i + 1) % n] = 1.0 / 3.0;
        W[i * n + (i + n - 1) % n] = 1.0 / 3.0;
    }
}

/* Static exponential-2 graph (P:446 cites [ying2021exponential]; reading R4):
 * directed edges i -> i + 2^j (mod n), j = 0..floor(log2(n-1)); node i
 * receives from i - 2^j; uniform weight 1/(deg+1) on self and in-edges. */
void ora_exp2(int n, double *W) {
    memset(W, 0, sizeof(double) * (size_t)n * n);
    if (n == 1) { W[0] = 1.0; return; }
    int deg = 0;
    for (int off = 1; off <= n - 1; off *= 2) ++deg;
    double w = 1.0 / (deg + 1);
    for (int i = 0; i < n; ++i) {
        W[i * n + i] = w;
        for (int off = 1; off <= n - 1; off *= 2)
            W[i * n + ((i - off) % n + n) % n] += w;
    }
}

/* Fully connected, uniform 1/n (default topology, reading R15). */
void ora_full(int n, double *W) {
    for (int i = 0; i < n * n; ++i) W[i] = 1.0 / n;
}

static int ceil_log2(int n) {
    int t = 0;
    while ((1 << t) < n) ++t;
    return t;
}

/* One-peer dynamic exponential graph ("each process only picks one
 * neighbor at each iteration"; reading R5): at round k, t = k mod ceil(log2 n),
 * node i pulls from i - 2^t and pushes to i + 2^t, self 1/2, effective 1/2. */
void ora_one_peer_exp2_peers(int n, long long k, int i, int *src, int *dst) {
    int tau = ceil_log2(n);
    if (tau == 0) { *src = -1; *dst = -1; return; }
    int off = 1 << (int)(k % tau);
    *src = ((i - off) % n + n) % n;
    *dst = (i + off) % n;
}

void ora_one_peer_exp2(int n, long long k, double *W) {
    memset(W, 0, sizeof(double) * (size_t)n * n);
    if (n == 1) { W[0] = 1.0; return; }
    for (int i = 0; i < n; ++i) {
        int src, dst;
        ora_one_peer_exp2_peers(n, k, i, &src, &dst);
        W[i * n + i] = 0.5;
        W[i * n + src] += 0.5;
    }
}

/* Inner-outer dynamic exponential-2 graph (named, not defined, in P:828 and
 * the caption at P:869; reading R27).  n agents on M = n / L machines of L.
 * At round k one local rank per machine, o = k mod L, talks OUTSIDE: agent
 * (m, o) pulls from machine m - 2^t (same local rank o) and pushes to m + 2^t,
 * t = (k div L) mod ceil(log2 M).  The other L - 1 agents of the machine talk
 * INSIDE: relabelled r = (l - o - 1) mod L in [0, L - 2], they run the one-peer
 * exp-2 rule over a group of L - 1, t' = k mod ceil(log2(L - 1)), and map back
 * l = (r + o + 1) mod L.  A group of one has no peer (self weight 1). */
void ora_inner_outer_exp2_peers(int n, int L, long long k, int i, int *src, int *dst) {
    int M = n / L, m = i / L, l = i % L;
    int o = (int)(k % L);
    *src = -1;
    *dst = -1;
    if (l == o) {
        int tau = ceil_log2(M);
        if (tau == 0) return;
        int off = 1 << (int)((k / L) % tau);
        *src = ((m - off) % M + M) % M * L + o;
        *dst = (m + off) % M * L + o;
    } else {
        int G = L - 1;
        int tau = ceil_log2(G);
        if (tau == 0) return;
        int off = 1 << (int)(k % tau);
        int r = ((l - o - 1) % L + L) % L;
        int rs = ((r - off) % G + G) % G, rd = (r + off) % G;
        *src = m * L + (rs + o + 1) % L;
        *dst = m * L + (rd + o + 1) % L;
    }
}

void ora_inner_outer_exp2(int n, int L, long long k, double *W) {
    memset(W, 0, sizeof(double) * (size_t)n * n);
    for (int i = 0; i < n; ++i) {
        int src, dst;
        ora_inner_outer_exp2_peers(n, L, k, i, &src, &dst);
        if (src < 0) {
            W[i * n + i] = 1.0;
        } else {
            W[i * n + i] = 0.5;
            W[i * n + src] += 0.5;
        }
    }
}

/* ========================================================================
 * Neighbour sets, Eq. 6-7: N(i) = {j : (j,i) in E},
 * M(i) = {j : (i,j) in E}; E = {(j,i) : w_ij != 0}.
 * ====================================================================== */
int ora_in_neighbors(int n, const double *W, int i, int *out) {
    int c = 0;
    for (int j = 0; j < n; ++j)
        if (j != i && W[i * n + j] != 0.0) out[c++] = j;
    return c;
}

int ora_out_neighbors(int n, const double *W, int i, int *out) {
    int c = 0;
    for (int j = 0; j < n; ++j)
        if (j != i && W[j * n + i] != 0.0) out[c++] = j;
    return c;
}

/* Weight classes: pull = every row sums to 1, push = every
 * column sums to 1, standard = both. */
int ora_classify(int n, const double *W, double tol) {
    int rows = 1, cols = 1;
    for (int i = 0; i < n; ++i) {
        double r = 0.0, c = 0.0;
        for (int j = 0; j < n; ++j) { r += W[i * n + j]; c += W[j * n + i]; }
        if (fabs(r - 1.0) > tol) rows = 0;
        if (fabs(c - 1.0) > tol) cols = 0;
    }
    return rows | (cols << 1);
}

/* ========================================================================
 * Local views -> W.  Eq. 9: x_i <- w_ii x_i + sum_j r_ij s_ij x_j,
 * with the four argument configurations of the P:381 footnote:
 *   pull (self+src): s = 1 unless the sender also declared i (reading R1);
 *   push (self+dst): r = 1, the receiver learns its sources from senders;
 *   push-pull: r*s, and every declaration must be matched.
 * ====================================================================== */
static int view_has_dst(const ora_view *v, int i, double *s_out) {
    for (int q = 0; q < v->n_dst; ++q)
        if (v->dst[q] == i) { if (s_out) *s_out = v->s[q]; return 1; }
    return 0;
}

int ora_assemble(int n, const ora_view *views, int check, double *W) {
    memset(W, 0, sizeof(double) * (size_t)n * n);
    for (int i = 0; i < n; ++i) {
        const ora_view *vi = &views[i];
        W[i * n + i] = vi->self_weight;
        if (vi->n_src >= 0) {
            /* receiver declares its sources (pull or push-pull): r_ij times
             * s_ij when the sender also declared i, else s = 1 (R1). */
            for (int q = 0; q < vi->n_src; ++q) {
                int j = vi->src[q];
                double s = 1.0;
                int declared = view_has_dst(&views[j], i, &s);
                if (!declared) s = 1.0;
                /* a sender that declares destinations but not i: i would wait
                 * for a message that never comes */
                if (check && views[j].n_dst >= 0 && !declared) return -(1 + i);
                W[i * n + j] = vi->r[q] * s;
            }
            if (check) {
                /* every sender that pushes to i must be a declared source */
                for (int j = 0; j < n; ++j) {
                    if (j == i || !view_has_dst(&views[j], i, NULL)) continue;
                    int listed = 0;
                    for (int q = 0; q < vi->n_src; ++q) listed |= (vi->src[q] == j);
                    if (!listed) return -(1 + i);
                }
            }
        } else {
            /* push-only or isolated receiver: sources are the senders that
             * declared i among their destinations, weight s (r = 1). */
            for (int j = 0; j < n; ++j) {
                double s;
                if (j != i && view_has_dst(&views[j], i, &s)) W[i * n + j] = s;
            }
        }
    }
    return 0;
}

/* ========================================================================
 * Partial averaging, Eq. 5:  x_i <- w_ii x_i + sum_{j in N(i)} w_ij x_j
 * written as the plain product Y = W X.
 * ====================================================================== */
void ora_mix(int n, long long count, const double *W, const double *X, double *Y) {
    for (int i = 0; i < n; ++i)
        for (long long e = 0; e < count; ++e) {
            double acc = 0.0;
            for (int j = 0; j < n; ++j)
                acc += W[i * n + j] * X[(long long)j * count + e];
            Y[(long long)i * count + e] = acc;
        }
}

/* ========================================================================
 * Casts (reading R17: round-to-nearest-even).
 * ====================================================================== */
float ora_f32(double v) { return (float)v; }

uint16_t ora_bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7FFFFFFFu) > 0x7F800000u) return (uint16_t)((u >> 16) | 0x40u); /* quiet NaN */
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7FFFu + lsb;
    return (uint16_t)(u >> 16);
}

static double bf16_value(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* ========================================================================
 * ATC-DSGD step.  Eq. 4 local update, then Eq. 5 partial
 * averaging of the adapted copies (ATC, Eq. 17, reading R6).
 * ====================================================================== */
void ora_atc(int n, long long count, const double *W, const double *X,
             const double *G, double lr, int wire_bf16, double *Y) {
    double *xh = (double *)malloc(sizeof(double) * (size_t)n * count);
    double *wire = (double *)malloc(sizeof(double) * (size_t)n * count);
    /* Eq. 4: x_i^{k+1/2} = x_i^k - gamma * g_i, held as fp32 (reading R18) */
    for (long long q = 0; q < (long long)n * count; ++q) {
        xh[q] = (double)ora_f32(X[q] - lr * G[q]);
        wire[q] = wire_bf16 ? bf16_value(ora_bf16_rne((float)xh[q])) : xh[q];
    }
    /* Eq. 5: self term from the unrounded x^{k+1/2}, neighbours from the wire */
    for (int i = 0; i < n; ++i)
        for (long long e = 0; e < count; ++e) {
            double acc = W[i * n + i] * xh[(long long)i * count + e];
            for (int j = 0; j < n; ++j)
                if (j != i) acc += W[i * n + j] * wire[(long long)j * count + e];
            Y[(long long)i * count + e] = acc;
        }
    free(xh);
    free(wire);
}

/* Exact-Diffusion, appendix Eqs. ed-1..ed-3 (Listing ED-static):
 *   psi_i^(k) = x_i^(k) - gamma * g_i                 (local update; stored as fp32 state, R25)
 *   phi_i^(k) = psi_i^(k) + x_i^(k) - psi_i^(k-1)     (bias correction; defined value fp32, R25)
 *   x_i^(k+1) = w_ii phi_i^(k) + sum_j w_ij phi_j^(k) (partial averaging; neighbours' phi as on the wire)
 * Psi_prev holds psi^(k-1); Psi_out receives psi^(k). */
void ora_exact_diffusion(int n, long long count, const double *W, const double *X, const double *G,
                         const double *Psi_prev, double lr, int wire_bf16, double *Y, double *Psi_out) {
    double *phi = (double *)malloc(sizeof(double) * (size_t)n * count);
    double *wire = (double *)malloc(sizeof(double) * (size_t)n * count);
    for (long long q = 0; q < (long long)n * count; ++q) {
        const double psi = (double)ora_f32(X[q] - lr * G[q]);
        Psi_out[q] = psi;
        phi[q] = (double)ora_f32(psi + X[q] - Psi_prev[q]);
        wire[q] = wire_bf16 ? bf16_value(ora_bf16_rne((float)phi[q])) : phi[q];
    }
    for (int i = 0; i < n; ++i)
        for (long long e = 0; e < count; ++e) {
            double acc = W[i * n + i] * phi[(long long)i * count + e];
            for (int j = 0; j < n; ++j)
                if (j != i) acc += W[i * n + j] * wire[(long long)j * count + e];
            Y[(long long)i * count + e] = acc;
        }
    free(phi);
    free(wire);
}

/* AWC, Eq. 16: x_i^k = sum_{j in N+(i)} w_ij x_j^{k-1} - gamma g_i. */
void ora_awc(int n, long long count, const double *W, const double *X,
             const double *G, double lr, double *Y) {
    ora_mix(n, count, W, X, Y);
    for (long long q = 0; q < (long long)n * count; ++q) Y[q] -= lr * G[q];
}

/* ========================================================================
 * Hierarchical neighbour allreduce: (1) intra-machine average,
 * (2) machine-level neighbour averaging with W_M, (3) every local node takes
 * the machine result.  machine_rank = rank // local_size.
 * Reading R12: stage (1) is an average (SUM / local_size).
 * ====================================================================== */
void ora_hier(int n_machines, int L, long long count, const double *WM,
              const double *X, double *Y) {
    double *avg = (double *)calloc((size_t)n_machines * count, sizeof(double));
    for (int m = 0; m < n_machines; ++m)                     /* stage 1 */
        for (long long e = 0; e < count; ++e) {
            double s = 0.0;
            for (int l = 0; l < L; ++l) s += X[(long long)(m * L + l) * count + e];
            avg[(long long)m * count + e] = s / L;
        }
    for (int m = 0; m < n_machines; ++m)                     /* stage 2 + 3 */
        for (long long e = 0; e < count; ++e) {
            double z = 0.0;
            for (int q = 0; q < n_machines; ++q)
                z += WM[m * n_machines + q] * avg[(long long)q * count + e];
            for (int l = 0; l < L; ++l) Y[(long long)(m * L + l) * count + e] = z;
        }
    free(avg);
}

/* H-ATC (caption P:869; Table): the ATC step of Eq. 17 with
 * the hierarchical combine of P:660 in place of W.  The adapted copy is held as
 * fp32 (reading R18, as in ora_atc):  Y = (W_M kron J_L/L) fp32(X - lr G). */
void ora_hier_atc(int n_machines, int L, long long count, const double *WM,
                  const double *X, const double *G, double lr, double *Y) {
    const long long N = (long long)n_machines * L * count;
    double *xh = (double *)malloc(sizeof(double) * (size_t)N);
    for (long long q = 0; q < N; ++q) xh[q] = (double)ora_f32(X[q] - lr * G[q]);   /* Eq. 4 */
    ora_hier(n_machines, L, count, WM, xh, Y);
    free(xh);
}

/* H-AWC (caption P:869): Eq. 16 with the hierarchical combine:
 * Y = (W_M kron J_L/L) X - lr G. */
void ora_hier_awc(int n_machines, int L, long long count, const double *WM,
                  const double *X, const double *G, double lr, double *Y) {
    const long long N = (long long)n_machines * L * count;
    ora_hier(n_machines, L, count, WM, X, Y);
    for (long long q = 0; q < N; ++q) Y[q] -= lr * G[q];
}

/* ========================================================================
 * Push-sum gradient tracking (appendix "Push-sum gradient tracking",
 * PAPER.md lines 1000-1006, listing GT-varying), split at the gradient
 * evaluation the caller performs between the two halves of a round:
 *   (a) u_i^{k+1} = sum_j w_ij (u_j^k - gamma y_j^k)          (line 1002)
 *       v_i^{k+1} = sum_j w_ij v_j^k                            (line 1003)
 *       x_i^{k+1} = u_i^{k+1} / v_i^{k+1}                       (line 1004)
 *   (b) y_i^{k+1} = sum_j w_ij (y_j^k + g_j^{k+1} - g_j^k)     (line 1006)
 * U, Y, G*: n x d; V: n x dv with dv = d (the paper's vector v) or dv = 1 (one
 * push-sum weight per agent: v^0 = 1 keeps every entry of v equal). */
void ora_gt_uv(int n, long long d, long long dv, const double *W, const double *U, const double *V,
               const double *Y, double lr, double *Un, double *Vn, double *Xn) {
    double *w = (double *)malloc(sizeof(double) * (size_t)n * d);
    for (long long q = 0; q < (long long)n * d; ++q) w[q] = U[q] - lr * Y[q];
    ora_mix(n, d, W, w, Un);
    ora_mix(n, dv, W, V, Vn);
    for (int i = 0; i < n; ++i)
        for (long long e = 0; e < d; ++e)
            Xn[(long long)i * d + e] = Un[(long long)i * d + e] / Vn[(long long)i * dv + (dv == 1 ? 0 : e)];
    free(w);
}

void ora_gt_y(int n, long long d, const double *W, const double *Y, const double *Gnew,
              const double *Gprev, double *Yn) {
    double *q = (double *)malloc(sizeof(double) * (size_t)n * d);
    for (long long e = 0; e < (long long)n * d; ++e) q[e] = Y[e] + Gnew[e] - Gprev[e];
    ora_mix(n, d, W, q, Yn);
    free(q);
}

/* ========================================================================
 * Window protocol event model (P:388-423 windows; P:551-585 async push-sum).
 * One slot per static in-neighbour in ascending rank, each with two
 * halves (reading R11).  Producer i -> consumer j: payload m lands in half
 * m&1 when the consumer has consumed payload m-2 (consumed >= version-1);
 * otherwise it stays in i's outbox (sender-side accumulation, no remote
 * read-modify-write).  Collect sums the ready payloads and releases them
 * (P:585 sum-and-reset, reading R9).  self_weight scales x in place (R8).
 * ====================================================================== */
struct ora_win {
    int n;
    long long count;
    int *nin, *in;          /* in[i*n + q]: q-th in-neighbour of i */
    int *nout, *out;        /* out[i*n + q] */
    double *x;              /* n * count */
    double *slot;           /* [dst][q][half][count] with q < n */
    long long *version, *consumed;  /* [dst*n + q] */
    double *outbox;         /* [src][q][count], q indexes out[src] */
    int *outbox_valid;      /* [src*n + q] */
};

static double *slot_ptr(const ora_win *w, int dst, int q, int half) {
    return w->slot + (((size_t)dst * w->n + q) * 2 + half) * w->count;
}

ora_win *ora_win_create(int n, long long count, const double *Wstatic,
                        const double *X0, int zero_init) {
    ora_win *w = (ora_win *)calloc(1, sizeof(ora_win));
    w->n = n;
    w->count = count;
    w->nin = (int *)calloc(n, sizeof(int));
    w->in = (int *)calloc((size_t)n * n, sizeof(int));
    w->nout = (int *)calloc(n, sizeof(int));
    w->out = (int *)calloc((size_t)n * n, sizeof(int));
    for (int i = 0; i < n; ++i) {
        w->nin[i] = ora_in_neighbors(n, Wstatic, i, w->in + (size_t)i * n);
        w->nout[i] = ora_out_neighbors(n, Wstatic, i, w->out + (size_t)i * n);
    }
    w->x = (double *)malloc(sizeof(double) * (size_t)n * count);
    memcpy(w->x, X0, sizeof(double) * (size_t)n * count);
    w->slot = (double *)calloc((size_t)n * n * 2 * count, sizeof(double));
    w->version = (long long *)calloc((size_t)n * n, sizeof(long long));
    w->consumed = (long long *)calloc((size_t)n * n, sizeof(long long));
    w->outbox = (double *)calloc((size_t)n * n * count, sizeof(double));
    w->outbox_valid = (int *)calloc((size_t)n * n, sizeof(int));
    if (!zero_init) {
        /* buffers start as a copy of the local tensor (reading R10); the copy
         * sits in half 1, the "latest" half while version == 0. */
        for (int i = 0; i < n; ++i)
            for (int q = 0; q < w->nin[i]; ++q)
                memcpy(slot_ptr(w, i, q, 1), w->x + (size_t)i * count, sizeof(double) * count);
    }
    return w;
}

void ora_win_free(ora_win *w) {
    if (!w) return;
    free(w->nin); free(w->in); free(w->nout); free(w->out); free(w->x);
    free(w->slot); free(w->version); free(w->consumed); free(w->outbox);
    free(w->outbox_valid); free(w);
}

static int in_index(const ora_win *w, int dst, int src) {
    for (int q = 0; q < w->nin[dst]; ++q)
        if (w->in[(size_t)dst * w->n + q] == src) return q;
    return -1;
}

int ora_win_accumulate(ora_win *w, int i, double self_weight, const double *s,
                       const int *dst_mask, int overwrite) {
    long long C = w->count;
    for (int q = 0; q < w->nout[i]; ++q) {
        int j = w->out[(size_t)i * w->n + q];
        if (!dst_mask[j]) continue;
        int qi = in_index(w, j, i);
        if (qi < 0) return -1;
        double *ob = w->outbox + ((size_t)i * w->n + q) * C;
        int *valid = &w->outbox_valid[(size_t)i * w->n + q];
        /* payload = (outbox +) s_ji * x_i   (push-style scaling, Eq. 10) */
        for (long long e = 0; e < C; ++e) {
            double base = (!overwrite && *valid) ? ob[e] : 0.0;
            ob[e] = base + s[j] * w->x[(size_t)i * C + e];
        }
        *valid = 1;
        long long *ver = &w->version[(size_t)j * w->n + qi];
        long long con = w->consumed[(size_t)j * w->n + qi];
        if (con >= *ver - 1) {          /* half (version & 1) is free */
            memcpy(slot_ptr(w, j, qi, (int)(*ver & 1)), ob, sizeof(double) * C);
            *ver += 1;
            *valid = 0;
        }
    }
    for (long long e = 0; e < C; ++e) w->x[(size_t)i * C + e] *= self_weight;
    return 0;
}

/* Local SGD step inside a window, before a push (SGP-style gradient-in-window,
 * SURVEY 8(f) rank 4): x_i <- x_i - lr g_i (Eq. 4) on the window tensor;
 * the p lane (the last element when the caller appends it) gets g = 0. */
void ora_win_adapt(ora_win *w, int i, const double *g, double lr) {
    for (long long e = 0; e < w->count; ++e) w->x[(size_t)i * w->count + e] -= lr * g[e];
}

void ora_win_collect(ora_win *w, int i) {
    long long C = w->count;
    for (int q = 0; q < w->nin[i]; ++q) {
        long long *con = &w->consumed[(size_t)i * w->n + q];
        long long ver = w->version[(size_t)i * w->n + q];
        while (*con < ver) {
            const double *h = slot_ptr(w, i, q, (int)(*con & 1));
            for (long long e = 0; e < C; ++e) w->x[(size_t)i * C + e] += h[e];
            *con += 1;
        }
    }
}

void ora_win_update(ora_win *w, int i, double self_weight, const double *r, double *out) {
    long long C = w->count;
    for (long long e = 0; e < C; ++e) out[e] = self_weight * w->x[(size_t)i * C + e];
    for (int q = 0; q < w->nin[i]; ++q) {
        int j = w->in[(size_t)i * w->n + q];
        long long ver = w->version[(size_t)i * w->n + q];
        const double *h = slot_ptr(w, i, q, (int)((ver - 1) & 1));
        for (long long e = 0; e < C; ++e) out[e] += r[j] * h[e];
        w->consumed[(size_t)i * w->n + q] = ver;   /* reading R10 */
    }
}

void ora_win_get_x(const ora_win *w, double *X) {
    memcpy(X, w->x, sizeof(double) * (size_t)w->n * w->count);
}

double ora_win_mass(const ora_win *w, long long e) {
    long long C = w->count;
    double m = 0.0;
    for (int i = 0; i < w->n; ++i) {
        m += w->x[(size_t)i * C + e];
        for (int q = 0; q < w->nout[i]; ++q)
            if (w->outbox_valid[(size_t)i * w->n + q])
                m += w->outbox[((size_t)i * w->n + q) * C + e];
        for (int q = 0; q < w->nin[i]; ++q)
            for (long long p = w->consumed[(size_t)i * w->n + q];
                 p < w->version[(size_t)i * w->n + q]; ++p)
                m += slot_ptr(w, i, q, (int)(p & 1))[e];
    }
    return m;
}

void ora_win_counters(const ora_win *w, int dst, int src, long long *version,
                      long long *consumed) {
    int q = in_index(w, dst, src);
    *version = q < 0 ? -1 : w->version[(size_t)dst * w->n + q];
    *consumed = q < 0 ? -1 : w->consumed[(size_t)dst * w->n + q];
}

/* ========================================================================
 * Least squares (Eq. 12) and its local gradient (Eq. 13,
 * P:440): g_i = A_i^T (A_i x - b_i).  x* solves the normal equations
 * sum_i A_i^T A_i x = sum_i A_i^T b_i, here by plain conjugate gradients.
 * ====================================================================== */
void ora_lsq_grad(int m, int d, const double *A, const double *b, const double *x, double *g) {
    double *res = (double *)malloc(sizeof(double) * m);
    for (int r = 0; r < m; ++r) {
        double acc = 0.0;
        for (int c = 0; c < d; ++c) acc += A[(size_t)r * d + c] * x[c];
        res[r] = acc - b[r];
    }
    for (int c = 0; c < d; ++c) g[c] = 0.0;
    for (int r = 0; r < m; ++r)
        for (int c = 0; c < d; ++c) g[c] += A[(size_t)r * d + c] * res[r];
    free(res);
}

static void normal_matvec(int n, int m, int d, const double *A, const double *v, double *out) {
    double *zero = (double *)calloc(m, sizeof(double));
    double *gi = (double *)malloc(sizeof(double) * d);
    for (int c = 0; c < d; ++c) out[c] = 0.0;
    for (int i = 0; i < n; ++i) {
        ora_lsq_grad(m, d, A + (size_t)i * m * d, zero, v, gi);   /* A_i^T A_i v */
        for (int c = 0; c < d; ++c) out[c] += gi[c];
    }
    free(zero);
    free(gi);
}

int ora_lsq_solve(int n, int m, int d, const double *A, const double *b, double tol,
                  int max_iter, double *x) {
    double *rhs = (double *)calloc(d, sizeof(double));
    double *r = (double *)malloc(sizeof(double) * d);
    double *p = (double *)malloc(sizeof(double) * d);
    double *Ap = (double *)malloc(sizeof(double) * d);
    for (int i = 0; i < n; ++i)
        for (int row = 0; row < m; ++row)
            for (int c = 0; c < d; ++c)
                rhs[c] += A[((size_t)i * m + row) * d + c] * b[(size_t)i * m + row];
    for (int c = 0; c < d; ++c) x[c] = 0.0;
    double rr = 0.0, rhs2 = 0.0;
    for (int c = 0; c < d; ++c) { r[c] = rhs[c]; p[c] = r[c]; rr += r[c] * r[c]; }
    rhs2 = rr;
    int it = 0;
    while (it < max_iter && sqrt(rr) > tol * sqrt(rhs2)) {
        normal_matvec(n, m, d, A, p, Ap);
        double pAp = 0.0;
        for (int c = 0; c < d; ++c) pAp += p[c] * Ap[c];
        double alpha = rr / pAp;
        double rr_new = 0.0;
        for (int c = 0; c < d; ++c) {
            x[c] += alpha * p[c];
            r[c] -= alpha * Ap[c];
            rr_new += r[c] * r[c];
        }
        double beta = rr_new / rr;
        for (int c = 0; c < d; ++c) p[c] = r[c] + beta * p[c];
        rr = rr_new;
        ++it;
    }
    free(rhs); free(r); free(p); free(Ap);
    return it;
}

/* ========================================================================
 * Paper-semantics window (P:388-403 windows, P:417-423 win_update, P:585
 * collect), written as the paper states it, with NO protocol: one buffer per
 * static in-neighbour (ascending rank);
 *   put        : buffer_i[j] <- s_ji x_j
 *   accumulate : buffer_i[j] <- buffer_i[j] + s_ji x_j
 *   both then  : x_j <- self_weight x_j                      (reading R8)
 *   collect    : x_i <- x_i + sum_j buffer_i[j]; buffers <- 0 (R9)
 *   update     : out = self_w x_i + sum_j r_j buffer_i[j]     (no reset)
 * It is the reference the double-buffered / outbox event model above must
 * equal whenever no payload waits in an outbox (tests/test_oracle.py).
 * ====================================================================== */
struct ora_winp {
    int n;
    long long count;
    int *nin, *in;          /* in[i*n + q] */
    double *x;              /* n * count */
    double *buf;            /* [i][q][count] */
};

ora_winp *ora_winp_create(int n, long long count, const double *Wstatic, const double *X0, int zero_init) {
    ora_winp *w = (ora_winp *)calloc(1, sizeof(ora_winp));
    w->n = n;
    w->count = count;
    w->nin = (int *)calloc(n, sizeof(int));
    w->in = (int *)calloc((size_t)n * n, sizeof(int));
    for (int i = 0; i < n; ++i) w->nin[i] = ora_in_neighbors(n, Wstatic, i, w->in + (size_t)i * n);
    w->x = (double *)malloc(sizeof(double) * (size_t)n * count);
    memcpy(w->x, X0, sizeof(double) * (size_t)n * count);
    w->buf = (double *)calloc((size_t)n * n * count, sizeof(double));
    if (!zero_init)   /* buffers start as the local tensor (reading R10; P:567 zero_init) */
        for (int i = 0; i < n; ++i)
            for (int q = 0; q < w->nin[i]; ++q)
                memcpy(w->buf + ((size_t)i * n + q) * count, w->x + (size_t)i * count, sizeof(double) * count);
    return w;
}

void ora_winp_free(ora_winp *w) {
    if (!w) return;
    free(w->nin); free(w->in); free(w->x); free(w->buf); free(w);
}

int ora_winp_accumulate(ora_winp *w, int j, double self_weight, const double *s, const int *dst_mask,
                        int overwrite) {
    const long long C = w->count;
    for (int i = 0; i < w->n; ++i) {
        if (!dst_mask[i]) continue;
        int q = -1;
        for (int t = 0; t < w->nin[i]; ++t)
            if (w->in[(size_t)i * w->n + t] == j) q = t;
        if (q < 0) return -1;   /* dst outside the creation topology */
        double *b = w->buf + ((size_t)i * w->n + q) * C;
        for (long long e = 0; e < C; ++e)
            b[e] = (overwrite ? 0.0 : b[e]) + s[i] * w->x[(size_t)j * C + e];
    }
    for (long long e = 0; e < C; ++e) w->x[(size_t)j * C + e] *= self_weight;
    return 0;
}

void ora_winp_collect(ora_winp *w, int i) {
    const long long C = w->count;
    for (int q = 0; q < w->nin[i]; ++q) {
        double *b = w->buf + ((size_t)i * w->n + q) * C;
        for (long long e = 0; e < C; ++e) {
            w->x[(size_t)i * C + e] += b[e];
            b[e] = 0.0;
        }
    }
}

void ora_winp_update(const ora_winp *w, int i, double self_weight, const double *r, double *out) {
    const long long C = w->count;
    for (long long e = 0; e < C; ++e) out[e] = self_weight * w->x[(size_t)i * C + e];
    for (int q = 0; q < w->nin[i]; ++q) {
        const int j = w->in[(size_t)i * w->n + q];
        const double *b = w->buf + ((size_t)i * w->n + q) * C;
        for (long long e = 0; e < C; ++e) out[e] += r[j] * b[e];
    }
}

void ora_winp_get_x(const ora_winp *w, double *X) {
    memcpy(X, w->x, sizeof(double) * (size_t)w->n * w->count);
}

/* ========================================================================
 * ATC-DSGD fixed point on the decentralized least-squares problem (Eq. 12
 * P:432-435, DGD/ATC Eq. 13-14 P:440-441 with Eq. 17): the unique X with
 *     x_i = sum_j w_ij (x_j - gamma A_j^T (A_j x_j - b_j)),
 * found by iterating that map in fp64 from X (in: start, out: x_inf) until the
 * largest change is <= tol * max|X|.  Returns the iterations used, or -1 if
 * max_iter was reached.  A: n x m x d, b: n x m, X: n x d.
 * ====================================================================== */
int ora_atc_fixed_point(int n, int m, int d, const double *W, const double *A, const double *b, double lr,
                        double tol, int max_iter, double *X) {
    double *xh = (double *)malloc(sizeof(double) * (size_t)n * d);
    double *Xn = (double *)malloc(sizeof(double) * (size_t)n * d);
    double *g = (double *)malloc(sizeof(double) * (size_t)d);
    int it = 0;
    for (; it < max_iter; ++it) {
        for (int i = 0; i < n; ++i) {   /* Eq. 4 in fp64: x_half = x - gamma g_i(x_i) */
            ora_lsq_grad(m, d, A + (size_t)i * m * d, b + (size_t)i * m, X + (size_t)i * d, g);
            for (int c = 0; c < d; ++c) xh[(size_t)i * d + c] = X[(size_t)i * d + c] - lr * g[c];
        }
        ora_mix(n, d, W, xh, Xn);       /* Eq. 5 */
        double dmax = 0.0, xmax = 0.0;
        for (long long q = 0; q < (long long)n * d; ++q) {
            dmax = fmax(dmax, fabs(Xn[q] - X[q]));
            xmax = fmax(xmax, fabs(Xn[q]));
            X[q] = Xn[q];
        }
        if (dmax <= tol * xmax) { ++it; break; }
    }
    free(xh); free(Xn); free(g);
    return it >= max_iter ? -1 : it;
}

/* ========================================================================
 * Communication cost model, Table 1 (after [ben2019]):
 * time of one averaging of an M-byte message over n nodes with link bandwidth
 * B (bytes/s) and direct-communication latency L (s).
 *   0 parameter server   nM/B + nL        (global averaging)
 *   1 ring-allreduce     2M/B + 2nL       (global averaging)
 *   2 Byte-PS            M/B + nL         (global averaging)
 *   3 partial averaging  M/B + L          (BlueFog, one neighbour at a time;
 *                        d_in in-neighbours over independent links: still M/B + L)
 * Returns a negative value for an unknown primitive.
 * ====================================================================== */
double ora_comm_cost(int primitive, int n, double M, double B, double L) {
    switch (primitive) {
        case 0: return n * M / B + n * L;
        case 1: return 2.0 * M / B + 2.0 * n * L;
        case 2: return M / B + n * L;
        case 3: return M / B + L;
        default: return -1.0;
    }
}
