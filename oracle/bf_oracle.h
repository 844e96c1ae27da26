/*
 * bf_oracle.h -- CPU reference ("oracle") for the BlueFog hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA library
 * (paper_2111_04287_b200/csrc) and neither includes the other.
 *
 * Everything is plain, single-threaded, fp64 C following the paper's
 * equations in the paper's order.  Citations: P:NNN = reference PAPER.md
 * line, S:NNN = reference SPEC.md line (interface ideas only).
 *
 * Matrices are row-major: W[i*n + j] = w_ij, the weight node i applies to
 * x_j (Eq. 8).  Stacked agent vectors: X[i*count + e].
 */
#ifndef BF_ORACLE_H
#define BF_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- topologies (global view) -------------------------------- */
void ora_ring(int n, double *W);            /* i<->i+-1, 1/3 (n=2: 1/2) */
void ora_exp2(int n, double *W);            /* i -> i+2^j, 1/(deg+1) */
void ora_full(int n, double *W);            /* uniform 1/n */
void ora_one_peer_exp2(int n, long long k, double *W); /* P:916 dynamic one-peer */
void ora_one_peer_exp2_peers(int n, long long k, int i, int *src, int *dst);
void ora_inner_outer_exp2(int n, int L, long long k, double *W); /* P:828, R27 */
void ora_inner_outer_exp2_peers(int n, int L, long long k, int i, int *src, int *dst);

/* ---- neighbour sets and classes (Eq. 6-8) -------------------- */
int ora_in_neighbors(int n, const double *W, int i, int *out);   /* ascending */
int ora_out_neighbors(int n, const double *W, int i, int *out);  /* ascending */
/* bit0: every row sums to 1 (pull), bit1: every column sums to 1 (push) */
int ora_classify(int n, const double *W, double tol);

/* ---- local views -> W  (Eq. 9-11) ---------------------------- */
typedef struct {
    double self_weight;                 /* w_ii */
    int n_src; const int *src; const double *r;   /* r_ij, pull side; n_src = -1: not given */
    int n_dst; const int *dst; const double *s;   /* s_ji, push side; n_dst = -1: not given */
} ora_view;
/* Returns 0, or -(1+i) for the first receiver i whose declaration does not
 * match its senders' (topology check) when check != 0. */
int ora_assemble(int n, const ora_view *views, int check, double *W);

/* ---- partial averaging (Eq. 5) ----------------------------------- */
void ora_mix(int n, long long count, const double *W, const double *X, double *Y);

/* ---- ATC-DSGD step (Eq. 4-5, Eq. 17) ---------------------
 * X, G hold exact fp32 (or bf16) input values.  Cast points (R18):
 *   xh   = fp32(x - lr*g)            (local update, Eq. 4)
 *   wire = xh rounded to the wire dtype (0 fp32, 1 bf16 RNE)
 *   y_i  = w_ii*xh_i + sum_j w_ij*wire(xh_j)   in fp64 (Eq. 5)          */
void ora_atc(int n, long long count, const double *W, const double *X,
             const double *G, double lr, int wire_bf16, double *Y);
/* AWC (Eq. 16): y_i = sum_j w_ij x_j - lr*g_i  */
void ora_exact_diffusion(int n, long long count, const double *W, const double *X, const double *G,
                         const double *Psi_prev, double lr, int wire_bf16, double *Y, double *Psi_out);
void ora_awc(int n, long long count, const double *W, const double *X,
             const double *G, double lr, double *Y);

/* ---- hierarchical neighbour allreduce ---------------- */
void ora_hier(int n_machines, int local_size, long long count, const double *WM,
              const double *X, double *Y);

/* H-ATC / H-AWC (caption P:869): Eq. 17 / Eq. 16 with the hierarchical combine */
void ora_hier_atc(int n_machines, int local_size, long long count, const double *WM,
                  const double *X, const double *G, double lr, double *Y);
void ora_hier_awc(int n_machines, int local_size, long long count, const double *WM,
                  const double *X, const double *G, double lr, double *Y);

/* ---- push-sum gradient tracking (appendix) -------
 * (a) u+ = W(u - lr y), v+ = W v, x+ = u+ / v+ ; (b) y+ = W(y + g+ - g).
 * V has dv = d columns (the paper's vector v) or dv = 1 (one weight per agent). */
void ora_gt_uv(int n, long long d, long long dv, const double *W, const double *U, const double *V,
               const double *Y, double lr, double *Un, double *Vn, double *Xn);
void ora_gt_y(int n, long long d, const double *W, const double *Y, const double *Gnew,
              const double *Gprev, double *Yn);

/* ---- casts ---------------------------------------------------------------- */
uint16_t ora_bf16_rne(float f);
float ora_f32(double v);

/* ---- window protocol event model ------------------
 * State of n agents with ext vectors of length count (x plus p as last
 * element, Listing 3).  Slots follow P:388: one per static in-neighbour,
 * ascending rank; each slot is double-buffered (halves), R11. */
typedef struct ora_win ora_win;
ora_win *ora_win_create(int n, long long count, const double *Wstatic,
                        const double *X0, int zero_init);
void ora_win_free(ora_win *w);
/* accumulate (put if overwrite != 0) by agent i: self_weight, dst weights s[n]
 * (s[j] used for j in dst set; dst_mask[j] != 0 selects) */
int ora_win_accumulate(ora_win *w, int i, double self_weight, const double *s,
                       const int *dst_mask, int overwrite);
/* local step x_i <- x_i - lr g_i before a push (gradient-in-window, SGP-style) */
void ora_win_adapt(ora_win *w, int i, const double *g, double lr);
/* update_then_collect by agent i (sum of ready halves, release) */
void ora_win_collect(ora_win *w, int i);
/* win_update by agent i: out = self_w*x_i + sum_j r_j*latest slot j (no reset) */
void ora_win_update(ora_win *w, int i, double self_weight, const double *r, double *out);
void ora_win_get_x(const ora_win *w, double *X);            /* n*count */
double ora_win_mass(const ora_win *w, long long e);         /* total mass of element e */
void ora_win_counters(const ora_win *w, int dst, int src, long long *version, long long *consumed);

/* ---- paper-semantics window ------------------
 * One plain buffer per in-neighbour: put overwrites, accumulate adds, collect
 * sums into x then zeroes, update reads without reset.  No protocol state. */
typedef struct ora_winp ora_winp;
ora_winp *ora_winp_create(int n, long long count, const double *Wstatic, const double *X0, int zero_init);
void ora_winp_free(ora_winp *w);
int ora_winp_accumulate(ora_winp *w, int i, double self_weight, const double *s, const int *dst_mask,
                        int overwrite);
void ora_winp_collect(ora_winp *w, int i);
void ora_winp_update(const ora_winp *w, int i, double self_weight, const double *r, double *out);
void ora_winp_get_x(const ora_winp *w, double *X);

/* ---- least squares (Eq. 12-13) ------------------------------- */
void ora_lsq_grad(int m, int d, const double *A, const double *b, const double *x, double *g);
/* CG on sum_i A_i^T A_i x = sum_i A_i^T b_i; returns iterations */
int ora_lsq_solve(int n, int m, int d, const double *A, const double *b, double tol,
                  int max_iter, double *x);
/* ATC-DSGD fixed point x_inf: iterate
 * X <- W(X - lr (A_i^T(A_i x_i - b_i))_i) in fp64 to stationarity; returns
 * iterations or -1.  X: start in, x_inf out (n x d). */
int ora_atc_fixed_point(int n, int m, int d, const double *W, const double *A, const double *b, double lr,
                        double tol, int max_iter, double *X);

/* ---- communication cost model, Table 1 ----------
 * 0 parameter server nM/B + nL, 1 ring-allreduce 2M/B + 2nL, 2 Byte-PS M/B + nL,
 * 3 partial averaging M/B + L (seconds; M bytes, B bytes/s, L seconds). */
double ora_comm_cost(int primitive, int n, double M, double B, double L);

#ifdef __cplusplus
}
#endif
#endif
