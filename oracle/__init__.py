"""Python marshalling for the C oracle (oracle/bf_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py may import this module.
The product (paper_2111_04287_b200) never imports it, and this module never
imports the product.  All arithmetic lives in bf_oracle.c (fp64, plain loops);
this file only converts numpy arrays to pointers.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bf_oracle.c")
_HDR = os.path.join(_HERE, "bf_oracle.h")
_SO = os.path.join(_HERE, "libbf_oracle.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, no FMA contraction, no fast-math)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-Wall", "-shared", "-fPIC", _SRC, "-o", _SO + ".tmp", "-lm"])
        os.replace(_SO + ".tmp", _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.ora_ring.argtypes = [C.c_int, _dp]
        L.ora_exp2.argtypes = [C.c_int, _dp]
        L.ora_full.argtypes = [C.c_int, _dp]
        L.ora_one_peer_exp2.argtypes = [C.c_int, C.c_longlong, _dp]
        L.ora_one_peer_exp2_peers.argtypes = [C.c_int, C.c_longlong, C.c_int, _ip, _ip]
        L.ora_inner_outer_exp2.argtypes = [C.c_int, C.c_int, C.c_longlong, _dp]
        L.ora_inner_outer_exp2_peers.argtypes = [C.c_int, C.c_int, C.c_longlong, C.c_int, _ip, _ip]
        L.ora_in_neighbors.argtypes = [C.c_int, _dp, C.c_int, _ip]
        L.ora_out_neighbors.argtypes = [C.c_int, _dp, C.c_int, _ip]
        L.ora_classify.argtypes = [C.c_int, _dp, C.c_double]
        L.ora_assemble.argtypes = [C.c_int, C.c_void_p, C.c_int, _dp]
        L.ora_mix.argtypes = [C.c_int, C.c_longlong, _dp, _dp, _dp]
        L.ora_atc.argtypes = [C.c_int, C.c_longlong, _dp, _dp, _dp, C.c_double, C.c_int, _dp]
        L.ora_awc.argtypes = [C.c_int, C.c_longlong, _dp, _dp, _dp, C.c_double, _dp]
        L.ora_exact_diffusion.argtypes = [C.c_int, C.c_longlong, _dp, _dp, _dp, _dp, C.c_double, C.c_int, _dp, _dp]
        L.ora_hier.argtypes = [C.c_int, C.c_int, C.c_longlong, _dp, _dp, _dp]
        L.ora_bf16_rne.argtypes = [C.c_float]
        L.ora_bf16_rne.restype = C.c_uint16
        L.ora_win_create.argtypes = [C.c_int, C.c_longlong, _dp, _dp, C.c_int]
        L.ora_win_create.restype = C.c_void_p
        L.ora_win_free.argtypes = [C.c_void_p]
        L.ora_win_accumulate.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp, _ip, C.c_int]
        L.ora_win_collect.argtypes = [C.c_void_p, C.c_int]
        L.ora_win_adapt.argtypes = [C.c_void_p, C.c_int, _dp, C.c_double]
        L.ora_win_update.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp, _dp]
        L.ora_win_get_x.argtypes = [C.c_void_p, _dp]
        L.ora_win_mass.argtypes = [C.c_void_p, C.c_longlong]
        L.ora_win_mass.restype = C.c_double
        L.ora_win_counters.argtypes = [C.c_void_p, C.c_int, C.c_int,
                                       C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]
        L.ora_lsq_grad.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, _dp]
        L.ora_lsq_solve.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_double, C.c_int, _dp]
        L.ora_hier_atc.argtypes = [C.c_int, C.c_int, C.c_longlong, _dp, _dp, _dp, C.c_double, _dp]
        L.ora_hier_awc.argtypes = [C.c_int, C.c_int, C.c_longlong, _dp, _dp, _dp, C.c_double, _dp]
        L.ora_gt_uv.argtypes = [C.c_int, C.c_longlong, C.c_longlong, _dp, _dp, _dp, _dp, C.c_double, _dp, _dp, _dp]
        L.ora_gt_y.argtypes = [C.c_int, C.c_longlong, _dp, _dp, _dp, _dp, _dp]
        L.ora_winp_create.argtypes = [C.c_int, C.c_longlong, _dp, _dp, C.c_int]
        L.ora_winp_create.restype = C.c_void_p
        L.ora_winp_free.argtypes = [C.c_void_p]
        L.ora_winp_accumulate.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp, _ip, C.c_int]
        L.ora_winp_collect.argtypes = [C.c_void_p, C.c_int]
        L.ora_winp_update.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp, _dp]
        L.ora_winp_get_x.argtypes = [C.c_void_p, _dp]
        L.ora_atc_fixed_point.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, C.c_double, C.c_double,
                                          C.c_int, _dp]
        L.ora_comm_cost.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double]
        L.ora_comm_cost.restype = C.c_double
    return _lib


def _d(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# ---- topologies -------------------------------------------------------------
def _topo(fn, n, *extra):
    W = np.zeros((n, n), np.float64)
    fn(n, *extra, _d(W))
    return W


def ring(n):
    return _topo(lib().ora_ring, n)


def exp2(n):
    return _topo(lib().ora_exp2, n)


def full(n):
    return _topo(lib().ora_full, n)


def one_peer_exp2(n, k):
    return _topo(lib().ora_one_peer_exp2, n, int(k))


def one_peer_exp2_peers(n, k, i):
    s, d = C.c_int(), C.c_int()
    lib().ora_one_peer_exp2_peers(n, int(k), i, C.byref(s), C.byref(d))
    return s.value, d.value


def inner_outer_exp2(n, local_size, k):
    """Inner-outer dynamic exp-2 graph at round k (reading R27)."""
    if local_size < 1 or n % local_size:
        raise ValueError("machines must tile the agents")
    return _topo(lib().ora_inner_outer_exp2, n, int(local_size), int(k))


def inner_outer_exp2_peers(n, local_size, k, i):
    s, d = C.c_int(), C.c_int()
    lib().ora_inner_outer_exp2_peers(n, int(local_size), int(k), i, C.byref(s), C.byref(d))
    return s.value, d.value


def in_neighbors(W, i):
    W = _f64(W)
    n = W.shape[0]
    out = np.zeros(n, np.int32)
    c = lib().ora_in_neighbors(n, _d(W), i, out.ctypes.data_as(_ip))
    return [int(v) for v in out[:c]]


def out_neighbors(W, i):
    W = _f64(W)
    n = W.shape[0]
    out = np.zeros(n, np.int32)
    c = lib().ora_out_neighbors(n, _d(W), i, out.ctypes.data_as(_ip))
    return [int(v) for v in out[:c]]


def classify(W, tol=1e-12):
    """Returns 'none' | 'pull' | 'push' | 'standard'."""
    W = _f64(W)
    c = lib().ora_classify(W.shape[0], _d(W), tol)
    return {0: "none", 1: "pull", 2: "push", 3: "standard"}[c]


# ---- local views -> W --------------------------------------------------------
class _View(C.Structure):
    _fields_ = [("self_weight", C.c_double),
                ("n_src", C.c_int), ("src", _ip), ("r", _dp),
                ("n_dst", C.c_int), ("dst", _ip), ("s", _dp)]


def assemble(views, check=True):
    """views: list of dicts {self_weight, src_weights: {j: r} | None, dst_weights: {j: s} | None}.

    Returns W, or raises ValueError(receiver) on a topology-check mismatch.
    """
    n = len(views)
    keep = []
    arr = (_View * n)()
    for i, v in enumerate(views):
        sw = v.get("src_weights")
        dw = v.get("dst_weights")
        src = np.array(sorted(sw) if sw is not None else [], np.int32)
        r = np.array([sw[j] for j in sorted(sw)] if sw is not None else [], np.float64)
        dst = np.array(sorted(dw) if dw is not None else [], np.int32)
        s = np.array([dw[j] for j in sorted(dw)] if dw is not None else [], np.float64)
        keep += [src, r, dst, s]
        arr[i].self_weight = float(v["self_weight"])
        arr[i].n_src = len(src) if sw is not None else -1
        arr[i].src = src.ctypes.data_as(_ip)
        arr[i].r = r.ctypes.data_as(_dp)
        arr[i].n_dst = len(dst) if dw is not None else -1
        arr[i].dst = dst.ctypes.data_as(_ip)
        arr[i].s = s.ctypes.data_as(_dp)
    W = np.zeros((n, n), np.float64)
    rc = lib().ora_assemble(n, C.cast(arr, C.c_void_p), 1 if check else 0, _d(W))
    if rc != 0:
        raise ValueError(f"topology mismatch at receiver {-rc - 1}")
    return W


# ---- the hot-path arithmetic ------------------------------------------------
def mix(W, X):
    """Eq. 5 partial averaging of stacked X (n, count) -> fp64 (n, count)."""
    W, X = _f64(W), _f64(X)
    Y = np.zeros_like(X)
    lib().ora_mix(W.shape[0], X.shape[1], _d(W), _d(X), _d(Y))
    return Y


def atc(W, X, G, lr, wire_bf16=False):
    W, X, G = _f64(W), _f64(X), _f64(G)
    Y = np.zeros_like(X)
    lib().ora_atc(W.shape[0], X.shape[1], _d(W), _d(X), _d(G), float(np.float32(lr)),
                  1 if wire_bf16 else 0, _d(Y))
    return Y


def exact_diffusion(W, X, G, Psi_prev, lr, wire_bf16=False):
    """One Exact-Diffusion step (appendix Eqs. ed-1..ed-3): returns (x^(k+1), psi^(k))."""
    W, X, G, P = _f64(W), _f64(X), _f64(G), _f64(Psi_prev)
    Y = np.zeros_like(X)
    Pout = np.zeros_like(X)
    lib().ora_exact_diffusion(W.shape[0], X.shape[1], _d(W), _d(X), _d(G), _d(P), float(np.float32(lr)),
                              1 if wire_bf16 else 0, _d(Y), _d(Pout))
    return Y, Pout


def gt_uv(W, U, V, Y, lr):
    """First half of a push-sum gradient-tracking round (appendix, PAPER.md lines
    1002-1004): u+ = W(u - lr y), v+ = W v, x+ = u+ / v+.  V: (n, d) or (n, 1)."""
    W, U, V, Y = _f64(W), _f64(U), _f64(V), _f64(Y)
    n, d = U.shape
    Un, Vn, Xn = np.zeros_like(U), np.zeros_like(V), np.zeros_like(U)
    lib().ora_gt_uv(n, d, V.shape[1], _d(W), _d(U), _d(V), _d(Y), float(lr), _d(Un), _d(Vn), _d(Xn))
    return Un, Vn, Xn


def gt_y(W, Y, Gnew, Gprev):
    """Second half (line 1006): y+ = W(y + g+ - g)."""
    W, Y, Gn, Gp = _f64(W), _f64(Y), _f64(Gnew), _f64(Gprev)
    Yn = np.zeros_like(Y)
    lib().ora_gt_y(Y.shape[0], Y.shape[1], _d(W), _d(Y), _d(Gn), _d(Gp), _d(Yn))
    return Yn


def gradient_tracking_step(W, U, V, Y, Gprev, grad, lr):
    """One round of push-sum gradient tracking (appendix):
        u+ = W (u - lr y);  v+ = W v;  x+ = u+ / v+;  g+ = grad(x+);  y+ = W (y + g+ - g).
    U, Y, Gprev: (n, d); V: (n, 1) or (n, d).  Returns (x+, u+, v+, y+, g+).
    The arithmetic is ora_gt_uv / ora_gt_y; `grad` is the caller's gradient."""
    Un, Vn, Xn = gt_uv(W, U, V, Y, lr)
    Gn = _f64(grad(Xn))
    Yn = gt_y(W, Y, Gn, Gprev)
    return Xn, Un, Vn, Yn, Gn


def awc(W, X, G, lr):
    W, X, G = _f64(W), _f64(X), _f64(G)
    Y = np.zeros_like(X)
    lib().ora_awc(W.shape[0], X.shape[1], _d(W), _d(X), _d(G), float(np.float32(lr)), _d(Y))
    return Y


def hier(WM, local_size, X):
    WM, X = _f64(WM), _f64(X)
    Y = np.zeros_like(X)
    lib().ora_hier(WM.shape[0], local_size, X.shape[1], _d(WM), _d(X), _d(Y))
    return Y


def hier_atc(WM, local_size, X, G, lr):
    """H-ATC (caption P:869): (W_M kron J_L/L) fp32(X - lr G) (ora_hier_atc)."""
    WM, X, G = _f64(WM), _f64(X), _f64(G)
    Y = np.zeros_like(X)
    lib().ora_hier_atc(WM.shape[0], local_size, X.shape[1], _d(WM), _d(X), _d(G), float(np.float32(lr)), _d(Y))
    return Y


def hier_awc(WM, local_size, X, G, lr):
    """H-AWC (caption P:869): (W_M kron J_L/L) X - lr G (ora_hier_awc)."""
    WM, X, G = _f64(WM), _f64(X), _f64(G)
    Y = np.zeros_like(X)
    lib().ora_hier_awc(WM.shape[0], local_size, X.shape[1], _d(WM), _d(X), _d(G), float(np.float32(lr)), _d(Y))
    return Y


def bf16_rne(values) -> np.ndarray:
    v = np.asarray(values, np.float32).ravel()
    f = lib().ora_bf16_rne
    return np.array([f(float(x)) for x in v], np.uint16)


# ---- window event model -----------------------------------------------------
class Window:
    """Event model of the window protocol."""

    def __init__(self, W_static, X0, zero_init=True):
        W_static, X0 = _f64(W_static), _f64(X0)
        self.n, self.count = X0.shape
        self._W = W_static
        self._h = lib().ora_win_create(self.n, self.count, _d(W_static), _d(X0), 1 if zero_init else 0)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ora_win_free(self._h)
            self._h = None

    def accumulate(self, i, self_weight, dst_weights, overwrite=False):
        s = np.zeros(self.n, np.float64)
        mask = np.zeros(self.n, np.int32)
        for j, w in dst_weights.items():
            s[j] = w
            mask[j] = 1
        rc = lib().ora_win_accumulate(self._h, i, float(self_weight), _d(s), mask.ctypes.data_as(_ip),
                                      1 if overwrite else 0)
        if rc != 0:
            raise ValueError("destination outside the creation topology (P:398)")

    def put(self, i, self_weight, dst_weights):
        self.accumulate(i, self_weight, dst_weights, overwrite=True)

    def collect(self, i):
        lib().ora_win_collect(self._h, i)

    def adapt(self, i, g, lr):
        """x_i <- x_i - lr g_i (ora_win_adapt; g covers the whole window row)."""
        g = _f64(g)
        assert g.shape == (self.count,)
        lib().ora_win_adapt(self._h, i, _d(g), float(np.float32(lr)))

    def update(self, i, self_weight, src_weights):
        r = np.zeros(self.n, np.float64)
        for j, w in src_weights.items():
            r[j] = w
        out = np.zeros(self.count, np.float64)
        lib().ora_win_update(self._h, i, float(self_weight), _d(r), _d(out))
        return out

    def x(self):
        X = np.zeros((self.n, self.count), np.float64)
        lib().ora_win_get_x(self._h, _d(X))
        return X

    def mass(self, e):
        return lib().ora_win_mass(self._h, e)

    def counters(self, dst, src):
        v, c = C.c_longlong(), C.c_longlong()
        lib().ora_win_counters(self._h, dst, src, C.byref(v), C.byref(c))
        return v.value, c.value


class WindowPaper:
    """Paper-semantics window: one plain buffer per
    in-neighbour, put overwrites, accumulate adds, collect sums then zeroes,
    update reads without reset (ora_winp_*)."""

    def __init__(self, W_static, X0, zero_init=True):
        W_static, X0 = _f64(W_static), _f64(X0)
        self.n, self.count = X0.shape
        self._h = lib().ora_winp_create(self.n, self.count, _d(W_static), _d(X0), 1 if zero_init else 0)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ora_winp_free(self._h)
            self._h = None

    def accumulate(self, i, self_weight, dst_weights, overwrite=False):
        s = np.zeros(self.n, np.float64)
        mask = np.zeros(self.n, np.int32)
        for j, w in dst_weights.items():
            s[j] = w
            mask[j] = 1
        if lib().ora_winp_accumulate(self._h, i, float(self_weight), _d(s), mask.ctypes.data_as(_ip),
                                     1 if overwrite else 0):
            raise ValueError("destination outside the creation topology (P:398)")

    def put(self, i, self_weight, dst_weights):
        self.accumulate(i, self_weight, dst_weights, overwrite=True)

    def collect(self, i):
        lib().ora_winp_collect(self._h, i)

    def update(self, i, self_weight, src_weights):
        r = np.zeros(self.n, np.float64)
        for j, w in src_weights.items():
            r[j] = w
        out = np.zeros(self.count, np.float64)
        lib().ora_winp_update(self._h, i, float(self_weight), _d(r), _d(out))
        return out

    def x(self):
        X = np.zeros((self.n, self.count), np.float64)
        lib().ora_winp_get_x(self._h, _d(X))
        return X


# ---- least squares ------------------------------------------------------------
def lsq_grad(A, b, x):
    A, b, x = _f64(A), _f64(b), _f64(x)
    m, d = A.shape
    g = np.zeros(d, np.float64)
    lib().ora_lsq_grad(m, d, _d(A), _d(b), _d(x), _d(g))
    return g


def lsq_solve(A_stack, b_stack, tol=1e-13, max_iter=10000):
    A, b = _f64(A_stack), _f64(b_stack)
    n, m, d = A.shape
    x = np.zeros(d, np.float64)
    it = lib().ora_lsq_solve(n, m, d, _d(A), _d(b), tol, max_iter, _d(x))
    return x, it


def atc_fixed_point(W, A_stack, b_stack, lr, X0=None, tol=1e-15, max_iter=200000):
    """ATC-DSGD fixed point x_inf on least squares (Eq. 12-14,
    Eq. 17): iterate X <- W(X - lr g(X)) in fp64 to stationarity (ora_atc_fixed_point).
    Returns (X_inf, iterations); raises if it did not converge."""
    W, A, b = _f64(W), _f64(A_stack), _f64(b_stack)
    n, m, d = A.shape
    X = np.zeros((n, d), np.float64) if X0 is None else _f64(X0).copy()
    it = lib().ora_atc_fixed_point(n, m, d, _d(W), _d(A), _d(b), float(lr), float(tol), int(max_iter), _d(X))
    if it < 0:
        raise RuntimeError("ATC fixed-point iteration did not converge")
    return X, it


COMM_PRIMITIVES = {"parameter_server": 0, "ring_allreduce": 1, "byte_ps": 2, "partial_averaging": 3}


def comm_cost(primitive, n, M, B, L):
    """Table 1: seconds for one averaging (ora_comm_cost)."""
    return lib().ora_comm_cost(COMM_PRIMITIVES[primitive], int(n), float(M), float(B), float(L))
