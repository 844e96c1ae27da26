"""GPU parity at the production shapes, and the round-2 boundary additions.

* The fused kernel at more than one sub-item per CTA (K = 1, 2: the U = 2 group
  path with nu = 2; K = 4), over consecutive one-peer rounds and every fused op,
  checked on sampled columns (every op is column-wise, so the oracle computes the
  sampled columns exactly; the GPU state is fed back each round).
* bf16 rows that are only 8-byte aligned (count = 4 mod 8).
* bf_set_topology_local: local views -> global W.
* Calls on different streams are serialised by the library.
* C2: ATC-DSGD on least squares reaches the oracle's fixed point x_inf.
* Windows whose rows span more items than the grid has CTAs.
Tolerance rule as in test_gpu_parity.py.
"""
import os

import numpy as np
import pytest
import torch

import oracle as ora
import synthetic

pytestmark = pytest.mark.gpu

os.environ.setdefault("BF_TIMEOUT_MS", "5000")

if torch.cuda.is_available():
    import paper_2111_04287_b200 as bfp
    from paper_2111_04287_b200 import BluefogError


def _ctx(k, heap=1 << 28):
    return bfp.Context(agents_per_proc=k, heap_bytes=heap, device=0)


def _np(t):
    return t.float().cpu().numpy().astype(np.float64)


def _gpu(X, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).to(dtype).cuda()


def assert_parity(y, ref, W, X, tol, extra=None, what=""):
    b = np.abs(W) @ np.abs(X)
    if extra is not None:
        b = b + extra
    err = np.abs(y - ref)
    bad = err > tol * b + 1e-30
    assert not bad.any(), f"{what}: max rel err {np.max(err / (b + 1e-30)):.3e} at {np.argwhere(bad)[:5].tolist()}"


def _sample_cols(count, seed=0, n_random=3000):
    # random columns plus the edges of fp32 / bf16 sub-items (1024 / 2048 elements),
    # of the first and last CTA's ownership and the ragged tail
    rng = np.random.default_rng(seed)
    edges = [0, 1, 1023, 1024, 2047, 2048, 4095, 4096, 296 * 1024 - 1, 296 * 1024, 296 * 2048,
             count - 1025, count - 1024, count - 8, count - 5, count - 4, count - 1]
    cols = np.concatenate([rng.integers(0, count, n_random), [e for e in edges if 0 <= e < count]])
    return np.unique(cols)


# ------------------------------------------- production shape on one GPU ---
@pytest.mark.parametrize("k", [1, 2, 4])
def test_fused_ops_production_shape_one_peer_rounds(k):
    """More than one sub-item per CTA (count = 2^22 + 5 per agent: ~14 fp32
    sub-items per CTA), every fused op over consecutive one-peer exp-2 rounds
    (R5), GPU state fed to the oracle each round (Eq. 4-5, 16, 17; ED)."""
    count, lr = (1 << 22) + 5, 0.1
    ctx = _ctx(k, heap=1 << 30)
    ctx.set_dynamic_schedule("one_peer_exp2", 0)
    n = ctx.n
    x = torch.empty(k, count, device="cuda")
    for r in range(k):
        bfp.Context.fill_uniform(x[r], synthetic.SEED_X0 + r)
    cols = _sample_cols(count)
    ct = torch.from_numpy(cols).cuda()
    sample = lambda t: _np(t[:, ct])

    def grad(step):
        g = torch.empty(k, count, device="cuda")
        for r in range(k):
            bfp.Context.fill_uniform(g[r], synthetic.grad_seed(step, r), scale=2.0 ** -7)
        return g

    rnd = 0
    # ATC, fp32 and bf16 wire (+ shadow)
    for wire, tol in ((torch.float32, 1e-6), (torch.bfloat16, 1e-2)):
        g = grad(rnd)
        X, G = sample(x), sample(g)
        shadow = torch.empty(k, count, dtype=torch.bfloat16, device="cuda") if wire == torch.bfloat16 else None
        ctx.atc_step(x, g, lr, wire=wire, shadow=shadow)
        torch.cuda.synchronize()
        Wk = ora.one_peer_exp2(n, rnd)
        got = sample(x)
        assert_parity(got, ora.atc(Wk, X, G, lr, wire_bf16=wire == torch.bfloat16), Wk, X, tol,
                      np.abs(Wk) @ (np.float32(lr) * np.abs(G)), f"atc {wire} k={k}")
        if shadow is not None:
            bits = shadow[:, ct].view(torch.int16).cpu().numpy().astype(np.uint16)
            assert np.array_equal(bits, ora.bf16_rne(got.astype(np.float32)).reshape(bits.shape))
        rnd += 1
    # AWC
    g = grad(rnd)
    X, G = sample(x), sample(g)
    ctx.awc_step(x, g, lr)
    torch.cuda.synchronize()
    Wk = ora.one_peer_exp2(n, rnd)
    assert_parity(sample(x), ora.awc(Wk, X, G, lr), Wk, X, 1e-6, np.float32(lr) * np.abs(G), f"awc k={k}")
    rnd += 1
    # neighbor_allreduce fp32 into a separate output
    X = sample(x)
    y = ctx.neighbor_allreduce(x)
    torch.cuda.synchronize()
    Wk = ora.one_peer_exp2(n, rnd)
    assert_parity(sample(y), ora.mix(Wk, X), Wk, X, 1e-6, None, f"nar k={k}")
    rnd += 1
    # Exact-Diffusion, two steps (psi_prev != x on the second)
    psi = x.clone()
    for _ in range(2):
        g = grad(rnd)
        X, G, P = sample(x), sample(g), sample(psi)
        ctx.exact_diffusion_step(x, g, psi, lr)
        torch.cuda.synchronize()
        Wk = ora.one_peer_exp2(n, rnd)
        ref, pref = ora.exact_diffusion(Wk, X, G, P, lr)
        phi_abs = np.abs(X) * 2 + np.float32(lr) * np.abs(G) + np.abs(P)
        assert_parity(sample(x), ref, Wk, phi_abs, 1e-6, None, f"ed k={k}")
        assert np.abs(sample(psi) - pref).max() <= 1e-6 * (np.abs(X) + lr * np.abs(G)).max()
        rnd += 1
    # bf16 neighbor_allreduce (8 elements per 16-byte vector)
    xb = x.to(torch.bfloat16)
    X = sample(xb)
    yb = ctx.neighbor_allreduce(xb)
    torch.cuda.synchronize()
    Wk = ora.one_peer_exp2(n, rnd)
    assert_parity(sample(yb), ora.mix(Wk, X), Wk, X, 1e-2, None, f"nar bf16 k={k}")
    ctx.close()


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_fused_static_exp2_production_shape(k):
    # static exponential-2 graph (R4) at > 1 sub-item per CTA, three chained ATC steps
    count, lr = (1 << 22) + 3, 0.05
    ctx = _ctx(k, heap=1 << 30)
    n = ctx.n
    W = ora.exp2(n)
    ctx.set_topology(W)
    x = torch.empty(k, count, device="cuda")
    for r in range(k):
        bfp.Context.fill_uniform(x[r], synthetic.SEED_X0 + 10 + r)
    cols = _sample_cols(count, seed=1)
    ct = torch.from_numpy(cols).cuda()
    for step in range(3):
        g = torch.empty(k, count, device="cuda")
        for r in range(k):
            bfp.Context.fill_uniform(g[r], synthetic.grad_seed(step, r), scale=2.0 ** -7)
        X, G = _np(x[:, ct]), _np(g[:, ct])
        ctx.atc_step(x, g, lr)
        torch.cuda.synchronize()
        assert_parity(_np(x[:, ct]), ora.atc(W, X, G, lr), W, X, 1e-6, np.abs(W) @ (np.float32(lr) * np.abs(G)),
                      f"exp2 step {step}")
    ctx.close()


# ------------------------------------------- bf16 rows aligned to 8 bytes only ---
@pytest.mark.parametrize("k", [2, 4, 8])
@pytest.mark.parametrize("count", [4, 100, 4100, 12292])
def test_bf16_rows_not_16_byte_aligned(k, count):
    """count = 4 mod 8: bf16 row a starts at a*count*2 bytes, 8-byte aligned for odd
    a.  The kernels must not issue 16-byte accesses there."""
    ctx = _ctx(k)
    W = ora.exp2(k) if k > 1 else np.eye(1)
    ctx.set_topology(W)
    X = synthetic.agents_x0(k, count)
    x = _gpu(X, torch.bfloat16)
    Xb = _np(x)
    y = ctx.neighbor_allreduce(x)
    torch.cuda.synchronize()
    assert_parity(_np(y), ora.mix(W, Xb), W, Xb, 1e-2, None, "nar bf16")
    if k % 2 == 0:   # the hierarchical Kronecker mix in the fused kernel, bf16
        WM = ora.exp2(k // 2) if k > 2 else np.ones((1, 1))
        ctx.set_machine_topology(WM, 2)
        y = ctx.hierarchical_neighbor_allreduce(x)
        torch.cuda.synchronize()
        assert_parity(_np(y), ora.hier(WM, 2, Xb), np.kron(WM, np.full((2, 2), 0.5)), Xb, 1e-2, None, "hier bf16")
    ctx.close()


# ------------------------------------------------- bf_set_topology_local ---
@pytest.mark.parametrize("style", ["pull", "push", "pushpull"])
def test_set_topology_local_equals_global(style):
    """SURVEY 8(b) bf_set_topology_local: static local views of every
    agent assemble the same W as the oracle's ora_assemble (Eq. 9, R1), and the
    static exchange over it matches the oracle."""
    n = 8
    rng = np.random.default_rng(5)
    A = (rng.random((n, n)) < 0.4) & ~np.eye(n, dtype=bool)
    Wt = A * rng.uniform(0.1, 0.9, (n, n))
    np.fill_diagonal(Wt, 0.5)
    views, sw, srcw, dstw = [], [], [], []
    for i in range(n):
        srcs = [j for j in range(n) if j != i and Wt[i, j] != 0]
        dsts = [j for j in range(n) if j != i and Wt[j, i] != 0]
        src = {j: Wt[i, j] for j in srcs} if style == "pull" else ({j: 0.5 for j in srcs} if style == "pushpull" else None)
        dst = {j: Wt[j, i] for j in dsts} if style == "push" else ({j: 2.0 * Wt[j, i] for j in dsts} if style == "pushpull" else None)
        views.append({"self_weight": 0.5, "src_weights": src, "dst_weights": dst})
        sw.append(0.5), srcw.append(src), dstw.append(dst)
    W = ora.assemble(views, check=True)
    assert np.allclose(W, Wt)
    ctx = _ctx(n)
    ctx.set_topology_local(sw, srcw, dstw)
    for i in range(n):
        assert ctx.in_neighbor_ranks(i) == ora.in_neighbors(W, i)
        assert ctx.out_neighbor_ranks(i) == ora.out_neighbors(W, i)
    X = synthetic.agents_x0(n, 5003)
    x = _gpu(X)
    y = ctx.neighbor_allreduce(x)
    torch.cuda.synchronize()
    assert_parity(_np(y), ora.mix(W, X.astype(np.float64)), W, X.astype(np.float64), 1e-6)
    ctx.close()


def test_set_topology_local_mismatch_is_topology_error():
    # agent 1 lists 0 as a source while 0 sends only to 2
    n = 4
    ctx = _ctx(n)
    sw = [0.5] * n
    srcw = [None, {0: 0.5}, None, None]
    dstw = [{2: 0.5}, None, {0: 0.5}, {0: 0.5}]
    with pytest.raises(BluefogError) as e:
        ctx.set_topology_local(sw, srcw, dstw)
    assert e.value.name == "BF_ERR_TOPOLOGY"
    ctx.close()


# -------------------------------------------- calls on different streams ---
def test_calls_on_other_streams_are_serialised():
    """A non-blocking call on the side stream followed at once (no wait) by calls
    on the current stream: the library orders them."""
    n, count, lr = 4, 3_000_001, 0.1
    W = ora.ring(n)
    ctx = _ctx(n, heap=1 << 30)
    ctx.set_topology(W)
    X = synthetic.agents_x0(n, count)
    G = synthetic.agents_grad(n, count, 3)
    x, g = _gpu(X), _gpu(G)
    x2 = x.clone()
    X64, G64 = X.astype(np.float64), G.astype(np.float64)
    for _ in range(3):
        h = ctx.neighbor_allreduce_nonblocking(x)
        ctx.atc_step(x2, g, lr)                     # current stream, no wait in between
        y = ctx.neighbor_allreduce(x2)
        y1 = bfp.Context.wait(h)
        torch.cuda.synchronize()
        assert_parity(_np(y1), ora.mix(W, X64), W, X64, 1e-6, None, "nonblocking")
        X2 = ora.atc(W, X64, G64, lr)
        assert_parity(_np(x2), X2, W, X64, 1e-6, np.abs(W) @ (np.float32(lr) * np.abs(G64)), "atc")
        assert_parity(_np(y), ora.mix(W, _np(x2)), W, _np(x2), 1e-6, None, "nar after atc")
        x2 = _gpu(X)
    ctx.close()


# ------------------------------------- C2: ATC-DSGD reaches the fixed point ---
def test_c2_atc_dsgd_reaches_oracle_fixed_point():
    """C2-shaped decentralized least squares (Eq. 12-13; 8 agents,
    static exp-2, full local gradients) run with the fused ATC step (Eq. 17) until
    stationary, against the oracle's x_inf.  The fixed point is
    unique (linear contraction with rate rho), so the fp32 GPU run lands within
    its rounding noise of x_inf: per step ~eps32 * |x| injected, amplified by at
    most 1 / (1 - rho)."""
    n, m, d = 8, 120, 40
    rng = np.random.default_rng(21)
    A = rng.standard_normal((n, m, d)) / np.sqrt(m)
    xnat = rng.standard_normal(d)
    b = np.einsum("imd,d->im", A, xnat) + 0.01 * rng.standard_normal((n, m))
    W = ora.exp2(n)
    lam = max(np.linalg.eigvalsh(A[i].T @ A[i]).max() for i in range(n))
    lr = float(np.float32(1.0 / lam))
    xinf, it = ora.atc_fixed_point(W, A, b, lr)
    # contraction rate of X -> W(X - lr(HX - c)) (library eigenvalues, for the tolerance only)
    H = np.zeros((n * d, n * d))
    for i in range(n):
        H[i * d:(i + 1) * d, i * d:(i + 1) * d] = A[i].T @ A[i]
    rho = np.abs(np.linalg.eigvals(np.kron(W, np.eye(d)) @ (np.eye(n * d) - lr * H))).max()
    assert rho < 1
    ctx = _ctx(n)
    ctx.set_topology(W)
    At, bt = torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda()
    x = torch.zeros(n, d, device="cuda")
    for _ in range(int(40 / (1 - rho)) + 200):
        x64 = x.double()
        g = torch.bmm(At.transpose(1, 2), (torch.bmm(At, x64.unsqueeze(2)).squeeze(2) - bt).unsqueeze(2))
        ctx.atc_step(x, g.squeeze(2).float().contiguous(), lr)
    torch.cuda.synchronize()
    err = np.abs(_np(x) - xinf).max() / np.abs(xinf).max()
    tol = 64 * 2.0 ** -24 / (1 - rho)
    assert err < tol, (err, tol, rho)
    # and x_inf is not x* (ATC's O(gamma) bias, the reason for Exact-Diffusion)
    xs = np.linalg.lstsq(A.reshape(n * m, d), b.reshape(n * m), rcond=None)[0]
    assert np.abs(xinf - xs).max() > 10 * tol * np.abs(xinf).max()
    ctx.close()


# ------------------------------------------ windows: more items than CTAs ---
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_window_sync_pushsum_items_exceed_grid(dtype):
    """Synchronous push-sum (Listing 3 weights) on 8 agents x (2^22 + 8)
    elements: every window kernel walks its grid-stride loop many times.  One
    round (all accumulate, then all collect) is one product with the
    column-stochastic W of Listing 3 (oracle pin test_window_sync_pushsum_equals_mix);
    each round is checked against ora.mix on the GPU's previous state."""
    n, count = 8, (1 << 22) + 8
    Wst = ora.exp2(n)
    Wps = np.zeros((n, n))
    for i in range(n):
        outs = ora.out_neighbors(Wst, i)
        w = 1.0 / (len(outs) + 1)
        Wps[i, i] = w
        for j in outs:
            Wps[j, i] = w
    ctx = _ctx(n, heap=3 << 30)
    ctx.set_topology(Wst)
    x = torch.empty(n, count, device="cuda", dtype=dtype)
    xf = torch.empty(n, count, device="cuda")
    for r in range(n):
        bfp.Context.fill_uniform(xf[r], synthetic.SEED_X0 + r)
    x.copy_(xf)
    ctx.win_create(x, "big", zero_init=True, with_p=True)
    cols = _sample_cols(count, seed=3)
    ct = torch.from_numpy(cols).cuda()
    p = np.ones(n)
    tol = 1e-6 if dtype == torch.float32 else 1e-2
    for rnd in range(3):
        X = _np(x[:, ct])
        ctx.win_accumulate("big")
        ctx.win_update_then_collect("big")
        torch.cuda.synchronize()
        assert_parity(_np(x[:, ct]), ora.mix(Wps, X), Wps, X, tol, None, f"round {rnd}")
        p = Wps @ p
        assert np.allclose(ctx.win_p("big"), p, rtol=0, atol=1e-12)
    ctx.win_free("big")
    ctx.close()


# ------------------------------- gradient-in-window push (SGP-style) ---
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_win_accumulate_grad_matches_event_model(dtype):
    """bf_win_accumulate_grad: x <- x - lr g (Eq. 4) fused into the push of
    win_accumulate, against ora.Window.adapt + accumulate, with random
    per-agent interleaving of pushes and collects."""
    n, count, lr = 8, 20011, 0.1
    Wst = ora.exp2(n)
    ctx = _ctx(n)
    ctx.set_topology(Wst)
    x = _gpu(synthetic.agents_x0(n, count), dtype)
    X0 = _np(x)
    ctx.win_create(x, "sgp", zero_init=True, with_p=True)
    win = ora.Window(Wst, np.concatenate([X0, np.ones((n, 1))], axis=1), zero_init=True)
    rng = np.random.default_rng(17)
    for step in range(40):
        i = int(rng.integers(n))
        if rng.random() < 0.6:
            g = _gpu(synthetic.agents_grad(n, count, step), dtype)
            G = _np(g)
            ctx.win_accumulate_grad("sgp", g, lr, agent_mask=1 << i)
            win.adapt(i, np.concatenate([G[i], [0.0]]), lr)
            outs = ora.out_neighbors(Wst, i)
            w = 1.0 / (len(outs) + 1)
            win.accumulate(i, w, {j: w for j in outs})
        else:
            ctx.win_update_then_collect("sgp", agent_mask=1 << i)
            win.collect(i)
    torch.cuda.synchronize()
    ref = win.x()
    tol = 3e-5 if dtype == torch.float32 else 2e-2
    assert np.abs(_np(x) - ref[:, :-1]).max() < tol
    assert np.allclose(ctx.win_p("sgp"), ref[:, -1], rtol=0, atol=1e-12)
    ctx.win_free("sgp")
    ctx.close()


# --------------------------- GPU windows against the paper's window semantics ---
def test_window_gpu_equals_paper_semantics_without_backlog():
    """The GPU window against the paper-semantics window (ora.WindowPaper: one buffer
    per in-neighbour, accumulate adds, collect sums then zeroes)
    under random per-agent interleavings in which no payload has to wait in an
    outbox (every destination half free at each accumulate, read from the GPU's own
    counters) -- where the two models must agree (oracle pin
    test_event_model_equals_paper_window_without_backlog).  Bound: every event rounds
    each touched fp32 value at most twice, |x| <= 1: 120 events -> 120*2*2^-24 ~ 1.5e-5."""
    n, count = 8, 5003
    Wst = ora.exp2(n)
    ctx = _ctx(n)
    ctx.set_topology(Wst)
    X0 = synthetic.agents_x0(n, count).astype(np.float64)
    x = _gpu(X0)
    ctx.win_create(x, "pw", zero_init=True, with_p=True)
    pw = ora.WindowPaper(Wst, np.concatenate([X0, np.ones((n, 1))], axis=1), zero_init=True)
    rng = np.random.default_rng(23)
    n_acc = 0
    for _ in range(120):
        i = int(rng.integers(n))
        outs = ora.out_neighbors(Wst, i)
        torch.cuda.synchronize()
        free = True
        for j in outs:   # the half the next payload i -> j lands in is free (no backlog)
            v, c = ctx.win_counters("pw", j % n, i)
            free = free and c >= v - 1
        if rng.random() < 0.5 and free:
            w = 1.0 / (len(outs) + 1)
            ctx.win_accumulate("pw", agent_mask=1 << i)
            pw.accumulate(i, w, {j: w for j in outs})
            n_acc += 1
        else:
            ctx.win_update_then_collect("pw", agent_mask=1 << i)
            pw.collect(i)
    torch.cuda.synchronize()
    ref = pw.x()
    assert n_acc > 20
    assert np.abs(_np(x) - ref[:, :-1]).max() < 3e-5
    assert np.allclose(ctx.win_p("pw"), ref[:, -1], rtol=0, atol=1e-12)
    ctx.win_free("pw")
    ctx.close()


def test_win_version_matches_counters():
    # SURVEY 8(b) bf_win_version: payloads delivered from src_rank to the first local agent
    # that has it as an in-neighbour (= bf_win_counters' version for that pair)
    n = 4
    W = ora.ring(n)
    ctx = _ctx(n)
    ctx.set_topology(W)
    x = _gpu(synthetic.agents_x0(n, 1001))
    ctx.win_create(x, "v", zero_init=True)
    for _ in range(2):
        ctx.win_put("v")
        ctx.win_update_then_collect("v")
    torch.cuda.synchronize()
    for src in range(n):
        first = min(i for i in range(n) if src in ora.in_neighbors(W, i))
        assert ctx.win_version("v", src) == ctx.win_counters("v", first, src)[0] == 2
    with pytest.raises(BluefogError):
        ctx.win_version("v", 99)   # no local agent receives from it
    ctx.win_free("v")
    ctx.close()
