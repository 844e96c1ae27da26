"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Single GPU: n agents run as `agents_per_proc = n` virtual agents of one
process; the exchange kernel is one cooperative launch over all of them, so
the cross-agent waits are between co-resident CTAs of one kernel.
Tolerance rule: |y - y_ref| <= tol * b elementwise,
b = sum_j |w_ij| |x_j| (ATC: |x_j| + lr |g_j|), tol = 1e-6 fp32, 1e-2 bf16.
"""
import os

import numpy as np
import pytest
import torch

import oracle as ora
import synthetic
from bfutil import golden

pytestmark = pytest.mark.gpu

os.environ.setdefault("BF_TIMEOUT_MS", "5000")

if torch.cuda.is_available():
    import paper_2111_04287_b200 as bfp
    from paper_2111_04287_b200 import BluefogError

TOL = {torch.float32: 1e-6, torch.bfloat16: 1e-2}
COUNTS = [1, 7, 4096, 4097, 3 * 4096 + 5, 100003]


def _ctx(k, heap=1 << 28):
    return bfp.Context(agents_per_proc=k, heap_bytes=heap, device=0)


def _gpu(X, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).to(dtype).cuda()


def _np(t):
    return t.float().cpu().numpy().astype(np.float64)


def _inputs(n, count, dtype=torch.float32):
    X = synthetic.agents_x0(n, count)
    t = _gpu(X, dtype)
    return t, _np(t)          # exact values the GPU holds (bf16-rounded if bf16)


def assert_parity(y, ref, W, X, tol, extra=None):
    b = np.abs(W) @ np.abs(X)
    if extra is not None:
        b = b + extra
    err = np.abs(y - ref)
    bad = err > tol * b + 1e-30
    assert not bad.any(), f"max rel err {np.max(err / (b + 1e-30)):.3e} at {np.argwhere(bad)[:5].tolist()}"


# ----------------------------------------------------------------- generator --
def test_fill_uniform_matches_synthetic():
    for dtype, scale in ((torch.float32, 1.0), (torch.float32, 2.0 ** -7), (torch.bfloat16, 1.0)):
        t = torch.empty(100003, dtype=dtype, device="cuda")
        bfp.Context.fill_uniform(t, seed=1234, offset=17, scale=scale)
        ref = torch.from_numpy(synthetic.uniform(1234, 100003, scale=scale, offset=17)).to(dtype)
        assert torch.equal(t.cpu(), ref)


# ------------------------------------------------------ neighbor_allreduce ---
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("topo,n", [("ring", 4), ("exp2", 8), ("full", 5), ("exp2", 3), ("ring", 2), ("exp2", 16)])
def test_nar_static(topo, n, dtype):
    ctx = _ctx(n)
    W = {"ring": ora.ring, "exp2": ora.exp2, "full": ora.full}[topo](n)
    ctx.set_topology(W)
    for count in COUNTS:
        x, X = _inputs(n, count, dtype)
        y = ctx.neighbor_allreduce(x)
        torch.cuda.synchronize()
        assert_parity(_np(y), ora.mix(W, X), W, X, TOL[dtype])
    ctx.close()


def test_nar_random_directed_and_inplace():
    n = 6
    rng = np.random.default_rng(1)
    W = (rng.random((n, n)) < 0.5) * rng.uniform(-1, 1, (n, n))
    np.fill_diagonal(W, rng.uniform(0.1, 1, n))
    ctx = _ctx(n)
    ctx.set_topology(W)
    x, X = _inputs(n, 50001)
    ctx.neighbor_allreduce(x, out=x)          # y aliases x
    torch.cuda.synchronize()
    assert_parity(_np(x), ora.mix(W, X), W, X, 1e-6)
    ctx.close()


def test_nar_default_topology_is_full_and_n1():
    ctx = _ctx(4)
    x = _gpu(np.array([[1.0], [2.0], [3.0], [4.0]]))
    y = ctx.neighbor_allreduce(x)
    torch.cuda.synchronize()
    assert np.allclose(_np(y), golden("spec_scalar_examples.json")["full4_expected"], atol=1e-7)
    ctx.close()
    ctx1 = _ctx(1)
    x, X = _inputs(1, 9999)
    y = ctx1.neighbor_allreduce(x)
    torch.cuda.synchronize()
    assert np.array_equal(_np(y), X)
    ctx1.close()


def _views(W, style):
    n = W.shape[0]
    sw, srcw, dstw = [], [], []
    for i in range(n):
        srcs = [j for j in range(n) if j != i and W[i, j] != 0]
        dsts = [j for j in range(n) if j != i and W[j, i] != 0]
        sw.append(W[i, i])
        if style == "pull":
            srcw.append({j: W[i, j] for j in srcs})
            dstw.append(None)
        elif style == "push":
            srcw.append(None)
            dstw.append({j: W[j, i] for j in dsts})
        else:
            srcw.append({j: 0.5 for j in srcs})
            dstw.append({j: 2.0 * W[j, i] for j in dsts})
    return sw, srcw, dstw


@pytest.mark.parametrize("style", ["pull", "push", "pushpull"])
def test_nar_dynamic_styles(style):
    g = golden("fig2_neighbor_sets.json")
    n = g["n"]
    rng = np.random.default_rng(4)
    W = np.eye(n)
    for a, b in g["edges_1indexed"]:
        W[b - 1, a - 1] = 1.0
    W = W * rng.uniform(0.1, 1.0, W.shape)
    sw, srcw, dstw = _views(W, style)
    ctx = _ctx(n)
    for count in (5, 8192, 40001):
        x, X = _inputs(n, count)
        y = ctx.neighbor_allreduce(x, self_weight=sw, src_weights=srcw, dst_weights=dstw)
        torch.cuda.synchronize()
        assert_parity(_np(y), ora.mix(W, X), W, X, 1e-6)
    ctx.close()


def test_nar_dynamic_time_varying_one_peer_push():
    # per-call weights that change every iteration: one-peer push form
    n = 8
    ctx = _ctx(n)
    x, X = _inputs(n, 20000)
    for k in range(5):
        dst = [{bfp.one_peer_exp2(n, i, k)[1]: 0.5} for i in range(n)]
        x = ctx.neighbor_allreduce(x, self_weight=[0.5] * n, dst_weights=dst)
        Wk = ora.one_peer_exp2(n, k)
        torch.cuda.synchronize()
        Y = _np(x)
        assert_parity(Y, ora.mix(Wk, X), Wk, X, 1e-6)
        X = Y
    ctx.close()


def test_nar_schedule_one_peer_exact_average():
    n = 8
    ctx = _ctx(n)
    ctx.set_dynamic_schedule("one_peer_exp2", 0)
    x, X0 = _inputs(n, 65537)
    X = X0
    for k in range(3):
        x = ctx.neighbor_allreduce(x)
        torch.cuda.synchronize()
        Wk = ora.one_peer_exp2(n, k)
        Y = _np(x)
        assert_parity(Y, ora.mix(Wk, X), Wk, X, 1e-6)
        X = Y
    mean = X0.mean(axis=0)
    assert np.abs(X - mean).max() <= 1e-6 * np.abs(X0).max()
    ctx.close()


@pytest.mark.parametrize("L", [4, 2, 8])
@pytest.mark.parametrize("op", ["nar", "atc"])
def test_schedule_inner_outer_exp2(L, op):
    # inner-outer dynamic exp-2 (R27), evaluated on device
    n = 8
    ctx = _ctx(n)
    ctx.set_machine_topology(ora.exp2(n // L) if n // L > 1 else np.ones((1, 1)), L)
    ctx.set_dynamic_schedule("inner_outer_exp2", 3)
    x, X = _inputs(n, 40003)
    for k in range(3, 3 + 2 * L):
        Wk = ora.inner_outer_exp2(n, L, k)
        if op == "nar":
            x = ctx.neighbor_allreduce(x)
            torch.cuda.synchronize()
            assert_parity(_np(x), ora.mix(Wk, X), Wk, X, 1e-6)
        else:
            g = _gpu(synthetic.agents_grad(n, 40003, k))
            G = _np(g)
            ctx.atc_step(x, g, 0.05)
            torch.cuda.synchronize()
            assert_parity(_np(x), ora.atc(Wk, X, G, 0.05), Wk, X, 1e-6, np.abs(Wk) @ (0.05 * np.abs(G)))
        X = _np(x).astype(np.float64)
    ctx.close()


@pytest.mark.parametrize("sched", ["one_peer_exp2", "inner_outer_exp2"])
def test_schedule_step_in_cuda_graph(sched):
    # The schedule round lives on the device (bf_set_dynamic_schedule), so one
    # captured ATC step replays as successive rounds (header: graph-capturable).
    n, L, count, lr = 8, 4, 20011, 0.05
    ctx = _ctx(n)
    ctx.set_machine_topology(ora.exp2(n // L), L)
    x, X = _inputs(n, count)
    g = _gpu(synthetic.agents_grad(n, count, 2))
    G = _np(g)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        ctx.atc_step(x, g, lr)                   # warm-up (allocates the exchange region)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    X = _np(x)
    ctx.set_dynamic_schedule(sched, 5)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        ctx.atc_step(x, g, lr)
    torch.cuda.synchronize()
    ctx.set_dynamic_schedule(sched, 5)           # capture does not run the kernel: restart at round 5
    for k in range(5, 5 + 2 * L):
        graph.replay()
        torch.cuda.synchronize()
        Wk = ora.one_peer_exp2(n, k) if sched == "one_peer_exp2" else ora.inner_outer_exp2(n, L, k)
        assert_parity(_np(x), ora.atc(Wk, X, G, lr), Wk, X, 1e-6, np.abs(Wk) @ (lr * np.abs(G)))
        X = _np(x)
    ctx.poll_error()
    del graph
    ctx.close()


# ---------------------------------------------------------------------- ATC ---
@pytest.mark.parametrize("wire", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("gdt", [torch.float32, torch.bfloat16])
def test_atc_step(wire, gdt):
    n = 8
    W = ora.exp2(n)
    ctx = _ctx(n)
    ctx.set_topology(W)
    lr = 0.1
    for count in (4096, 12345, 100000):
        x, X = _inputs(n, count)
        g = _gpu(synthetic.agents_grad(n, count, 3), gdt)
        G = _np(g)
        shadow = torch.empty(n, count, dtype=torch.bfloat16, device="cuda")
        ctx.atc_step(x, g, lr, wire=wire, shadow=shadow)
        torch.cuda.synchronize()
        ref = ora.atc(W, X, G, lr, wire_bf16=(wire == torch.bfloat16))
        extra = np.abs(W) @ (np.float32(lr) * np.abs(G))
        assert_parity(_np(x), ref, W, X, TOL[wire], extra)
        # the shadow is RNE(bf16) of the fp32 master
        assert torch.equal(shadow.cpu(), x.cpu().to(torch.bfloat16))
    ctx.close()


def test_atc_one_peer_schedule_and_lr0():
    n = 8
    ctx = _ctx(n)
    ctx.set_dynamic_schedule("one_peer_exp2", 0)
    x, X = _inputs(n, 30000)
    for k in range(4):
        g = _gpu(synthetic.agents_grad(n, 30000, k))
        G = _np(g)
        ctx.atc_step(x, g, 0.05)
        torch.cuda.synchronize()
        Wk = ora.one_peer_exp2(n, k)
        Y = _np(x)
        assert_parity(Y, ora.atc(Wk, X, G, 0.05), Wk, X, 1e-6, np.abs(Wk) @ (0.05 * np.abs(G)))
        X = Y
    ctx.close()


def test_atc_host_pointers_end_to_end():
    n = 4
    W = ora.ring(n)
    ctx = _ctx(n)
    ctx.set_topology(W)
    X = synthetic.agents_x0(n, 10000)
    G = synthetic.agents_grad(n, 10000, 0)
    xh = torch.from_numpy(X.copy()).pin_memory()
    gh = torch.from_numpy(G.copy()).pin_memory()
    ctx.atc_step(xh, gh, 0.1)
    torch.cuda.synchronize()
    ref = ora.atc(W, X.astype(np.float64), G.astype(np.float64), 0.1)
    assert_parity(xh.numpy().astype(np.float64), ref, W, X.astype(np.float64), 1e-6,
                  np.abs(W) @ (0.1 * np.abs(G.astype(np.float64))))
    ctx.close()


def test_c1_consensus_ring4_20_iterations():
    # C1: n=4 ring, fp32[4096], 20 iterations; chained per-step parity and the
    # end state against the fp64 trajectory (normalised by ||X0||_inf)
    n = 4
    W = ora.ring(n)
    ctx = _ctx(n)
    ctx.set_topology(W)
    x, X0 = _inputs(n, 4096)
    X = X0
    Xf = X0
    for _ in range(20):
        x = ctx.neighbor_allreduce(x)
        torch.cuda.synchronize()
        Y = _np(x)
        assert_parity(Y, ora.mix(W, X), W, X, 1e-6)
        X = Y
        Xf = ora.mix(W, Xf)
    assert np.abs(X - Xf).max() <= 1e-6 * np.abs(X0).max()
    ctx.close()


# --------------------------------------------------------- topology check ---
def test_topology_check_mismatch_is_an_error_not_a_hang():
    os.environ["BF_TIMEOUT_MS"] = "2000"
    ctx = _ctx(2)
    x, _ = _inputs(2, 1000)
    # agent 0 pushes to 1; agent 1 declares no source
    with pytest.raises(BluefogError):
        ctx.neighbor_allreduce(x, self_weight=[0.5, 1.0], src_weights=[None, {}], dst_weights=[{1: 0.5}, {}])
        torch.cuda.synchronize()
        ctx.poll_error()
    with pytest.raises(BluefogError) as e:
        ctx.neighbor_allreduce(x)
    assert e.value.name == "BF_ERR_STATE"
    ctx.close()
    os.environ["BF_TIMEOUT_MS"] = "5000"


def test_invalid_configurations_rejected_on_host():
    ctx = _ctx(2)
    x, _ = _inputs(2, 100)
    bad = [dict(self_weight=None, src_weights=[{1: 0.5}, {0: 0.5}]),          # no self weight
           dict(self_weight=[0.5, 0.5]),                                       # self only
           dict(self_weight=[0.5, 0.5], src_weights=[{0: 0.5}, {0: 0.5}]),     # self rank
           dict(self_weight=[0.5, 0.5], src_weights=[{5: 0.5}, {0: 0.5}]),     # out of range
           dict(self_weight=[float("nan"), 0.5], src_weights=[{1: 0.5}, {0: 0.5}])]
    for kw in bad:
        with pytest.raises(BluefogError) as e:
            ctx.neighbor_allreduce(x, **kw)
        assert e.value.name == "BF_ERR_ARG"
    ctx.neighbor_allreduce(x)                    # context still healthy
    torch.cuda.synchronize()
    ctx.close()


# ------------------------------------------------------------- hierarchical ---
@pytest.mark.parametrize("impl", ["fused", "staged"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("nm,L", [(4, 2), (2, 4), (1, 8), (8, 1), (2, 2)])
def test_hierarchical(nm, L, dtype, impl, monkeypatch):
    # one GPU: "fused" = the Kronecker mix W_M (x) J/L in the fused exchange kernel,
    # "staged" = the leader-free sliced kernel used across GPUs (BF_HIER=staged)
    monkeypatch.setenv("BF_HIER", impl)
    n = nm * L
    WM = ora.exp2(nm)
    ctx = _ctx(n)
    ctx.set_machine_topology(WM, L)
    K = np.kron(WM, np.full((L, L), 1.0 / L))
    for count in (3, 4096 * 3 + 1, 50000):
        x, X = _inputs(n, count, dtype)
        y = ctx.hierarchical_neighbor_allreduce(x)
        torch.cuda.synchronize()
        assert_parity(_np(y), ora.hier(WM, L, X), K, X, TOL[dtype])
    ctx.close()


@pytest.mark.parametrize("impl", ["fused", "staged"])
@pytest.mark.parametrize("gdt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("nm,L", [(4, 2), (2, 4), (1, 8)])
@pytest.mark.parametrize("style", ["atc", "awc"])
def test_hierarchical_atc_awc(style, nm, L, gdt, impl, monkeypatch):
    # H-ATC / H-AWC (caption P:869): the adapt fused into the hierarchical combine
    monkeypatch.setenv("BF_HIER", impl)
    n = nm * L
    WM = ora.exp2(nm)
    ctx = _ctx(n)
    ctx.set_machine_topology(WM, L)
    K = np.kron(WM, np.full((L, L), 1.0 / L))
    lr = 0.1
    for count in (3, 4096 * 3 + 1, 50000):
        x, X = _inputs(n, count)
        g = _gpu(synthetic.agents_grad(n, count, 7), gdt)
        G = _np(g)
        if style == "atc":
            ctx.hierarchical_atc_step(x, g, lr)
            ref, extra = ora.hier_atc(WM, L, X, G, lr), np.abs(K) @ (np.float32(lr) * np.abs(G))
        else:
            ctx.hierarchical_awc_step(x, g, lr)
            ref, extra = ora.hier_awc(WM, L, X, G, lr), np.float32(lr) * np.abs(G)
        torch.cuda.synchronize()
        assert_parity(_np(x), ref, K, X, 1e-6, extra)
    ctx.close()


def test_hierarchical_spec_example():
    gd = golden("hier_2x2_example.json")
    ctx = _ctx(4)
    ctx.set_machine_topology(np.array(gd["machine_W"]), gd["local_size"])
    x = _gpu(np.array(gd["inputs"]).reshape(4, 1))
    y = ctx.hierarchical_neighbor_allreduce(x)
    torch.cuda.synchronize()
    assert np.array_equal(_np(y).ravel(), np.array(gd["expected"]))
    ctx.close()


# ------------------------------------------------------------------ windows ---
def _fig2_static():
    g = golden("fig2_neighbor_sets.json")
    W = np.eye(g["n"])
    for a, b in g["edges_1indexed"]:
        W[b - 1, a - 1] = 1.0
    return W


def test_window_slot_layout_p388():
    gd = golden("window_layout_p388.json")
    n = 6                                   # nodes 0..5, paper node ids used directly
    W = np.eye(n)
    for s in gd["in_neighbors"]:
        W[gd["owner"], s] = 1.0
    ctx = _ctx(n)
    ctx.set_topology(W)
    numel = int(np.prod(gd["shape"]))
    x = torch.zeros(n, numel, device="cuda")
    ctx.win_create(x, "w")
    offs = [ctx.win_slot_offset("w", gd["owner"], s) for s in gd["slot_order"]]
    assert offs == [0, numel]
    assert numel * len(gd["in_neighbors"]) == gd["logical_elements"]
    ctx.win_free("w")
    ctx.close()


def test_window_sync_pushsum_matches_oracle():
    """Synchronous push-sum rounds (all accumulate, then all collect; Listing 3
    weights 1/(outdeg+1)) on the Fig. 2 graph.  One round is one product
    with the column-stochastic push matrix (oracle pin test_window_sync_pushsum_equals_mix);
    each round is checked on the GPU's previous state by the 1e-6 forward-error rule
    (DESIGN.md "Parity"), and the fp64 p lane exactly against the event model."""
    Wst = _fig2_static()
    n = Wst.shape[0]
    count = 9000
    X0 = synthetic.agents_x0(n, count).astype(np.float64)
    ctx = _ctx(n)
    ctx.set_topology(Wst)
    x = _gpu(X0)
    ctx.win_create(x, "ps", zero_init=True, with_p=True)
    Wps = np.zeros((n, n))
    for i in range(n):
        outs = ora.out_neighbors(Wst, i)
        w = 1.0 / (len(outs) + 1)
        Wps[i, i] = w
        for j in outs:
            Wps[j, i] = w
    ext = np.concatenate([X0, np.ones((n, 1))], axis=1)
    win = ora.Window(Wst, ext, zero_init=True)
    for _ in range(6):
        X = _np(x)
        ctx.win_accumulate("ps")                 # Listing 3 weights 1/(outdeg+1)
        ctx.win_update_then_collect("ps")
        for i in range(n):
            outs = ora.out_neighbors(Wst, i)
            w = 1.0 / (len(outs) + 1)
            win.accumulate(i, w, {j: w for j in outs})
        for i in range(n):
            win.collect(i)
        torch.cuda.synchronize()
        assert_parity(_np(x), ora.mix(Wps, X), Wps, X, 1e-6)
    ref = win.x()
    assert np.allclose(ctx.win_p("ps"), ref[:, -1], rtol=0, atol=1e-12)
    ctx.win_free("ps")
    ctx.close()


@pytest.mark.parametrize("dtype,ef", [(torch.float32, False), (torch.bfloat16, False), (torch.bfloat16, True)])
def test_window_async_event_model(dtype, ef):
    # random per-agent interleaving of accumulate / collect (agent_mask selects
    # the acting agent); the GPU follows the oracle's state machine event by event
    # (bf16: with and without error feedback of the wire rounding, R24)
    Wst = _fig2_static()
    n = Wst.shape[0]
    count = 4099
    ctx = _ctx(n)
    ctx.set_topology(Wst)
    x = _gpu(synthetic.agents_x0(n, count), dtype)
    X0 = _np(x)
    ctx.win_create(x, "a", zero_init=True, with_p=True)
    if ef:
        ctx.win_set_error_feedback("a", True)
    win = ora.Window(Wst, np.concatenate([X0, np.ones((n, 1))], axis=1), zero_init=True)
    rng = np.random.default_rng(7)
    mass0 = X0.sum(axis=0)
    for _ in range(150):
        i = int(rng.integers(n))
        if rng.random() < 0.5:
            ctx.win_accumulate("a", agent_mask=1 << i)
            outs = ora.out_neighbors(Wst, i)
            w = 1.0 / (len(outs) + 1)
            win.accumulate(i, w, {j: w for j in outs})
        else:
            ctx.win_update_then_collect("a", agent_mask=1 << i)
            win.collect(i)
    torch.cuda.synchronize()
    for i in range(n):
        for j in ora.out_neighbors(Wst, i):
            v, c = ctx.win_counters("a", j, i)
            assert (v, c) == win.counters(j, i)
    ref = win.x()
    assert np.allclose(ctx.win_p("a"), ref[:, -1], rtol=0, atol=1e-12)
    # the window's internal state (slots, outboxes) cannot be fed back event by
    # event, so the end state is compared with the fp64 event model: every event
    # rounds each touched value at most twice (payload, x) to the window dtype, and
    # |x| <= 1, so after 150 events the absolute error is at most
    # 150 * 2 * 2^-24 ~ 1.8e-5 (fp32) -> 3e-5; bf16 storage: 2^-8 per rounding of a
    # value <= 1, a few roundings per value along a chain -> 2e-2
    tol = 3e-5 if dtype == torch.float32 else 2e-2
    assert np.abs(_np(x) - ref[:, :-1]).max() < tol
    # flush: every agent pushes its outbox and collects, twice -> mass conserved
    for _ in range(3):
        ctx.win_accumulate("a", self_weight=[1.0] * n, dst_weights=[{j: 0.0 for j in ora.out_neighbors(Wst, i)}
                                                                   for i in range(n)])
        ctx.win_update_then_collect("a")
    torch.cuda.synchronize()
    mass = _np(x).sum(axis=0)
    mtol = 1e-4 if dtype == torch.float32 else 5e-2
    assert np.abs(mass - mass0).max() < mtol
    assert abs(ctx.win_p("a").sum() - n) < 1e-12
    ctx.win_free("a")
    ctx.close()


def test_window_put_and_update():
    # S:454 example: ring(3) after each in-neighbour puts {3, 9} and local 0,
    # uniform 1/3 -> 4; idempotent when called twice
    W = ora.ring(3)
    ctx = _ctx(3)
    ctx.set_topology(W)
    x = _gpu(np.array([[0.0], [3.0], [9.0]]))
    ctx.win_create(x, "u", zero_init=True)
    ctx.win_put("u", self_weight=[1.0] * 3, dst_weights=[{1: 1.0, 2: 1.0}, {0: 1.0, 2: 1.0}, {0: 1.0, 1: 1.0}])
    out = torch.empty_like(x)
    ctx.win_update("u", out=out)
    torch.cuda.synchronize()
    assert abs(_np(out)[0, 0] - 4.0) < 1e-6
    ctx.win_update("u", out=out)
    torch.cuda.synchronize()
    assert abs(_np(out)[0, 0] - 4.0) < 1e-6
    # non-zero-init: buffers start as the local tensor -> update returns x
    ctx.win_create(x, "v", zero_init=False)
    ctx.win_update("v", out=out)
    torch.cuda.synchronize()
    assert np.allclose(_np(out), _np(x), atol=1e-6)
    ctx.win_free("v")
    ctx.win_free("u")
    ctx.close()


def test_window_dst_outside_creation_topology():
    W = ora.ring(4)
    ctx = _ctx(4)
    ctx.set_topology(W)
    x = torch.zeros(4, 10, device="cuda")
    ctx.win_create(x, "d")
    with pytest.raises(BluefogError) as e:
        ctx.win_accumulate("d", self_weight=[0.5] * 4, dst_weights=[{2: 0.5}, {2: 0.5}, {3: 0.5}, {0: 0.5}])
    assert e.value.name == "BF_ERR_WINDOW"
    ctx.win_free("d")
    ctx.close()


# ------------------------------------------------ bench configuration (C4) ---
def test_bench_config_c4_sampled():
    """8 agents x 25.6M fp32, the launch configuration bench.py times; outputs
    checked on sampled columns the oracle computes one by one."""
    n, count, lr = 8, 25_600_000, 0.1
    ctx = _ctx(n, heap=3 << 30)
    ctx.set_dynamic_schedule("one_peer_exp2", 0)
    x = torch.empty(n, count, device="cuda")
    g = torch.empty(n, count, device="cuda")
    for r in range(n):
        bfp.Context.fill_uniform(x[r], synthetic.SEED_X0 + r)
        bfp.Context.fill_uniform(g[r], synthetic.grad_seed(0, r), scale=2.0 ** -7)
    rng = np.random.default_rng(0)
    cols = np.unique(np.concatenate([rng.integers(0, count, 2000), [0, 1, 4095, 4096, count - 1]]))
    Xs = np.stack([np.concatenate([synthetic.uniform(synthetic.SEED_X0 + r, 1, offset=int(c)) for c in cols])
                   for r in range(n)]).astype(np.float64)
    Gs = np.stack([np.concatenate([synthetic.uniform(synthetic.grad_seed(0, r), 1, scale=2.0 ** -7, offset=int(c))
                                   for c in cols]) for r in range(n)]).astype(np.float64)
    assert np.array_equal(x[:, torch.from_numpy(cols).cuda()].cpu().numpy(), Xs.astype(np.float32))
    ctx.atc_step(x, g, lr)
    torch.cuda.synchronize()
    W0 = ora.one_peer_exp2(n, 0)
    ref = ora.atc(W0, Xs, Gs, lr)
    got = x[:, torch.from_numpy(cols).cuda()].cpu().numpy().astype(np.float64)
    assert_parity(got, ref, W0, Xs, 1e-6, np.abs(W0) @ (lr * np.abs(Gs)))
    ctx.close()


# ------------------------------------------------------- AWC / non-blocking ---
@pytest.mark.parametrize("gdt", [torch.float32, torch.bfloat16])
def test_awc_step(gdt):
    # Eq. 16: x_i <- sum_j w_ij x_j - lr * g_i
    n, lr = 8, 0.1
    W = ora.exp2(n)
    ctx = _ctx(n)
    ctx.set_topology(W)
    for count in (4096, 50001):
        x, X = _inputs(n, count)
        g = _gpu(synthetic.agents_grad(n, count, 7), gdt)
        G = _np(g)
        ctx.awc_step(x, g, lr)
        torch.cuda.synchronize()
        assert_parity(_np(x), ora.awc(W, X, G, lr), W, X, 1e-6, np.float32(lr) * np.abs(G))
    ctx.close()


def test_nonblocking_equals_blocking():
    # neighbor_allreduce_nonblocking + wait == the blocking call
    n = 4
    ctx = _ctx(n)
    ctx.set_topology(ora.ring(n))
    x, X = _inputs(n, 30001)
    h = ctx.neighbor_allreduce_nonblocking(x)
    z = torch.ones(1000, device="cuda").sum()      # computation overlapping the exchange
    y1 = bfp.Context.wait(h)
    y2 = ctx.neighbor_allreduce(x)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2) and float(z) == 1000.0
    assert_parity(_np(y1), ora.mix(ora.ring(n), X), ora.ring(n), X, 1e-6)
    ctx.close()


def test_hierarchical_machine_size_change():
    n = 8
    ctx = _ctx(n)
    x, X = _inputs(n, 20000)
    for L in (2, 4, 2):
        WM = ora.exp2(n // L)
        ctx.set_machine_topology(WM, L)
        y = ctx.hierarchical_neighbor_allreduce(x)
        torch.cuda.synchronize()
        assert_parity(_np(y), ora.hier(WM, L, X), np.kron(WM, np.full((L, L), 1.0 / L)), X, 1e-6)
    ctx.close()


# ------------------------------------------- exchange kernels x local agents ---
@pytest.mark.parametrize("kernel", ["fused", "chunk"])
@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_exchange_kernels_all_ops(kernel, n, monkeypatch):
    """Every exchange kernel (BF_EXCH) against the oracle for the three fused
    ops -- neighbor_allreduce (Eq. 5), ATC (Eq. 4-5, 17), AWC (Eq. 16) -- with
    n virtual agents on one GPU (the fused kernel applies W in registers),
    over sizes with ragged tails and unaligned rows (count % 4 != 0)."""
    monkeypatch.setenv("BF_EXCH", kernel)
    lr = 0.1
    ctx = _ctx(n)
    rng = np.random.default_rng(n)
    W = ora.exp2(n) if n > 1 else np.eye(1)
    if n > 2:   # a directed random graph with negative weights as well
        W = W + (rng.random((n, n)) < 0.3) * rng.uniform(-0.5, 0.5, (n, n))
    ctx.set_topology(W)
    for count in (1, 7, 1023, 1024, 4097, 70001):
        x, X = _inputs(n, count)
        y = ctx.neighbor_allreduce(x)
        torch.cuda.synchronize()
        assert_parity(_np(y), ora.mix(W, X), W, X, 1e-6)
        for wire in (torch.float32, torch.bfloat16):
            g = _gpu(synthetic.agents_grad(n, count, 5))
            G = _np(g)
            xa = x.clone()
            ctx.atc_step(xa, g, lr, wire=wire)
            torch.cuda.synchronize()
            extra = np.abs(W) @ (np.float32(lr) * np.abs(G))
            assert_parity(_np(xa), ora.atc(W, X, G, lr, wire_bf16=(wire == torch.bfloat16)), W, X,
                          TOL[wire], extra)
        xw = x.clone()
        ctx.awc_step(xw, g, lr)
        torch.cuda.synchronize()
        assert_parity(_np(xw), ora.awc(W, X, G, lr), W, X, 1e-6, np.float32(lr) * np.abs(G))
    ctx.close()


# ----------------------------------------- optimizer wrapper: tensor fusion + ATC ---
@pytest.mark.parametrize("overlap", [False, True])
@pytest.mark.parametrize("awc", [False, True])
def test_optimizer_bucketed_matches_oracle(overlap, awc):
    """DistributedAdaptThenCombineOptimizer: parameters re-homed into
    bucket buffers, one fused call per bucket (from backward hooks when
    overlap) == the oracle's ATC / AWC (Eq. 17 / Eq. 16) of the concatenated
    per-agent vectors: bucketing is invisible to the result."""
    from paper_2111_04287_b200.optim import DistributedAdaptThenCombineOptimizer
    n, lr = 4, 0.05
    ctx = _ctx(n)
    W = ora.exp2(n)
    ctx.set_topology(W)
    shapes = [(7, 3), (129,), (64, 65), (5,), (1000,), (33, 17)]
    torch.manual_seed(0)
    params = [torch.nn.Parameter(torch.randn(n, *s, device="cuda")) for s in shapes]
    X = np.concatenate([_np(p.detach().reshape(n, -1)) for p in params], axis=1)
    # with overlap: steps on a side stream during backward, exchange capped at 24 CTAs
    opt = DistributedAdaptThenCombineOptimizer(ctx, params, lr, bucket_bytes=4 * 2000, overlap=overlap, awc=awc,
                                               overlap_ctas=24 if overlap else 0)
    assert len(opt.buckets) >= 3
    # gradients from a real backward: loss = sum_i c_i * sum(p_i^2) / 2  ->  g_i = c_i * p_i
    coef = [0.1 * (i + 1) for i in range(len(params))]
    loss = sum(c * (p * p).sum() / 2 for c, p in zip(coef, params))
    opt.zero_grad()
    loss.backward()
    widths = [int(np.prod(sh)) for sh in shapes]
    G = X * np.concatenate([np.full(w_, np.float32(c)) for c, w_ in zip(coef, widths)])[None, :]
    # the gradient buffers hold exactly what backward produced
    Gb = np.concatenate([_np(p.grad.reshape(n, -1)) for p in params], axis=1)
    assert np.allclose(Gb, G, rtol=1e-6, atol=1e-7)
    opt.step()
    torch.cuda.synchronize()
    Y = np.concatenate([_np(p.detach().reshape(n, -1)) for p in params], axis=1)
    ref = ora.awc(W, X, Gb, lr) if awc else ora.atc(W, X, Gb, lr)
    extra = np.float32(lr) * np.abs(Gb) if awc else np.abs(W) @ (np.float32(lr) * np.abs(Gb))
    assert_parity(Y, ref, W, X, 1e-6, extra)
    assert opt.steps_launched == len(opt.buckets)
    opt.remove_hooks()
    ctx.close()


# ------------------------------------ Exact-Diffusion (appendix ed-1..ed-3, §8(f) 4) ---
@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("wire,gdt", [(torch.float32, torch.float32), (torch.bfloat16, torch.float32),
                                      (torch.float32, torch.bfloat16)])
def test_exact_diffusion_step(n, wire, gdt):
    lr = 0.1
    ctx = _ctx(n)
    W = ora.exp2(n) if n > 1 else np.eye(1)
    ctx.set_topology(W)
    for count in (1, 7, 1023, 4097, 70001):
        x, X = _inputs(n, count)
        g = _gpu(synthetic.agents_grad(n, count, 2), gdt)
        G = _np(g)
        psi = _gpu(synthetic.agents_grad(n, count, 9) * 64.0)
        P = _np(psi)
        ctx.exact_diffusion_step(x, g, psi, lr, wire=wire)
        torch.cuda.synchronize()
        ref, pref = ora.exact_diffusion(W, X, G, P, lr, wire_bf16=(wire == torch.bfloat16))
        scale = np.abs(W) @ (2 * np.abs(X) + np.float32(lr) * np.abs(G) + np.abs(P))
        assert_parity(_np(x), ref, W, X, TOL[wire], scale - np.abs(W) @ np.abs(X))
        assert np.abs(_np(psi) - pref).max() <= 1e-6 * (np.abs(X) + lr * np.abs(G)).max()
    ctx.close()


def test_exact_diffusion_reaches_exact_minimiser_on_gpu():
    # least squares (Eq. 12-13 shape, small): ED with a constant step converges to x*
    # (the appendix's bias correction), gradients by torch bmm (workload plumbing)
    # exp-2 on 8 agents: weights 1/4, exactly doubly stochastic in fp32.  (With 1/3
    # weights the fp32 rows sum to 1 + 3e-8; ED integrates that into a ~1e-4 offset
    # of its fixed point -- reading R25 in DESIGN.md.)
    n, m, d, lr = 8, 64, 32, 0.5
    rng = np.random.default_rng(5)
    A = rng.standard_normal((n, m, d)) / np.sqrt(m)
    b = rng.standard_normal((n, m))
    xs = np.linalg.lstsq(A.reshape(n * m, d), b.reshape(n * m), rcond=None)[0]
    ctx = _ctx(n)
    ctx.set_topology(ora.exp2(n))
    # the gradient in fp64 (plumbing; a TF32 GEMM would move the fixed point by ~1e-4)
    At = torch.from_numpy(A).cuda()
    bt = torch.from_numpy(b).cuda()
    x = torch.zeros(n, d, device="cuda")
    psi = x.clone()
    for _ in range(4000):
        x64 = x.double()
        g = torch.bmm(At.transpose(1, 2), (torch.bmm(At, x64.unsqueeze(2)).squeeze(2) - bt).unsqueeze(2)).squeeze(2)
        ctx.exact_diffusion_step(x, g.float().contiguous(), psi, lr)
    torch.cuda.synchronize()
    err = np.abs(_np(x) - xs[None, :]).max()
    assert err < 1e-5 * np.abs(xs).max(), err   # the fp32 oracle reaches 3e-7 on this problem
    ctx.close()


# ------------------------- push-sum gradient tracking: two fused launches per round ---
@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_gradient_tracking_matches_oracle_and_converges(n):
    """appendix "Push-sum gradient tracking" (lines 1000-1006): gt_uv_step (MODE 5:
    u <- W(u - lr y), v <- W v, x = u / v) and gt_y_step (MODE 4: y <- W(y + g - g_prev)),
    a directed column-stochastic W; each launch checked against ora.gt_uv / ora.gt_y
    on the GPU's state (tolerance rule with b = sum_j |w_ij| (|u_j| + lr|y_j|), resp.
    (|y_j| + |g_j| + |g_prev_j|)); then convergence to the least-squares minimiser."""
    from paper_2111_04287_b200.algorithms import gradient_tracking_step
    m, d, lr = 10, 4099, 0.05
    rng = np.random.default_rng(8)
    A = rng.standard_normal((n, m, d)) / np.sqrt(m) / 8
    b = rng.standard_normal((n, m))
    Adj = np.eye(n, dtype=bool)
    r2 = np.random.default_rng(2)
    for i in range(n):
        Adj[(i + 1) % n, i] = True
        for j in r2.choice(n, min(2, n), replace=False):
            Adj[j, i] = True
    W = Adj / Adj.sum(axis=0, keepdims=True)
    ctx = _ctx(n)
    ctx.set_topology(W)
    At = torch.from_numpy(A).cuda()
    bt = torch.from_numpy(b).cuda()

    def grad_gpu(X):   # fp64 GEMV plumbing, fp32 result
        X64 = X.double()
        return torch.bmm(At.transpose(1, 2), (torch.bmm(At, X64.unsqueeze(2)).squeeze(2) - bt).unsqueeze(2)) \
            .squeeze(2).float().contiguous()
    u = _gpu(synthetic.agents_x0(n, d) * 0.1)
    v = torch.ones(n, device="cuda")
    g = grad_gpu(u)
    y = g.clone()
    x = torch.empty_like(u)
    for step in range(4):
        U, V, Y = _np(u), _np(v)[:, None], _np(y)
        ctx.gt_uv_step(u, v, y, x, lr)
        torch.cuda.synchronize()
        Ur, Vr, Xr = ora.gt_uv(W, U, V, Y, lr)
        bu = np.abs(W) @ (np.abs(U) + np.float32(lr) * np.abs(Y))
        assert np.all(np.abs(_np(u) - Ur) <= 1e-6 * bu + 1e-30), f"u step {step}"
        assert np.allclose(_np(v), Vr[:, 0], rtol=1e-6, atol=0)
        # x = u / v: the forward error of u scaled by 1/v, plus one fp32 rounding
        assert np.all(np.abs(_np(x) - Xr) <= (1e-6 * bu + 2.0 ** -24 * np.abs(Xr)) / np.abs(Vr) * 1.001 + 1e-30)
        gn = grad_gpu(x)
        Y0, Gn, Gp = _np(y), _np(gn), _np(g)
        ctx.gt_y_step(y, gn, g)
        torch.cuda.synchronize()
        by = np.abs(W) @ (np.abs(Y0) + np.abs(Gn) + np.abs(Gp))
        assert np.all(np.abs(_np(y) - ora.gt_y(W, Y0, Gn, Gp)) <= 1e-6 * by + 1e-30), f"y step {step}"
        g = gn
    # convergence (small problem, d = 4): the listing's loop through the library's two launches
    ctx.close()
    d2 = 4
    A2 = rng.standard_normal((n, m, d2)) / np.sqrt(m)
    b2 = rng.standard_normal((n, m))
    xs = np.linalg.lstsq(A2.reshape(n * m, d2), b2.reshape(n * m), rcond=None)[0]
    ctx = _ctx(n)
    ctx.set_topology(W)
    A2t, b2t = torch.from_numpy(A2).cuda(), torch.from_numpy(b2).cuda()
    g2 = lambda X: torch.bmm(A2t.transpose(1, 2), (torch.bmm(A2t, X.double().unsqueeze(2)).squeeze(2) - b2t)
                             .unsqueeze(2)).squeeze(2).float().contiguous()
    u = torch.zeros(n, d2, device="cuda")
    v = torch.ones(n, device="cuda")
    gp = g2(u)
    y = gp.clone()
    for _ in range(3000):
        x, u, v, y, gp = gradient_tracking_step(ctx, u, v, y, gp, g2, 0.05)
    torch.cuda.synchronize()
    assert abs(float(v.sum()) - n) < 1e-4                      # column-stochastic: sum v = n
    assert np.abs(_np(x) - xs[None, :]).max() < 1e-4 * max(1.0, np.abs(xs).max())
    ctx.close()


# ------------------------------------------------ neighbor_win_get (R26) ---
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_window_get(dtype):
    Wst = _fig2_static()
    n = Wst.shape[0]
    count = 10007
    ctx = _ctx(n)
    ctx.set_topology(Wst)
    x = ctx.alloc((n, count), dtype)                       # symmetric heap: readable by the neighbours
    x.copy_(_gpu(synthetic.agents_x0(n, count), dtype))
    X = _np(x)
    ctx.win_create(x, "g", zero_init=True)
    rng = np.random.default_rng(3)
    ins = [[j for j in range(n) if j != i and Wst[i, j] != 0] for i in range(n)]
    Wg = np.zeros((n, n))
    views = []
    for i in range(n):
        sel = {j: float(rng.uniform(0.1, 1.0)) for j in ins[i] if rng.random() < 0.8}
        for j, w in sel.items():
            Wg[i, j] = w
        views.append(sel)
    ctx.win_get("g", src_weights=views)
    out = torch.empty_like(x)
    # win_update with self 0 and unit weights: out_i = sum_j (fetched w_ij x_j)
    ctx.win_update("g", self_weight=[0.0] * n, src_weights=[{j: 1.0 for j in views[i]} for i in range(n)], out=out)
    torch.cuda.synchronize()
    ref = ora.mix(Wg, X)
    tol = 1e-6 if dtype == torch.float32 else 2e-2
    assert_parity(_np(out), ref, Wg, X, tol)
    # default: every in-neighbour, weight 1
    ctx.win_get("g")
    ctx.win_update("g", self_weight=[0.0] * n, src_weights=[{j: 1.0 for j in ins[i]} for i in range(n)], out=out)
    torch.cuda.synchronize()
    W1 = (Wst != 0).astype(np.float64)
    np.fill_diagonal(W1, 0.0)
    assert_parity(_np(out), ora.mix(W1, X), W1, X, tol)
    ctx.win_free("g")
    # a window on memory outside the heap cannot be read by the neighbours
    y = _gpu(synthetic.agents_x0(n, 64), dtype)
    ctx.win_create(y, "h", zero_init=True)
    with pytest.raises(BluefogError) as ei:
        ctx.win_get("h")
    assert ei.value.name == "BF_ERR_UNSUPPORTED"
    ctx.win_free("h")
    ctx.close()


def test_empty_inputs_are_noops():
    # count = 0 (an empty layer, a ragged split): every data call returns without
    # launching a kernel and without touching the epoch (the next call still works)
    n = 4
    ctx = _ctx(n)
    ctx.set_topology(ora.ring(n))
    e = torch.empty(n, 0, device="cuda")
    l0 = ctx.kernel_launches()
    ctx.neighbor_allreduce(e)
    ctx.atc_step(e, e, 0.1)
    ctx.awc_step(e, e, 0.1)
    ctx.exact_diffusion_step(e, e, e.clone(), 0.1)
    torch.cuda.synchronize()
    assert ctx.kernel_launches() == l0
    x, X = _inputs(n, 4097)
    y = ctx.neighbor_allreduce(x)
    torch.cuda.synchronize()
    assert_parity(_np(y), ora.mix(ora.ring(n), X), ora.ring(n), X, 1e-6)
    ctx.close()
