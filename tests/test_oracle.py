"""Pins for the CPU oracle (oracle/), checked against what the paper and the
mathematics fix -- never against the CUDA path.  CPU only (-m "not gpu").

Each test names the passage it pins (P:NNN = PAPER.md line, S:NNN = SPEC.md
line used for worked scalar examples).
"""
import numpy as np
import pytest

import oracle as ora
import synthetic
from bfutil import golden


def _edges_to_W(n, edges, one_indexed=False):
    """Adjacency-weighted matrix with W[i][j] != 0 iff edge j -> i."""
    W = np.eye(n)
    for (a, b) in edges:
        if one_indexed:
            a, b = a - 1, b - 1
        W[b, a] = 1.0
    return W


# ---------------------------------------------------------------- topology ---
def test_neighbor_sets_fig2():
    g = golden("fig2_neighbor_sets.json")
    W = _edges_to_W(g["n"], g["edges_1indexed"], one_indexed=True)
    node = g["node"] - 1
    assert [j + 1 for j in ora.in_neighbors(W, node)] == g["in_neighbors"]
    assert [j + 1 for j in ora.out_neighbors(W, node)] == g["out_neighbors"]
    # reversing every edge swaps N and M (Eq. 6-7 definitions)
    Wt = W.T.copy()
    assert [j + 1 for j in ora.out_neighbors(Wt, node)] == g["in_neighbors"]


def test_weight_classes():
    # pull = rows sum to 1, push = columns, standard = both
    assert ora.classify(np.eye(3)) == "standard"
    assert ora.classify(np.full((4, 4), 0.25)) == "standard"
    P = np.array([[0.5, 0.5, 0.0], [0.0, 0.2, 0.8], [0.3, 0.3, 0.4]])
    assert ora.classify(P) == "pull"
    assert ora.classify(P.T) == "push"
    assert ora.classify(P * 2) == "none"


def test_exp2_structure():
    # P:446 static exponential graph (reading R4): node 0 of n=8 sends to {1,2,4}
    W = ora.exp2(8)
    assert ora.out_neighbors(W, 0) == [1, 2, 4]
    assert ora.in_neighbors(W, 0) == [4, 6, 7]
    assert np.allclose(W[W != 0], 0.25)
    degs = [len(ora.in_neighbors(ora.exp2(n), 0)) for n in range(2, 9)]
    assert degs == [1, 2, 2, 3, 3, 3, 3]
    for n in range(2, 17):
        assert ora.classify(ora.exp2(n)) == "standard"   # P:231 "special directed graphs such as the exponential graph"


def test_exp2_circulant_spectrum():
    # exp2(n) is circulant: eigenvalues are the DFT of its first column pattern
    n = 8
    W = ora.exp2(n)
    c = W[0]                                       # W[i][j] = c[(j - i) mod n]
    for i in range(n):
        assert np.array_equal(W[i], np.roll(c, i))
    omega = np.exp(2j * np.pi / n)
    lam = np.array([sum(c[k] * omega ** (m * k) for k in range(n)) for m in range(n)])
    ev = np.linalg.eigvals(W)
    assert np.allclose(np.sort(np.abs(ev)), np.sort(np.abs(lam)), atol=1e-12)
    assert abs(np.sort(np.abs(lam))[-2] - 0.5) < 1e-12


def test_ring_structure():
    W = ora.ring(5)
    assert ora.in_neighbors(W, 0) == [1, 4]
    assert np.allclose(W[W != 0], 1 / 3)
    assert ora.classify(W) == "standard"
    W2 = ora.ring(2)
    assert np.allclose(W2, 0.5)


def test_one_peer_schedule_and_exact_average():
    # P:916 one-peer dynamic exponential graph; reading R5.  For n = 2^tau the
    # product over t of (I + S^{2^t})/2 is J/n: exact average after tau rounds.
    assert ora.one_peer_exp2_peers(8, 0, 0) == (7, 1)
    assert ora.one_peer_exp2_peers(8, 1, 0) == (6, 2)
    assert ora.one_peer_exp2_peers(8, 2, 0) == (4, 4)
    assert ora.one_peer_exp2_peers(8, 3, 0) == (7, 1)
    assert ora.one_peer_exp2_peers(2, 5, 1) == (0, 0)
    for n in (2, 4, 8, 16):
        tau = n.bit_length() - 1
        X = synthetic.agents_x0(n, 257).astype(np.float64)
        mean = X.sum(axis=0) / n                  # exact in fp64 for these dyadic inputs
        for k in range(tau):
            Wk = ora.one_peer_exp2(n, k)
            assert ora.classify(Wk) == "standard"
            X = ora.mix(Wk, X)
        assert np.array_equal(X, np.broadcast_to(mean, X.shape))
    # non power of two: defined but not exact (reading R20)
    X = synthetic.agents_x0(6, 64).astype(np.float64)
    Y = X
    for k in range(3):
        Y = ora.mix(ora.one_peer_exp2(6, k), Y)
    assert np.abs(Y - X.mean(axis=0)).max() > 1e-3


def test_inner_outer_exp2_schedule():
    # P:828 / P:869, reading R27: hand-derived tables, then properties.
    g = golden("inner_outer_exp2_tables.json")
    for case in g["cases"]:
        n, L = case["n"], case["local_size"]
        for k, srcs in enumerate(case["src_by_round"]):
            for i in range(n):
                assert ora.inner_outer_exp2_peers(n, L, k, i)[0] == srcs[i], (n, L, k, i)
    for n, L in ((8, 4), (8, 2), (16, 4), (12, 3), (8, 8), (6, 1), (16, 8)):
        M = n // L
        for k in range(2 * n):
            W = ora.inner_outer_exp2(n, L, k)
            assert np.allclose(W.sum(axis=0), 1) and np.allclose(W.sum(axis=1), 1)   # doubly stochastic
            assert ((W != 0).sum(axis=1) <= 2).all() and ((W != 0).sum(axis=0) <= 2).all()  # one peer
            crossing = 0
            for i in range(n):
                s, d = ora.inner_outer_exp2_peers(n, L, k, i)
                if s < 0:
                    assert d < 0 and W[i, i] == 1.0
                    continue
                assert ora.inner_outer_exp2_peers(n, L, k, d)[0] == i      # dst's source is i
                if s // L != i // L:
                    crossing += 1
                    assert s % L == i % L == k % L                           # the outer rank, same slot
                    dm = (i // L - s // L) % M
                    assert dm & (dm - 1) == 0                                # distance 2^t
            assert crossing == (M if M > 1 else 0)                          # one outer agent per machine
    for k in range(12):   # L = 1: every agent is its own machine -> the plain one-peer exp-2 graph
        assert np.array_equal(ora.inner_outer_exp2(8, 1, k), ora.one_peer_exp2(8, k))


def test_hierarchical_atc_awc_special_cases():
    # H-ATC / H-AWC: L = 1 reduces to the plain ATC / AWC over W_M
    # (Eqs. 17, 16); one machine (L = n) gives every agent the exact average.
    n, d, lr = 8, 333, 0.25
    X = synthetic.agents_x0(n, d).astype(np.float64)
    G = synthetic.agents_grad(n, d, 5).astype(np.float64)
    W = ora.exp2(n)
    assert np.allclose(ora.hier_atc(W, 1, X, G, lr), ora.atc(W, X, G, lr), rtol=0, atol=1e-14)
    assert np.allclose(ora.hier_awc(W, 1, X, G, lr), ora.awc(W, X, G, lr), rtol=0, atol=1e-14)
    one = np.ones((1, 1))
    mean_adapted = (X - lr * G).astype(np.float32).astype(np.float64).mean(axis=0)   # fp32 adapted copy (R18)
    assert np.allclose(ora.hier_atc(one, n, X, G, lr), np.broadcast_to(mean_adapted, X.shape), rtol=0, atol=1e-14)
    assert np.allclose(ora.hier_awc(one, n, X, G, lr), X.mean(axis=0) - lr * G, rtol=0, atol=1e-14)
    assert np.array_equal(ora.hier_atc(ora.ring(4), 2, X, G, 0.0), ora.hier(ora.ring(4), 2, X))


# ------------------------------------------------------------------- mixing ---
def test_mix_identity_and_uniform():
    g = golden("spec_scalar_examples.json")
    X = synthetic.agents_x0(3, 100).astype(np.float64)
    assert np.array_equal(ora.mix(np.eye(3), X), X)
    Y = ora.mix(ora.full(4), np.array(g["full4_inputs"]).reshape(4, 1))
    assert np.allclose(Y, g["full4_expected"], rtol=0, atol=1e-15)


def test_mix_bruteforce_small():
    rng = np.random.default_rng(0)
    for n in (1, 2, 3, 5, 8):
        W = rng.standard_normal((n, n))
        X = rng.standard_normal((n, 7))
        Y = ora.mix(W, X)
        for i in range(n):
            for e in range(7):
                ref = sum(W[i, j] * X[j, e] for j in range(n))
                assert abs(Y[i, e] - ref) <= 1e-14 * (1 + sum(abs(W[i, j] * X[j, e]) for j in range(n)))


def test_mean_preservation_and_fixed_point():
    # a doubly stochastic W preserves column sums; a row-stochastic
    # (pull) W keeps constant vectors fixed (consensus is a fixed point).
    X = synthetic.agents_x0(8, 333).astype(np.float64)
    for W in (ora.exp2(8), ora.ring(8), ora.one_peer_exp2(8, 1)):
        assert np.allclose(ora.mix(W, X).sum(axis=0), X.sum(axis=0), atol=1e-13)
    P = np.array([[0.5, 0.5, 0.0], [0.0, 0.2, 0.8], [0.3, 0.3, 0.4]])
    c = np.ones((3, 5)) * 0.75
    assert np.allclose(ora.mix(P, c), c, atol=1e-15)


def test_matrix_power_bruteforce():
    for n in (2, 3, 4, 5, 8):
        W = ora.exp2(n)
        X = synthetic.agents_x0(n, 33).astype(np.float64)
        Y = X
        for _ in range(6):
            Y = ora.mix(W, Y)
        assert np.allclose(Y, np.linalg.matrix_power(W, 6) @ X, atol=1e-13)


def test_ring4_consensus_closed_form_c1():
    # C1: n=4 ring, 20 iterations.  Ring W is circulant with eigenvalues
    # {1, 1/3, -1/3, 1/3}; X^20 = F^-1 diag(lambda^20) F X in closed form.
    n, K = 4, 20
    W = ora.ring(n)
    X0 = synthetic.agents_x0(n, 4096).astype(np.float64)
    X = X0
    for _ in range(K):
        X = ora.mix(W, X)
    c = W[0]
    omega = np.exp(2j * np.pi / n)
    F = np.array([[omega ** (-m * i) for i in range(n)] for m in range(n)])
    lam = np.array([sum(c[k] * omega ** (m * k) for k in range(n)) for m in range(n)])
    assert np.allclose(sorted(lam.real), [-1 / 3, 1 / 3, 1 / 3, 1.0])
    closed = (np.linalg.inv(F) @ np.diag(lam ** K) @ F @ X0).real
    assert np.allclose(X, closed, atol=1e-12)
    assert np.abs(X - X0.mean(axis=0)).max() < 2 * 3.0 ** -20 * np.abs(X0).max() * n


# ---------------------------------------------------------- local views -> W ---
def _views_from_W(W, style):
    n = W.shape[0]
    views = []
    for i in range(n):
        v = {"self_weight": W[i, i], "src_weights": None, "dst_weights": None}
        srcs = [j for j in range(n) if j != i and W[i, j] != 0]
        dsts = [j for j in range(n) if j != i and W[j, i] != 0]
        if style == "pull":
            v["src_weights"] = {j: W[i, j] for j in srcs}
        elif style == "push":
            v["dst_weights"] = {j: W[j, i] for j in dsts}
        elif style == "pushpull":
            v["src_weights"] = {j: 0.5 for j in srcs}
            v["dst_weights"] = {j: 2.0 * W[j, i] for j in dsts}
        views.append(v)
    return views


@pytest.mark.parametrize("style", ["pull", "push", "pushpull"])
def test_assemble_push_pull_equivalence(style):
    # Eq. 9-11: push (r=1, s=w), pull (r=w, s=1) and push-pull
    # (r*s = w) all realise the same W.
    g = golden("fig2_neighbor_sets.json")
    rng = np.random.default_rng(3)
    Wmask = _edges_to_W(g["n"], g["edges_1indexed"], one_indexed=True)
    W = Wmask * rng.uniform(0.1, 1.0, Wmask.shape)
    Wa = ora.assemble(_views_from_W(W, style))
    assert np.allclose(Wa, W, atol=1e-15)


def test_one_peer_views_match_schedule():
    # one-peer exp2 in pull form (src {i-2^t: 1/2}) and push form (dst {i+2^t: 1/2})
    n = 8
    for k in range(5):
        pull, push = [], []
        for i in range(n):
            s, d = ora.one_peer_exp2_peers(n, k, i)
            pull.append({"self_weight": 0.5, "src_weights": {s: 0.5}, "dst_weights": None})
            push.append({"self_weight": 0.5, "src_weights": None, "dst_weights": {d: 0.5}})
        assert np.array_equal(ora.assemble(pull), ora.one_peer_exp2(n, k))
        assert np.array_equal(ora.assemble(push), ora.one_peer_exp2(n, k))


def test_topology_check_mismatch():
    # "user fills in dst_weights in process i to push information to
    # process j, but does not provide src_weights in process j ... hangs".
    views = [{"self_weight": 0.5, "src_weights": None, "dst_weights": {1: 0.5}},
             {"self_weight": 1.0, "src_weights": {}, "dst_weights": {}}]
    with pytest.raises(ValueError):
        ora.assemble(views, check=True)
    W = ora.assemble(views, check=False)         # unchecked: receiver ignores the push
    assert W[1, 0] == 0.0
    # receiver lists a source that declares destinations but not the receiver
    views = [{"self_weight": 1.0, "src_weights": None, "dst_weights": {}},
             {"self_weight": 0.5, "src_weights": {0: 0.5}, "dst_weights": {}}]
    with pytest.raises(ValueError):
        ora.assemble(views, check=True)


# ---------------------------------------------------------------------- ATC ---
def test_atc_hand_example():
    # Eq. 4-5: x_half = x - lr*g = [0.5, 3.5], uniform W -> 2.0 for both
    W = np.full((2, 2), 0.5)
    Y = ora.atc(W, np.array([[1.0], [3.0]]), np.array([[1.0], [-1.0]]), 0.5)
    assert np.array_equal(Y, np.array([[2.0], [2.0]]))


def test_atc_wire_cast_points():
    # reading R18: self term from fp32 x_half, neighbour terms from the wire copy
    W = np.full((2, 2), 0.5)
    x = np.array([[1.0 + 2.0 ** -10], [0.0]])
    Y = ora.atc(W, x, np.zeros_like(x), 0.0, wire_bf16=True)
    assert Y[0, 0] == 0.5 + 2.0 ** -11            # own value unrounded
    assert Y[1, 0] == 0.5                         # bf16(1 + 2^-10) = 1.0 (RNE)
    Y32 = ora.atc(W, x, np.zeros_like(x), 0.0, wire_bf16=False)
    assert Y32[1, 0] == 0.5 + 2.0 ** -11


def test_atc_special_cases():
    n, cnt = 8, 500
    X = synthetic.agents_x0(n, cnt).astype(np.float64)
    G = synthetic.agents_grad(n, cnt, 0).astype(np.float64)
    W = ora.exp2(n)
    # lr = 0 -> pure averaging (Eq. 5 with the gradient ignored); X is fp32 so exact
    assert np.array_equal(ora.atc(W, X, G, 0.0), ora.mix(W, X))
    # n = 1 -> plain SGD, x - lr*g rounded once to fp32
    Y1 = ora.atc(np.eye(1), X[:1], G[:1], 0.1)
    ref = (X[:1] - np.float64(np.float32(0.1)) * G[:1]).astype(np.float32).astype(np.float64)
    assert np.array_equal(Y1, ref)
    # AWC with lr = 0 is also pure averaging (Eq. 16)
    assert np.array_equal(ora.awc(W, X, G, 0.0), ora.mix(W, X))


def test_atc_centralized_gd_equivalence():
    # S:532 / Eq. 13-14: identical data and iterates on every agent and a
    # doubly stochastic W reduce DGD to centralised gradient descent.
    n, m, d = 4, 30, 6
    rng = np.random.default_rng(5)
    A = rng.standard_normal((m, d)) / np.sqrt(m)
    b = rng.standard_normal(m)
    x = np.zeros(d)
    X = np.zeros((n, d))
    W = ora.ring(n)
    lr = 0.2
    for _ in range(25):
        g = ora.lsq_grad(A, b, X[0])
        assert np.allclose(g, A.T @ (A @ X[0] - b), atol=1e-13)
        X = ora.atc(W, X, np.tile(g, (n, 1)), lr)
        x = x - np.float32(lr) * (A.T @ (A @ x - b))
    assert np.allclose(X, np.tile(x, (n, 1)), rtol=1e-5, atol=1e-6)


def test_lsq_solve_matches_normal_equations():
    n, m, d = 3, 40, 12
    rng = np.random.default_rng(7)
    A = rng.standard_normal((n, m, d)) / np.sqrt(m)
    b = rng.standard_normal((n, m))
    x, it = ora.lsq_solve(A, b)
    ref, *_ = np.linalg.lstsq(A.reshape(n * m, d), b.reshape(n * m), rcond=None)
    assert np.allclose(x, ref, atol=1e-10)


# ------------------------------------------------------------- hierarchical ---
def test_hier_spec_example():
    g = golden("hier_2x2_example.json")
    X = np.array(g["inputs"]).reshape(4, 1)
    Y = ora.hier(np.array(g["machine_W"]), g["local_size"], X)
    assert np.array_equal(Y.ravel(), np.array(g["expected"]))


def test_hier_kronecker_and_degenerate():
    # (W_M kron J_L/L) X; one machine -> plain intra-machine average
    for nm, L in ((4, 2), (2, 4), (1, 8), (8, 1)):
        WM = ora.exp2(nm)
        X = synthetic.agents_x0(nm * L, 50).astype(np.float64)
        K = np.kron(WM, np.full((L, L), 1.0 / L))
        assert np.allclose(ora.hier(WM, L, X), K @ X, atol=1e-14)
    X = synthetic.agents_x0(8, 20).astype(np.float64)
    assert np.allclose(ora.hier(np.eye(1), 8, X), np.tile(X.mean(axis=0), (8, 1)), atol=1e-15)
    # hierarchical != flat neighbor_allreduce
    X = synthetic.agents_x0(8, 20).astype(np.float64)
    assert not np.allclose(ora.hier(ora.exp2(4), 2, X), ora.mix(ora.exp2(8), X))


# -------------------------------------------------------------------- casts ---
def test_bf16_rne_matches_torch():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(11)
    vals = np.concatenate([
        rng.standard_normal(2000).astype(np.float32),
        synthetic.uniform(1, 2000),
        # exact ties: low 16 bits 0x8000, both parities of the kept lsb
        (np.array([0x3F808000, 0x3F818000, 0xBF808000, 0x40490000 | 0x8000], np.uint32)).view(np.float32),
        np.array([0.0, -0.0, 1e-40, 3.4e38, np.inf, -np.inf], np.float32),
    ])
    ours = ora.bf16_rne(vals)
    ref = torch.from_numpy(vals).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)


def test_synthetic_generator_properties():
    u = synthetic.uniform(1000, 100000)
    assert u.dtype == np.float32 and u.min() >= -1.0 and u.max() < 1.0
    assert abs(u.mean()) < 0.01
    # exactly representable: multiples of 2^-23
    assert np.array_equal(np.round(u.astype(np.float64) * 2 ** 23), u.astype(np.float64) * 2 ** 23)
    # offset addressing is a pure counter
    assert np.array_equal(synthetic.uniform(5, 10, offset=90), synthetic.uniform(5, 100)[90:])


# ------------------------------------------------------------------ windows ---
def test_window_scalar_examples():
    g = golden("spec_scalar_examples.json")
    W = np.array([[1.0, 1.0, 1.0], [1.0, 1.0, 0.0], [1.0, 0.0, 1.0]])   # 1 <- 0, 2 <- 0 ... 0 <- {1,2}
    X0 = np.zeros((3, 1))
    X0[0, 0] = g["collect_local"]
    X0[1, 0] = g["collect_buffers"][0]
    X0[2, 0] = g["collect_buffers"][1]
    win = ora.Window(W, X0, zero_init=True)
    win.put(1, 0.0, {0: 1.0})
    win.put(2, 0.0, {0: 1.0})
    win.collect(0)
    assert win.x()[0, 0] == g["collect_expected"]
    # additive contract: two accumulates before the collect
    W2 = np.array([[1.0, 1.0], [1.0, 1.0]])
    win = ora.Window(W2, np.array([[0.0], [1.0]]), zero_init=True)
    win.accumulate(1, 1.0, {0: g["accumulate_twice"][0]})
    win.accumulate(1, 1.0, {0: g["accumulate_twice"][1]})
    win.collect(0)
    assert win.x()[0, 0] == g["accumulate_expected"]
    assert win.counters(0, 1) == (2, 2)


def test_window_backpressure_to_outbox():
    # a third accumulate before any collect cannot take a half: it waits in the
    # sender's outbox and is delivered later without loss (P:585 invariant)
    W2 = np.array([[1.0, 1.0], [1.0, 1.0]])
    win = ora.Window(W2, np.array([[0.0], [1.0]]), zero_init=True)
    m0 = win.mass(0)
    for k in range(5):
        win.accumulate(1, 1.0, {0: 1.0})      # s = 1 with self 1: each call adds 1 unit
        assert win.mass(0) == m0 + (k + 1)
    assert win.counters(0, 1) == (2, 0)
    win.collect(0)
    assert win.x()[0, 0] == 2.0
    win.accumulate(1, 1.0, {0: 0.0})          # flushes the outbox (3 more units)
    win.collect(0)
    assert win.x()[0, 0] == 5.0


def test_window_sync_pushsum_equals_mix():
    # synchronous schedule (all accumulate, then all collect) = one product
    # with the column-stochastic push matrix of Listing 3
    gold = golden("fig2_neighbor_sets.json")
    n = gold["n"]
    Wst = _edges_to_W(n, gold["edges_1indexed"], one_indexed=True)
    Wps = np.zeros((n, n))
    for i in range(n):
        outs = ora.out_neighbors(Wst, i)
        w = 1.0 / (len(outs) + 1)
        Wps[i, i] = w
        for j in outs:
            Wps[j, i] = w
    assert ora.classify(Wps) in ("push", "standard")
    X = np.concatenate([synthetic.agents_x0(n, 6).astype(np.float64), np.ones((n, 1))], axis=1)
    win = ora.Window(Wst, X, zero_init=True)
    ref = X
    for _ in range(4):
        for i in range(n):
            outs = ora.out_neighbors(Wst, i)
            w = 1.0 / (len(outs) + 1)
            win.accumulate(i, w, {j: w for j in outs})
        for i in range(n):
            win.collect(i)
        ref = ora.mix(Wps, ref)
    assert np.allclose(win.x(), ref, atol=1e-14)


def test_window_async_pushsum_invariants():
    # P:551-557 push-sum with random delays + P:585 mass invariant: total mass
    # (x + outboxes + unconsumed halves) is constant; y = x/p -> mean(x0).
    gold = golden("fig2_neighbor_sets.json")
    n = gold["n"]
    Wst = _edges_to_W(n, gold["edges_1indexed"], one_indexed=True)
    cnt = 4
    X = np.concatenate([synthetic.agents_x0(n, cnt - 1).astype(np.float64), np.ones((n, 1))], axis=1)
    target = X[:, :-1].mean(axis=0)
    win = ora.Window(Wst, X, zero_init=True)
    m0 = [win.mass(e) for e in range(cnt)]
    rng = np.random.default_rng(2024)
    for step in range(20000):
        i = int(rng.integers(n))
        if rng.random() < 0.5:
            outs = ora.out_neighbors(Wst, i)
            w = 1.0 / (len(outs) + 1)
            win.accumulate(i, w, {j: w for j in outs})
        else:
            win.collect(i)
        if step % 997 == 0:
            for e in range(cnt):
                assert abs(win.mass(e) - m0[e]) < 1e-12 * n
    Xf = win.x()
    y = Xf[:, :-1] / Xf[:, -1:]
    assert np.abs(y - target).max() < 1e-9
    assert abs(win.mass(cnt - 1) - n) < 1e-12


# ------------------------------------------- Exact-Diffusion (appendix ed-1..ed-3) ---
def _lsq_problem(n=4, m=12, d=5, seed=11):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, m, d)) / np.sqrt(m)
    b = rng.standard_normal((n, m))
    # global minimiser of sum_i ||A_i x - b_i||^2 / 2 by a library solver (independent of the oracle)
    xs = np.linalg.lstsq(A.reshape(n * m, d), b.reshape(n * m), rcond=None)[0]
    return A, b, xs


def test_exact_diffusion_converges_to_exact_minimiser():
    # The appendix's claim: ED "can correct the bias suffered by
    # decentralized gradient descent" -- with a constant step it reaches the exact
    # minimiser x*, while ATC-DGD stops at an O(gamma) distance.  Ring topology (Listing ED).
    n = 4
    A, b, xs = _lsq_problem(n)
    W = ora.ring(n)
    lr = 0.3
    grad = lambda X: np.einsum("imd,im->id", A, np.einsum("imd,id->im", A, X) - b)
    X = np.zeros((n, A.shape[2]))
    psi = X.copy()                 # psi^(-1) = x^(0): the first ED step is an ATC step
    Xa = X.copy()
    for _ in range(3000):
        X, psi = ora.exact_diffusion(W, X, grad(X), psi, lr)
        Xa = ora.atc(W, Xa, grad(Xa), lr)
    err_ed = np.abs(X - xs[None, :]).max()
    err_atc = np.abs(Xa - xs[None, :]).max()
    assert err_ed < 2e-6, err_ed          # fp32 state: exact up to single precision
    assert err_atc > 1e3 * err_ed, (err_atc, err_ed)


def test_exact_diffusion_special_cases():
    rng = np.random.default_rng(3)
    n, c, lr = 3, 64, 0.25
    X = rng.uniform(-1, 1, (n, c)).astype(np.float32).astype(np.float64)
    G = rng.uniform(-1, 1, (n, c)).astype(np.float32).astype(np.float64)
    P = rng.uniform(-1, 1, (n, c)).astype(np.float32).astype(np.float64)
    # W = I: x+ = phi = (x - lr g) + x - psi_prev, psi = x - lr g  (ed-1, ed-2 written out)
    Y, Pout = ora.exact_diffusion(np.eye(n), X, G, P, lr)
    psi = X - np.float32(lr) * G
    assert np.allclose(Pout, psi, rtol=0, atol=1e-7)
    assert np.allclose(Y, psi + X - P, rtol=0, atol=2e-7)
    # psi_prev = x: phi = psi, i.e. the step is exactly the ATC step (Eq. 17)
    W = ora.exp2(n)
    Y1, _ = ora.exact_diffusion(W, X, G, X, lr)
    assert np.allclose(Y1, ora.atc(W, X, G, lr), rtol=0, atol=1e-12)
    # doubly stochastic W preserves the sum over agents of phi (ed-3 + P:231-234)
    Y2, _ = ora.exact_diffusion(W, X, G, P, lr)
    phi = psi + X - P
    assert np.allclose(Y2.sum(axis=0), phi.sum(axis=0), rtol=0, atol=1e-6)


# ------------------------------- push-sum gradient tracking (appendix listing) ---
def _column_stochastic_directed(n, seed=2):
    # directed, strongly connected (ring i -> i+1 plus random extra edges), push weights
    # 1 / (out-degree + 1) on every out-edge and on the self loop: column-stochastic only
    rng = np.random.default_rng(seed)
    A = np.eye(n, dtype=bool)
    for i in range(n):
        A[(i + 1) % n, i] = True
        for j in rng.choice(n, 2, replace=False):
            A[j, i] = True
    W = A / A.sum(axis=0, keepdims=True)
    return W


def test_gradient_tracking_invariants_and_convergence():
    n, m, d = 5, 10, 4
    A, b, xs = _lsq_problem(n, m, d, seed=8)
    W = _column_stochastic_directed(n)
    assert np.allclose(W.sum(axis=0), 1.0) and not np.allclose(W.sum(axis=1), 1.0)
    grad = lambda X: np.einsum("imd,im->id", A, np.einsum("imd,id->im", A, X) - b)
    U = np.zeros((n, d)); V = np.ones((n, 1))
    G = grad(U / V); Y = G.copy()          # y^(0) = g^(0)
    lr = 0.05
    for _ in range(3000):
        X, U, V, Y, G = ora.gradient_tracking_step(W, U, V, Y, G, grad, lr)
        # column-stochastic W: sum_i v_i = n, and y tracks the sum of the gradients
        assert abs(V.sum() - n) < 1e-9
        assert np.allclose(Y.sum(axis=0), G.sum(axis=0), rtol=0, atol=1e-9)
    assert np.abs(X - xs[None, :]).max() < 1e-8      # exact convergence on a directed graph
    assert np.abs(V - 1).max() > 1e-2                 # and the push-sum weights really matter


# ------------------------------------------- hand examples with a nonzero step ---
def test_awc_hand_example_nonzero_lr():
    # Eq. 16: the gradient term with gamma != 0, checked by hand
    g = golden("awc_hier_hand_examples.json")["awc"]
    W = np.full((2, 2), 0.5)
    Y = ora.awc(W, np.array(g["x"])[:, None], np.array(g["g"])[:, None], g["lr"])
    assert np.array_equal(Y[:, 0], np.array(g["expected"]))


def test_hier_atc_awc_hand_examples_nonzero_lr():
    # caption P:869 H-ATC / H-AWC on 2 machines x 2 agents, hand-computed values
    g = golden("awc_hier_hand_examples.json")["hier"]
    X = np.array(g["x"])[:, None]
    G = np.array(g["g"])[:, None]
    I2, U2 = np.eye(2), np.full((2, 2), 0.5)
    assert np.array_equal(ora.hier_atc(I2, 2, X, G, g["lr"])[:, 0], g["atc_identity"])
    assert np.array_equal(ora.hier_atc(U2, 2, X, G, g["lr"])[:, 0], g["atc_uniform"])
    assert np.array_equal(ora.hier_awc(I2, 2, X, G, g["lr"])[:, 0], g["awc_identity"])
    assert np.array_equal(ora.hier_awc(U2, 2, X, G, g["lr"])[:, 0], g["awc_uniform"])


# --------------------------------------------------------- win_update pins ---
@pytest.mark.parametrize("model", ["event", "paper"])
def test_win_update_spec_example_and_idempotent(model):
    # S:454 ring(3) example: local 0, in-neighbours put 3 and 9,
    # uniform 1/3 -> 4; a second call with no traffic in between returns the same
    g = golden("spec_win_update_example.json")
    n = g["n"]
    W = ora.ring(n)
    X0 = np.array([[g["local"]], [g["puts"]["1"]], [g["puts"]["2"]]])
    Win = ora.Window if model == "event" else ora.WindowPaper
    win = Win(W, X0, zero_init=True)
    win.put(1, 1.0, {0: 1.0})
    win.put(2, 1.0, {0: 1.0})
    u = 1.0 / (len(ora.in_neighbors(W, 0)) + 1)
    out1 = win.update(0, u, {1: u, 2: u})
    out2 = win.update(0, u, {1: u, 2: u})
    assert abs(out1[0] - g["expected"]) < 1e-15
    assert np.array_equal(out1, out2)
    assert win.x()[0, 0] == g["local"]            # update does not touch x (no collect)
    # zero-initialised buffers before any traffic contribute nothing
    X1 = np.full((n, 1), g["zero_init_local"])
    win = Win(W, X1, zero_init=True)
    assert abs(win.update(0, u, {1: u, 2: u})[0] - g["zero_init_expected"]) < 1e-15
    # not zero-initialised: buffers hold the local tensor, uniform average returns x
    win = Win(W, X1, zero_init=False)
    assert abs(win.update(0, u, {1: u, 2: u})[0] - g["zero_init_local"]) < 1e-14


def test_win_update_weights_select_sources():
    # P:420 win_update(name, self_weight, src_weights): explicit weights, one source at 0
    W = ora.ring(3)
    X0 = np.array([[1.0], [2.0], [5.0]])
    for Win in (ora.Window, ora.WindowPaper):
        win = Win(W, X0, zero_init=True)
        win.put(1, 1.0, {0: 1.0})
        win.put(2, 1.0, {0: 1.0})
        assert win.update(0, 0.25, {1: 0.75, 2: 0.0})[0] == 0.25 * 1.0 + 0.75 * 2.0


# ------------------------ paper-semantics window vs the double-buffered model ---
def _fig2_W():
    gold = golden("fig2_neighbor_sets.json")
    return gold["n"], _edges_to_W(gold["n"], gold["edges_1indexed"], one_indexed=True)


def test_paper_window_accumulate_collect_by_hand():
    # P:402-403 accumulate adds into the neighbour's buffer; P:585 collect sums, then zeroes
    W2 = np.array([[1.0, 1.0], [1.0, 1.0]])
    win = ora.WindowPaper(W2, np.array([[1.0], [2.0]]), zero_init=True)
    win.accumulate(1, 0.5, {0: 0.5})      # buffer_0[1] = 1, x_1 = 1
    win.accumulate(1, 1.0, {0: 2.0})      # buffer_0[1] = 1 + 2 = 3
    assert win.update(0, 0.0, {1: 1.0})[0] == 3.0
    win.collect(0)
    assert win.x()[:, 0].tolist() == [4.0, 1.0]
    win.collect(0)                        # buffers were zeroed: nothing more arrives
    assert win.x()[:, 0].tolist() == [4.0, 1.0]
    win.put(1, 1.0, {0: 7.0})             # put overwrites
    win.put(1, 1.0, {0: 1.0})
    assert win.update(0, 0.0, {1: 1.0})[0] == 1.0


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_event_model_equals_paper_window_without_backlog(seed):
    # Whenever no payload has to wait in a sender's outbox (the destination half is
    # free at every accumulate), the double-buffered protocol model gives exactly the
    # paper's window: x after every event equal (push-sum, Listing 3 weights)
    n, Wst = _fig2_W()
    cnt = 3
    X = np.concatenate([synthetic.agents_x0(n, cnt - 1).astype(np.float64), np.ones((n, 1))], axis=1)
    ev, pw = ora.Window(Wst, X, zero_init=True), ora.WindowPaper(Wst, X, zero_init=True)
    rng = np.random.default_rng(seed)
    n_acc = 0
    for _ in range(3000):
        i = int(rng.integers(n))
        outs = ora.out_neighbors(Wst, i)
        free = all(ev.counters(j, i)[1] >= ev.counters(j, i)[0] - 1 for j in outs)
        if rng.random() < 0.5 and free:
            w = 1.0 / (len(outs) + 1)
            ev.accumulate(i, w, {j: w for j in outs})
            pw.accumulate(i, w, {j: w for j in outs})
            n_acc += 1
        else:
            ev.collect(i)
            pw.collect(i)
        assert np.allclose(ev.x(), pw.x(), rtol=0, atol=1e-13)
    assert n_acc > 500


def test_event_model_equals_paper_window_put_update():
    # put + win_update: the latest payload of each slot is the
    # paper's buffer value, whenever the half was free at the put
    n, Wst = _fig2_W()
    X = synthetic.agents_x0(n, 4).astype(np.float64)
    ev, pw = ora.Window(Wst, X, zero_init=False), ora.WindowPaper(Wst, X, zero_init=False)
    rng = np.random.default_rng(9)
    for step in range(400):
        i = int(rng.integers(n))
        if rng.random() < 0.5:
            outs = ora.out_neighbors(Wst, i)
            s = {j: float(rng.uniform(-1, 1)) for j in outs if rng.random() < 0.7}
            if all(ev.counters(j, i)[1] >= ev.counters(j, i)[0] - 1 for j in s):
                sw = float(rng.uniform(0.5, 1.5))
                ev.put(i, sw, s)
                pw.put(i, sw, s)
        else:
            ins = ora.in_neighbors(Wst, i)
            r = {j: float(rng.uniform(-1, 1)) for j in ins}
            sw = float(rng.uniform(-1, 1))
            assert np.allclose(ev.update(i, sw, r), pw.update(i, sw, r), rtol=0, atol=1e-13)
        assert np.allclose(ev.x(), pw.x(), rtol=0, atol=1e-13)


def test_event_model_with_backlog_conserves_the_paper_mass():
    # with backlog a payload reaches its destination later than in the paper's window
    # (it waits in the outbox), so the trajectories differ -- asynchronous results are
    # interleaving-dependent (R19) -- but after a drain (every payload delivered and
    # collected) both models hold the same total mass sum_i x_i = sum_i x_i^0
    n, Wst = _fig2_W()
    X = np.concatenate([synthetic.agents_x0(n, 2).astype(np.float64), np.ones((n, 1))], axis=1)
    ev, pw = ora.Window(Wst, X, zero_init=True), ora.WindowPaper(Wst, X, zero_init=True)
    rng = np.random.default_rng(3)
    for _ in range(2000):
        i = int(rng.integers(n))
        outs = ora.out_neighbors(Wst, i)
        if rng.random() < 0.7:   # producers run ahead of the consumers: outboxes fill
            w = 1.0 / (len(outs) + 1)
            ev.accumulate(i, w, {j: w for j in outs})
            pw.accumulate(i, w, {j: w for j in outs})
        else:
            ev.collect(i)
            pw.collect(i)
    # drain: zero-weight accumulates flush the outboxes (self 1, s 0 adds nothing new)
    for _ in range(4):
        for i in range(n):
            outs = ora.out_neighbors(Wst, i)
            ev.accumulate(i, 1.0, {j: 0.0 for j in outs})
            pw.accumulate(i, 1.0, {j: 0.0 for j in outs})
        for i in range(n):
            ev.collect(i)
            pw.collect(i)
    assert np.allclose(ev.x().sum(axis=0), X.sum(axis=0), rtol=0, atol=1e-12)
    assert np.allclose(pw.x().sum(axis=0), X.sum(axis=0), rtol=0, atol=1e-12)
    assert np.abs(ev.x() - pw.x()).max() > 1e-6      # the interleavings really differed


# -------------------------------------------------- ATC fixed point x_inf ---
def _atc_fixed_point_linear_solve(W, A, b, lr):
    # the fixed point written as one linear system (a library solve, independent of
    # the oracle's iteration): vec X = (W kron I)(vec X - lr (H vec X - c))
    n, m, d = A.shape
    H = np.zeros((n * d, n * d))
    c = np.zeros(n * d)
    for i in range(n):
        H[i * d:(i + 1) * d, i * d:(i + 1) * d] = A[i].T @ A[i]
        c[i * d:(i + 1) * d] = A[i].T @ b[i]
    Wk = np.kron(W, np.eye(d))
    M = np.eye(n * d) - Wk @ (np.eye(n * d) - lr * H)
    return np.linalg.solve(M, lr * Wk @ c).reshape(n, d)


@pytest.mark.parametrize("topo", ["ring", "exp2", "one_peer0"])
def test_atc_fixed_point_matches_linear_solve(topo):
    # x_inf, the unique fixed point of X = W(X - gamma(HX - c))
    n = 4
    A, b, xs = _lsq_problem(n, m=12, d=5, seed=11)
    W = {"ring": ora.ring(n), "exp2": ora.exp2(n), "one_peer0": ora.one_peer_exp2(n, 0)}[topo]
    lr = 0.3
    X, it = ora.atc_fixed_point(W, A, b, lr)
    ref = _atc_fixed_point_linear_solve(W, A, b, lr)
    assert np.abs(X - ref).max() < 1e-12 * np.abs(ref).max(), (np.abs(X - ref).max(), it)
    # uniqueness: any start reaches the same point (linear contraction)
    X2, _ = ora.atc_fixed_point(W, A, b, lr, X0=np.random.default_rng(1).standard_normal((n, 5)) * 10)
    assert np.abs(X2 - X).max() < 1e-12 * np.abs(ref).max()


def test_atc_fixed_point_special_cases():
    n = 4
    A, b, xs = _lsq_problem(n, m=12, d=5, seed=11)
    # full averaging (W = J/n): every row is the global minimiser x* (the mean gradient vanishes)
    X, _ = ora.atc_fixed_point(ora.full(n), A, b, 0.3)
    assert np.abs(X - xs[None, :]).max() < 1e-12
    # one agent: plain gradient descent's fixed point is its own least-squares solution
    x1 = np.linalg.lstsq(A[0], b[0], rcond=None)[0]
    X1, _ = ora.atc_fixed_point(np.eye(1), A[:1], b[:1], 0.3)
    assert np.abs(X1[0] - x1).max() < 1e-12
    # ring with distinct data: ATC stops at an O(gamma) bias from x* (the bias
    # Exact-Diffusion corrects, appendix); halving gamma roughly halves it
    e1 = np.abs(ora.atc_fixed_point(ora.ring(n), A, b, 0.2)[0] - xs).max()
    e2 = np.abs(ora.atc_fixed_point(ora.ring(n), A, b, 0.1)[0] - xs).max()
    assert e1 > 1e-4 and 1.6 < e1 / e2 < 2.4, (e1, e2)


# ------------------------------------------------ gradient-tracking halves ---
def test_gradient_tracking_halves_by_hand_and_vector_v():
    # lines 1002-1006 on 2 agents, W = [[1/2,1/2],[1/2,1/2]], hand values
    W = np.full((2, 2), 0.5)
    U = np.array([[2.0], [4.0]]); V = np.array([[1.0], [3.0]]); Y = np.array([[2.0], [0.0]])
    Un, Vn, Xn = ora.gt_uv(W, U, V, Y, 0.5)      # u - lr y = (1, 4) -> 2.5 ; v -> 2
    assert Un[:, 0].tolist() == [2.5, 2.5] and Vn[:, 0].tolist() == [2.0, 2.0] and Xn[:, 0].tolist() == [1.25, 1.25]
    Yn = ora.gt_y(W, Y, np.array([[1.0], [1.0]]), np.array([[0.0], [3.0]]))   # y + g - g' = (3, -2) -> 0.5
    assert Yn[:, 0].tolist() == [0.5, 0.5]
    # the paper's vector v with equal entries == one weight per agent
    n, d = 5, 4
    Wd = _column_stochastic_directed(n)
    rng = np.random.default_rng(4)
    U, Y = rng.standard_normal((n, d)), rng.standard_normal((n, d))
    v1 = rng.uniform(0.5, 2, (n, 1))
    a = ora.gt_uv(Wd, U, v1, Y, 0.1)
    b_ = ora.gt_uv(Wd, U, np.tile(v1, (1, d)), Y, 0.1)
    assert np.array_equal(a[0], b_[0]) and np.array_equal(a[2], b_[2]) and np.array_equal(np.tile(a[1], (1, d)), b_[1])


def test_win_adapt_then_accumulate_by_hand():
    # gradient-in-window (SGP-style): x_1 = 2 - 0.5 * 2 = 1, then accumulate s = 1/2, self 1/2
    W2 = np.array([[1.0, 1.0], [1.0, 1.0]])
    win = ora.Window(W2, np.array([[0.0], [2.0]]), zero_init=True)
    win.adapt(1, np.array([2.0]), 0.5)
    win.accumulate(1, 0.5, {0: 0.5})
    win.collect(0)
    assert win.x()[:, 0].tolist() == [0.5, 0.5]
    # mass after the step: the step removes lr * g from the total, nothing else does
    assert win.mass(0) == 1.0


def test_comm_cost_table1_by_hand():
    # Table 1 evaluated by hand for n = 8, M = 100 MB,
    # B = 1e9 B/s, L = 1e-5 s; and P:242 "O(1) latency and O(1) transmission time,
    # independent of n" for partial averaging, O(n) for every global primitive
    M, B, L = 1e8, 1e9, 1e-5
    assert ora.comm_cost("parameter_server", 8, M, B, L) == 8 * 0.1 + 8e-5
    assert ora.comm_cost("ring_allreduce", 8, M, B, L) == 0.2 + 16e-5
    assert ora.comm_cost("byte_ps", 8, M, B, L) == 0.1 + 8e-5
    assert ora.comm_cost("partial_averaging", 8, M, B, L) == 0.1 + 1e-5
    for prim in ("parameter_server", "ring_allreduce", "byte_ps"):
        assert ora.comm_cost(prim, 64, M, B, L) > ora.comm_cost(prim, 8, M, B, L)
    assert ora.comm_cost("partial_averaging", 64, M, B, L) == ora.comm_cost("partial_averaging", 8, M, B, L)
