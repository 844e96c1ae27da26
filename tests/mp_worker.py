"""Multi-process parity worker (one process per GPU, launched by torchrun from
tests/test_multigpu.py).  Every process holds `BF_TEST_K` agents; neighbours
on other GPUs are read over NVLink through CUDA-IPC peer pointers.  Each rank
checks its own rows against the oracle run on the full stacked input."""
import os
import sys
import traceback

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("BF_TIMEOUT_MS", "8000")

import oracle as ora  # noqa: E402
import synthetic  # noqa: E402
import paper_2111_04287_b200 as bfp  # noqa: E402
from paper_2111_04287_b200 import BluefogError  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    rank = int(os.environ["RANK"])
    # BF_TEST_SHARE_GPUS=G: more processes than GPUs (process p on GPU p mod G, gloo bootstrap,
    # time-sliced contexts) -- the 8-process logic of the 8-GPU setting on a smaller box
    share = int(os.environ.get("BF_TEST_SHARE_GPUS", "0"))
    dev = local % share if share else local
    torch.cuda.set_device(dev)
    if share:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    k = int(os.environ.get("BF_TEST_K", "1"))
    ctx = bfp.Context(agents_per_proc=k, heap_bytes=1 << 29, device=dev)
    n, r0 = ctx.n, ctx.rank
    rows = slice(r0, r0 + k)
    failures = []

    def check(name, y, ref, W, X, tol, extra=None):
        b = (np.abs(W) @ np.abs(X))[rows]
        if extra is not None:
            b = b + extra[rows]
        err = np.abs(y - ref[rows])
        if (err > tol * b + 1e-30).any():
            failures.append(f"{name}: max rel {np.max(err / (b + 1e-30)):.3e}")

    def inputs(count, dtype=torch.float32, seed_off=0):
        X = np.stack([synthetic.uniform(synthetic.SEED_X0 + seed_off + r, count) for r in range(n)])
        xt = torch.from_numpy(X[rows].copy()).to(dtype).cuda()
        Xf = torch.from_numpy(X).to(dtype).float().numpy().astype(np.float64)
        return xt, Xf

    def np_(t):
        return t.float().cpu().numpy().astype(np.float64)

    # ---- static topologies --------------------------------------------------
    for topo in ("exp2", "ring", "full"):
        W = {"exp2": ora.exp2, "ring": ora.ring, "full": ora.full}[topo](n)
        ctx.set_topology(W)
        for dtype, tol in ((torch.float32, 1e-6), (torch.bfloat16, 1e-2)):
            for count in (1, 4097, 3 * 4096 + 5, 200003):
                x, X = inputs(count, dtype)
                y = ctx.neighbor_allreduce(x)
                torch.cuda.synchronize()
                check(f"static {topo} {dtype} {count}", np_(y), ora.mix(W, X), W, X, tol)

    # ---- around the small-message thresholds (tagged words <= 262144 elements, or <= 32768
    # when the heap is small; push above) ----
    ctx.set_topology(ora.exp2(n))
    We = ora.exp2(n)
    for count in (32767, 32768, 32769, 262143, 262144, 262145):
        for dtype, tol in ((torch.float32, 1e-6), (torch.bfloat16, 1e-2)):
            x, X = inputs(count, dtype, seed_off=11)
            y = ctx.neighbor_allreduce(x)
            torch.cuda.synchronize()
            check(f"threshold nar {dtype} {count}", np_(y), ora.mix(We, X), We, X, tol)
        x, X = inputs(count, seed_off=12)
        G = np.stack([synthetic.uniform(synthetic.grad_seed(2, r), count, scale=2.0 ** -7) for r in range(n)])
        g = torch.from_numpy(G[rows].copy()).cuda()
        ctx.atc_step(x, g, 0.1, wire=torch.bfloat16)
        torch.cuda.synchronize()
        check(f"threshold atc bf16 wire {count}", np_(x), ora.atc(We, X, G.astype(np.float64), 0.1, wire_bf16=True),
              We, X, 1e-2, np.abs(We) @ (0.1 * np.abs(G.astype(np.float64))))

    # ---- the push path with several progress batches per CTA (> 4 sub-items per CTA
    # at every K; bf16 at K = 4 has a lag of 3 sub-items, so its batches are shorter) ----
    for count, dtype, tol in ((1_300_001, torch.float32, 1e-6), (2_600_003, torch.bfloat16, 1e-2)):
        x, X = inputs(count, dtype, seed_off=13)
        for topo in ("exp2", "one_peer"):
            if topo == "exp2":
                ctx.set_topology(We)
                Wr = We
            else:
                ctx.set_dynamic_schedule("one_peer_exp2", 0)
                Wr = ora.one_peer_exp2(n, 0)
            y = ctx.neighbor_allreduce(x)
            torch.cuda.synchronize()
            ctx.set_dynamic_schedule("none")
            check(f"multi-batch nar {topo} {dtype} {count}", np_(y), ora.mix(Wr, X), Wr, X, tol)
        del x, y

    # ---- dynamic push / pull / push-pull ------------------------------------
    rng = np.random.default_rng(11)
    W = (rng.random((n, n)) < 0.6) * rng.uniform(0.1, 1.0, (n, n))
    np.fill_diagonal(W, 0.5)
    for style in ("pull", "push", "pushpull"):
        sw, srcw, dstw = [], [], []
        for i in range(r0, r0 + k):
            srcs = [j for j in range(n) if j != i and W[i, j] != 0]
            dsts = [j for j in range(n) if j != i and W[j, i] != 0]
            sw.append(W[i, i])
            srcw.append({j: W[i, j] for j in srcs} if style == "pull" else
                        ({j: 0.5 for j in srcs} if style == "pushpull" else None))
            dstw.append({j: W[j, i] for j in dsts} if style == "push" else
                        ({j: 2.0 * W[j, i] for j in dsts} if style == "pushpull" else None))
        x, X = inputs(50001)
        y = ctx.neighbor_allreduce(x, self_weight=sw, src_weights=srcw, dst_weights=dstw)
        torch.cuda.synchronize()
        check(f"dynamic {style}", np_(y), ora.mix(W, X), W, X, 1e-6)

    # ---- one-peer schedule (device round counter) ----------------------------
    ctx.set_dynamic_schedule("one_peer_exp2", 0)
    x, X = inputs(70001)
    for kk in range(4):
        x = ctx.neighbor_allreduce(x)
        torch.cuda.synchronize()
        Wk = ora.one_peer_exp2(n, kk)
        Y = ora.mix(Wk, X)
        check(f"schedule round {kk}", np_(x), Y, Wk, X, 1e-6)
        X = Y   # continue from the oracle state (rows of other ranks are not visible here)
        x = torch.from_numpy(X[rows].astype(np.float32)).cuda()
    # ---- inner-outer exp-2 schedule (R27): machines of 2 agents ----------------------
    if n % 2 == 0:
        ctx.set_machine_topology(ora.exp2(n // 2) if n > 2 else np.ones((1, 1)), 2)
        ctx.set_dynamic_schedule("inner_outer_exp2", 1)
        x, X = inputs(60013)
        for kk in range(1, 5):
            x = ctx.neighbor_allreduce(x)
            torch.cuda.synchronize()
            Wk = ora.inner_outer_exp2(n, 2, kk)
            Y = ora.mix(Wk, X)
            check(f"inner-outer round {kk}", np_(x), Y, Wk, X, 1e-6)
            X = Y
            x = torch.from_numpy(X[rows].astype(np.float32)).cuda()
        ctx.set_dynamic_schedule("one_peer_exp2", 4)
    # ---- fused ATC --------------------------------------------------------------
    for wire, tol in ((torch.float32, 1e-6), (torch.bfloat16, 1e-2)):
        x, X = inputs(123457)
        G = np.stack([synthetic.uniform(synthetic.grad_seed(1, r), 123457, scale=2.0 ** -7) for r in range(n)])
        g = torch.from_numpy(G[rows].copy()).cuda()
        kk = 4 if wire == torch.float32 else 5
        ctx.atc_step(x, g, 0.1, wire=wire)
        torch.cuda.synchronize()
        Wk = ora.one_peer_exp2(n, kk)
        check(f"atc {wire}", np_(x), ora.atc(Wk, X, G.astype(np.float64), 0.1, wire_bf16=wire == torch.bfloat16),
              Wk, X, tol, np.abs(Wk) @ (0.1 * np.abs(G.astype(np.float64))))
    ctx.set_dynamic_schedule("none")

    # Exact-Diffusion and gradient tracking need the fused kernels (K = 1, 2, 4 across
    # GPUs); other K take the chunked kernel and report BF_ERR_UNSUPPORTED for them
    fused = k in (1, 2, 4)
    if not fused:
        try:
            x, X = inputs(1001)
            ctx.exact_diffusion_step(x, x.clone(), x.clone(), 0.1)
            failures.append("ED accepted on the chunked kernel")
        except BluefogError as e:
            if e.name != "BF_ERR_UNSUPPORTED":
                failures.append(f"ED on the chunked kernel: {e.name}")

    if fused:
        # ---- Exact-Diffusion (appendix ed-1..ed-3), static exp-2 ------------------------
        We = ora.exp2(n)
        ctx.set_topology(We)
        x, X = inputs(50003)
        Ge = np.stack([synthetic.uniform(synthetic.grad_seed(3, r), 50003, scale=2.0 ** -7) for r in range(n)])
        Pe = np.stack([synthetic.uniform(synthetic.grad_seed(4, r), 50003) for r in range(n)])
        g = torch.from_numpy(Ge[rows].copy()).cuda()
        psi = torch.from_numpy(Pe[rows].copy()).cuda()
        ctx.exact_diffusion_step(x, g, psi, 0.1)
        torch.cuda.synchronize()
        ref, _ = ora.exact_diffusion(We, X, Ge.astype(np.float64), Pe.astype(np.float64), 0.1)
        check("exact diffusion", np_(x), ref, We, X, 1e-6,
              np.abs(We) @ (np.abs(X) + 0.1 * np.abs(Ge.astype(np.float64)) + np.abs(Pe.astype(np.float64))))

        # ---- push-sum gradient tracking (appendix): MODE 5 / MODE 4 ----
        Adj = np.eye(n, dtype=bool)
        rg = np.random.default_rng(31)
        for i in range(n):
            Adj[(i + 1) % n, i] = True
            for j in rg.choice(n, min(2, n), replace=False):
                Adj[j, i] = True
        Wg = Adj / Adj.sum(axis=0, keepdims=True)          # directed, column stochastic
        ctx.set_topology(Wg)
        cnt = 30011
        u, U = inputs(cnt, seed_off=3)
        y, Y = inputs(cnt, seed_off=4)
        Vf = np.linspace(0.5, 1.5, n)
        v = torch.from_numpy(Vf[rows].astype(np.float32)).cuda()
        xo = torch.empty_like(u)
        ctx.gt_uv_step(u, v, y, xo, 0.05)
        torch.cuda.synchronize()
        Ur, Vr, Xr = ora.gt_uv(Wg, U, Vf.astype(np.float32).astype(np.float64)[:, None], Y, 0.05)
        check("gt u", np_(u), Ur, Wg, np.abs(U) + 0.05 * np.abs(Y), 1e-6)
        if np.abs(v.cpu().numpy() - Vr[rows, 0]).max() > 1e-6 * np.abs(Vr).max():
            failures.append("gt v")
        if np.abs(np_(xo) - Xr[rows]).max() > 1e-5 * np.abs(Xr).max():
            failures.append("gt x = u / v")
        gn, Gn = inputs(cnt, seed_off=5)
        gp, Gp = inputs(cnt, seed_off=6)
        ctx.gt_y_step(y, gn, gp)
        torch.cuda.synchronize()
        check("gt y", np_(y), ora.gt_y(Wg, Y, Gn, Gp), Wg, np.abs(Y) + np.abs(Gn) + np.abs(Gp), 1e-6)

    # ---- C2 across GPUs: ATC-DSGD on least squares reaches the oracle's fixed point ----
    # (Eq. 12-13, Eq. 17) -- hundreds of consecutive small
    # exchanges (the tagged-word path), gradients of the local agents by torch bmm
    if fused:
        m2, d2 = 40, 24
        rs = np.random.default_rng(77)
        A2 = rs.standard_normal((n, m2, d2)) / np.sqrt(m2)
        b2 = np.einsum("imd,d->im", A2, rs.standard_normal(d2)) + 0.01 * rs.standard_normal((n, m2))
        W2 = ora.exp2(n)
        lam = max(np.linalg.eigvalsh(A2[i].T @ A2[i]).max() for i in range(n))
        lr2 = float(np.float32(1.0 / lam))
        xinf, _ = ora.atc_fixed_point(W2, A2, b2, lr2)
        H = np.zeros((n * d2, n * d2))
        for i in range(n):
            H[i * d2:(i + 1) * d2, i * d2:(i + 1) * d2] = A2[i].T @ A2[i]
        rho = np.abs(np.linalg.eigvals(np.kron(W2, np.eye(d2)) @ (np.eye(n * d2) - lr2 * H))).max()
        ctx.set_topology(W2)
        At2 = torch.from_numpy(A2[rows].copy()).cuda()
        bt2 = torch.from_numpy(b2[rows].copy()).cuda()
        xc = torch.zeros(k, d2, device="cuda")
        for _ in range(int(40 / (1 - rho)) + 200):
            gr = torch.bmm(At2.transpose(1, 2), (torch.bmm(At2, xc.double().unsqueeze(2)).squeeze(2) - bt2).unsqueeze(2))
            ctx.atc_step(xc, gr.squeeze(2).float().contiguous(), lr2)
        torch.cuda.synchronize()
        err = np.abs(np_(xc) - xinf[rows]).max() / np.abs(xinf).max()
        if err > 64 * 2.0 ** -24 / (1 - rho):
            failures.append(f"C2 fixed point: {err:.3e} (rho {rho:.3f})")

    # ---- hierarchical -------------------------------------------------------------
    for L in sorted({1, 2, n}):
        if n % L or n // L < 1:
            continue
        nm = n // L
        WM = ora.exp2(nm)
        ctx.set_machine_topology(WM, L)
        x, X = inputs(40000)
        y = ctx.hierarchical_neighbor_allreduce(x)
        torch.cuda.synchronize()
        check(f"hier L={L}", np_(y), ora.hier(WM, L, X), np.kron(WM, np.full((L, L), 1.0 / L)), X, 1e-6)
        xb, Xb = inputs(40000, torch.bfloat16)
        yb = ctx.hierarchical_neighbor_allreduce(xb)
        torch.cuda.synchronize()
        check(f"hier bf16 L={L}", np_(yb), ora.hier(WM, L, Xb), np.kron(WM, np.full((L, L), 1.0 / L)), Xb, 1e-2)
        Gh = np.stack([synthetic.uniform(synthetic.grad_seed(6, r), 40000, scale=2.0 ** -7) for r in range(n)])
        gh = torch.from_numpy(Gh[rows].copy()).cuda()
        Kh = np.kron(WM, np.full((L, L), 1.0 / L))
        ctx.hierarchical_atc_step(x, gh, 0.1)
        torch.cuda.synchronize()
        check(f"H-ATC L={L}", np_(x), ora.hier_atc(WM, L, X, Gh, 0.1), Kh, X, 1e-6,
              np.abs(Kh) @ (0.1 * np.abs(Gh.astype(np.float64))))
        x, X = inputs(40000)
        ctx.hierarchical_awc_step(x, gh, 0.1)
        torch.cuda.synchronize()
        check(f"H-AWC L={L}", np_(x), ora.hier_awc(WM, L, X, Gh, 0.1), Kh, X, 1e-6,
              0.1 * np.abs(Gh.astype(np.float64)))

    # ---- NVLS: machines spanning 2 processes, average in the switch (hier_nvls.cu) ----
    if ctx.nprocs % 2 == 0 and not share:   # multicast objects need one process per GPU
        L = 2 * k
        nm = n // L
        WM = ora.exp2(nm) if nm > 1 else np.ones((1, 1))
        ctx.set_machine_topology(WM, L)
        if ctx.enable_nvls(L, 60000):
            Kh = np.kron(WM, np.full((L, L), 1.0 / L))
            x, X = inputs(40003)
            y = ctx.hierarchical_neighbor_allreduce(x)
            torch.cuda.synchronize()
            check(f"nvls hier L={L}", np_(y), ora.hier(WM, L, X), Kh, X, 1e-6)
            Gh = np.stack([synthetic.uniform(synthetic.grad_seed(9, r), 40003, scale=2.0 ** -7) for r in range(n)])
            gh = torch.from_numpy(Gh[rows].copy()).cuda()
            xa = x.clone()
            ctx.hierarchical_atc_step(xa, gh, 0.1)
            torch.cuda.synchronize()
            check(f"nvls H-ATC L={L}", np_(xa), ora.hier_atc(WM, L, X, Gh, 0.1), Kh, X, 1e-6,
                  np.abs(Kh) @ (0.1 * np.abs(Gh.astype(np.float64))))
            xw = x.clone()
            ctx.hierarchical_awc_step(xw, gh, 0.1)
            torch.cuda.synchronize()
            check(f"nvls H-AWC L={L}", np_(xw), ora.hier_awc(WM, L, X, Gh, 0.1), Kh, X, 1e-6,
                  0.1 * np.abs(Gh.astype(np.float64)))
            ctx.disable_nvls()
            if rank == 0:
                print("NVLS path checked", flush=True)
        elif rank == 0:
            print("NVLS: no multicast support on this box", flush=True)

    # ---- neighbor_win_get on a symmetric-heap tensor (reads over NVLink) ------------
    Wst = ora.exp2(n)
    ctx.set_topology(Wst)
    Xg = np.stack([synthetic.uniform(synthetic.SEED_X0 + 50 + r, 7001) for r in range(n)]).astype(np.float32)
    xg = ctx.alloc((k, 7001))
    xg.copy_(torch.from_numpy(Xg[rows]))
    ctx.win_create(xg, "get", zero_init=True)
    torch.cuda.synchronize()
    dist.barrier()   # every owner's tensor is in place before anybody reads it
    ins = [[j for j in range(n) if j != i and Wst[i, j] != 0] for i in range(n)]
    ctx.win_get("get", src_weights=[{j: 0.5 for j in ins[r0 + a]} for a in range(k)])
    outg = torch.empty_like(xg)
    ctx.win_update("get", self_weight=[0.0] * k, src_weights=[{j: 1.0 for j in ins[r0 + a]} for a in range(k)],
                   out=outg)
    torch.cuda.synchronize()
    Wg = 0.5 * (Wst != 0)
    np.fill_diagonal(Wg, 0.0)
    check("win_get", np_(outg), ora.mix(Wg, Xg.astype(np.float64)), Wg, Xg.astype(np.float64), 1e-6)
    dist.barrier()
    ctx.win_free("get")

    # ---- windows: synchronous push-sum ------------------------------------------
    Wst = ora.exp2(n)
    ctx.set_topology(Wst)
    x, X = inputs(9001)
    ctx.win_create(x, "ps", zero_init=True, with_p=True)
    win = ora.Window(Wst, np.concatenate([X, np.ones((n, 1))], axis=1), zero_init=True)
    for _ in range(4):
        ctx.win_accumulate("ps")
        ctx.barrier()
        ctx.win_update_then_collect("ps")
        ctx.barrier()
        for i in range(n):
            outs = ora.out_neighbors(Wst, i)
            w = 1.0 / (len(outs) + 1)
            win.accumulate(i, w, {j: w for j in outs})
        for i in range(n):
            win.collect(i)
    torch.cuda.synchronize()
    ref = win.x()
    if np.abs(np_(x) - ref[rows, :-1]).max() > 1e-5:
        failures.append("window sync push-sum x")
    if np.abs(ctx.win_p("ps") - ref[rows, -1]).max() > 1e-12:
        failures.append("window sync push-sum p")

    # ---- windows: asynchronous push-sum (no inter-agent synchronisation) --------
    x2, X2 = inputs(20000, seed_off=7)
    ctx.win_create(x2, "async", zero_init=True, with_p=True)
    mass0 = X2.sum(axis=0)
    lr_ = np.random.default_rng(100 + rank)
    for _ in range(60):
        if lr_.random() < 0.5:
            ctx.win_accumulate("async", agent_mask=1 << int(lr_.integers(k)))
        else:
            ctx.win_update_then_collect("async", agent_mask=1 << int(lr_.integers(k)))
    for _ in range(3):   # quiesce: flush outboxes, collect everything
        ctx.barrier()
        ctx.win_accumulate("async", self_weight=[1.0] * k,
                           dst_weights=[{j: 0.0 for j in ora.out_neighbors(Wst, i)} for i in range(r0, r0 + k)])
        ctx.barrier()
        ctx.win_update_then_collect("async")
    ctx.barrier()
    torch.cuda.synchronize()
    tot = torch.tensor(np.concatenate([np_(x2).sum(axis=0), [ctx.win_p("async").sum()]]), device="cuda")
    dist.all_reduce(tot)
    tot = tot.cpu().numpy()
    if np.abs(tot[:-1] - mass0).max() > 1e-4 or abs(tot[-1] - n) > 1e-12:
        failures.append(f"async window mass {np.abs(tot[:-1] - mass0).max():.3e} p {tot[-1]}")
    ctx.win_free("async")
    ctx.win_free("ps")

    # ---- topology-check mismatch: an error, never a hang -------------------
    x, X = inputs(1000)
    got = None
    try:
        sw = [0.5] * k
        if r0 == 0:   # agent 0 pushes to agent n-1, which declares no sources
            dstw = [{n - 1: 0.5}] + [{}] * (k - 1)
        else:
            dstw = [{}] * k
        srcw = [None] * k if r0 == 0 else [{}] * k
        ctx.neighbor_allreduce(x, self_weight=sw, src_weights=srcw, dst_weights=dstw)
        torch.cuda.synchronize()
        ctx.poll_error()
    except BluefogError as e:
        got = e.name
    # the receiver detects the mismatch; it aborts every process, so after a
    # host barrier every rank reports the fault (the sender included)
    dist.barrier()
    if got is None:
        try:
            ctx.poll_error()
        except BluefogError as e:
            got = e.name
    if got not in ("BF_ERR_TOPOLOGY", "BF_ERR_TIMEOUT", "BF_ERR_STATE"):
        failures.append(f"mismatch not reported: {got}")

    dist.barrier()
    if failures:
        print(f"RANK {rank} FAIL: " + "; ".join(failures), flush=True)
    else:
        print(f"RANK {rank} ALL OK", flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    try:
        main()
    except Exception:
        traceback.print_exc()
        print(f"RANK {os.environ.get('RANK')} FAIL: exception", flush=True)
        sys.exit(1)
