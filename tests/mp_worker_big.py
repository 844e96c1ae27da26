"""Multi-process parity at the production shape (one process per GPU, launched by
torchrun from tests/test_multigpu.py): 25.6M fp32 elements per agent (the C4 /
ResNet-50 buffer), BF_TEST_K agents per process, so the cross-GPU fused
kernel runs its full pipeline -- many sub-items per CTA, the publish-ahead
(kLead), batch releases, the TMA ring wrapping, the U = 2 groups of K <= 2.

Every op is column-wise, so each round is checked on sampled columns: the
sampled columns of every rank are all-gathered (NCCL, test plumbing), the oracle
computes the round on them, each rank checks its own rows.  The GPU state is fed
to the oracle every round (step-by-step chaining)."""
import os
import sys
import time
import traceback

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("BF_TIMEOUT_MS", "10000")

import oracle as ora  # noqa: E402
import synthetic  # noqa: E402
import paper_2111_04287_b200 as bfp  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    rank = int(os.environ["RANK"])
    # BF_TEST_SHARE_GPUS=G: more processes than GPUs (process p on GPU p mod G, gloo bootstrap)
    share = int(os.environ.get("BF_TEST_SHARE_GPUS", "0"))
    if share:
        local = local % share
    torch.cuda.set_device(local)
    if share:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    k = int(os.environ.get("BF_TEST_K", "1"))
    count = int(os.environ.get("BF_TEST_COUNT", str(25_600_000)))
    ctx = bfp.Context(agents_per_proc=k, heap_bytes=3 << 30, device=local)
    n, r0 = ctx.n, ctx.rank
    rows = slice(r0, r0 + k)
    failures = []
    t0 = time.time()

    rng = np.random.default_rng(0)
    edges = [0, 1, 1023, 1024, 2047, 2048, 296 * 1024 - 1, 296 * 1024, 296 * 2048 + 5, count - 2049,
             count - 1024, count - 5, count - 1]
    cols = np.unique(np.concatenate([rng.integers(0, count, 4000), [e for e in edges if 0 <= e < count]]))
    ct = torch.from_numpy(cols).cuda()

    def gather(t):
        """(n, ncols) fp64: the sampled columns of every agent (all ranks)."""
        mine = t[:, ct].float().contiguous()
        if share:   # gloo: gather on the host
            mine = mine.cpu()
        out = [torch.empty_like(mine) for _ in range(dist.get_world_size())]
        dist.all_gather(out, mine)
        return torch.cat(out).cpu().numpy().astype(np.float64)

    def check(name, y, ref, W, X, tol, extra=None):
        b = np.abs(W) @ np.abs(X)
        if extra is not None:
            b = b + extra
        err = np.abs(y[rows] - ref[rows])
        bb = b[rows]
        if (err > tol * bb + 1e-30).any():
            failures.append(f"{name}: max rel {np.max(err / (bb + 1e-30)):.3e}")

    def fill(seed_fn, scale=1.0, dtype=torch.float32):
        t = torch.empty(k, count, device="cuda", dtype=dtype)
        for a in range(k):
            bfp.Context.fill_uniform(t[a], seed_fn(r0 + a), scale=scale)
        return t

    lr = 0.1
    # ---- one-peer exp-2 schedule: every fused op, consecutive rounds ----
    ctx.set_dynamic_schedule("one_peer_exp2", 0)
    x = fill(lambda r: synthetic.SEED_X0 + r)
    rnd = 0
    for step, wire in enumerate([torch.float32] * 3 + [torch.bfloat16] * 2):
        g = fill(lambda r: synthetic.grad_seed(step, r), 2.0 ** -7)
        X, G = gather(x), gather(g)
        ctx.atc_step(x, g, lr, wire=wire)
        Wk = ora.one_peer_exp2(n, rnd)
        check(f"one-peer atc {wire} round {rnd}", gather(x),
              ora.atc(Wk, X, G, lr, wire_bf16=wire == torch.bfloat16), Wk, X,
              1e-6 if wire == torch.float32 else 1e-2, np.abs(Wk) @ (np.float32(lr) * np.abs(G)))
        rnd += 1
    g = fill(lambda r: synthetic.grad_seed(7, r), 2.0 ** -7)
    X, G = gather(x), gather(g)
    ctx.awc_step(x, g, lr)
    Wk = ora.one_peer_exp2(n, rnd)
    check(f"one-peer awc round {rnd}", gather(x), ora.awc(Wk, X, G, lr), Wk, X, 1e-6, np.float32(lr) * np.abs(G))
    rnd += 1
    X = gather(x)
    y = ctx.neighbor_allreduce(x)
    Wk = ora.one_peer_exp2(n, rnd)
    check(f"one-peer nar round {rnd}", gather(y), ora.mix(Wk, X), Wk, X, 1e-6)
    rnd += 1
    psi = x.clone()
    for step in range(2):
        g = fill(lambda r: synthetic.grad_seed(8 + step, r), 2.0 ** -7)
        X, G, P = gather(x), gather(g), gather(psi)
        ctx.exact_diffusion_step(x, g, psi, lr)
        Wk = ora.one_peer_exp2(n, rnd)
        ref, _ = ora.exact_diffusion(Wk, X, G, P, lr)
        check(f"one-peer ED round {rnd}", gather(x), ref, Wk, 2 * np.abs(X) + lr * np.abs(G) + np.abs(P), 1e-6)
        rnd += 1
    xb = x.to(torch.bfloat16)
    X = gather(xb)
    yb = ctx.neighbor_allreduce(xb)
    Wk = ora.one_peer_exp2(n, rnd)
    check(f"one-peer nar bf16 round {rnd}", gather(yb), ora.mix(Wk, X), Wk, X, 1e-2)
    ctx.set_dynamic_schedule("none")
    del xb, yb, psi, y

    # ---- static exponential-2: chained ATC steps + neighbor_allreduce ----
    We = ora.exp2(n)
    ctx.set_topology(We)
    for step in range(2):
        g = fill(lambda r: synthetic.grad_seed(20 + step, r), 2.0 ** -7)
        X, G = gather(x), gather(g)
        ctx.atc_step(x, g, lr)
        check(f"exp2 atc step {step}", gather(x), ora.atc(We, X, G, lr), We, X, 1e-6,
              np.abs(We) @ (np.float32(lr) * np.abs(G)))
    X = gather(x)
    y = ctx.neighbor_allreduce(x)
    check("exp2 nar", gather(y), ora.mix(We, X), We, X, 1e-6)
    del y

    # ---- hierarchical at the production size (machines of 2) -------------
    if n % 2 == 0 and n >= 4:
        WM = ora.exp2(n // 2)
        ctx.set_machine_topology(WM, 2)
        Kh = np.kron(WM, np.full((2, 2), 0.5))
        X = gather(x)
        y = ctx.hierarchical_neighbor_allreduce(x)
        check("hier L=2", gather(y), ora.hier(WM, 2, X), Kh, X, 1e-6)
        g = fill(lambda r: synthetic.grad_seed(30, r), 2.0 ** -7)
        G = gather(g)
        ctx.hierarchical_atc_step(x, g, lr)
        check("H-ATC L=2", gather(x), ora.hier_atc(WM, 2, X, G, lr), Kh, X, 1e-6,
              np.abs(Kh) @ (np.float32(lr) * np.abs(G)))
        del y
    del x, g

    # ---- windows at > grid items: synchronous push-sum (Listing 3) ----
    wc = (1 << 22) + 8
    Wst = ora.exp2(n)
    ctx.set_topology(Wst)
    Wps = np.zeros((n, n))
    for i in range(n):
        outs = ora.out_neighbors(Wst, i)
        w = 1.0 / (len(outs) + 1)
        Wps[i, i] = w
        for j in outs:
            Wps[j, i] = w
    for dtype, tol in ((torch.float32, 1e-6), (torch.bfloat16, 1e-2)):
        xw = torch.empty(k, wc, device="cuda", dtype=dtype)
        tmp = torch.empty(k, wc, device="cuda")
        for a in range(k):
            bfp.Context.fill_uniform(tmp[a], synthetic.SEED_X0 + 60 + r0 + a)
        xw.copy_(tmp)
        del tmp
        name = f"w{int(dtype == torch.bfloat16)}"
        ctx.win_create(xw, name, zero_init=True, with_p=True)
        cw = torch.from_numpy(np.unique(np.concatenate([rng.integers(0, wc, 3000), [0, wc - 1]]))).cuda()
        gw = lambda t: _gather_cols(t, cw)
        p = np.ones(n)
        for rr in range(3):
            X = gw(xw)
            ctx.win_accumulate(name)
            ctx.barrier()
            ctx.win_update_then_collect(name)
            ctx.barrier()
            check(f"window {dtype} round {rr}", gw(xw), ora.mix(Wps, X), Wps, X, tol)
            p = Wps @ p
            torch.cuda.synchronize()
            if np.abs(ctx.win_p(name) - p[rows]).max() > 1e-12:
                failures.append(f"window {dtype} p round {rr}")
        torch.cuda.synchronize()
        dist.barrier()
        ctx.win_free(name)
        del xw

    dist.barrier()
    el = time.time() - t0
    if failures:
        print(f"RANK {rank} FAIL ({el:.0f}s): " + "; ".join(failures), flush=True)
    else:
        print(f"RANK {rank} ALL OK ({el:.0f}s)", flush=True)
    ctx.close()
    dist.destroy_process_group()


def _gather_cols(t, cw):
    mine = t[:, cw].float().contiguous()
    if dist.get_backend() == "gloo":   # BF_TEST_SHARE_GPUS: gather on the host
        mine = mine.cpu()
    out = [torch.empty_like(mine) for _ in range(dist.get_world_size())]
    dist.all_gather(out, mine)
    return torch.cat(out).cpu().numpy().astype(np.float64)


if __name__ == "__main__":
    try:
        main()
    except Exception:
        traceback.print_exc()
        print(f"RANK {os.environ.get('RANK')} FAIL: exception", flush=True)
        sys.exit(1)
