"""Multi-process stress of the exchange protocol (run under torchrun): many
back-to-back calls of every fused op with random sizes, topologies and
schedules, each result checked against the oracle on the rows of this process.

  torchrun --nproc-per-node N scripts/stress_mp.py K ITERS
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as ora  # noqa: E402
import paper_2111_04287_b200 as bfp  # noqa: E402
import synthetic  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    ctx = bfp.Context(agents_per_proc=k, heap_bytes=1 << 29, device=local)
    n = ctx.n
    rows = slice(ctx.rank, ctx.rank + k)
    rng = np.random.default_rng(1234)          # same stream on every rank: same choices
    worst = {}
    bad = 0
    for it in range(iters):
        count = int(rng.choice([1, 5, 1023, 4096, 9999, 65537, 300001]))
        op = rng.choice(["nar", "atc", "atc_bf16", "awc", "ed"])
        topo = rng.choice(["exp2", "ring", "one_peer", "random"])
        if topo == "one_peer":
            r0 = int(rng.integers(0, 6))
            ctx.set_dynamic_schedule("one_peer_exp2", r0)
            W = ora.one_peer_exp2(n, r0)
        else:
            ctx.set_dynamic_schedule("none")
            if topo == "random":
                W = (rng.random((n, n)) < 0.4) * rng.uniform(-0.5, 1.0, (n, n))
                np.fill_diagonal(W, rng.uniform(0.2, 1.0, n))
            else:
                W = ora.exp2(n) if topo == "exp2" else ora.ring(n)
            ctx.set_topology(W)
        X = np.stack([synthetic.uniform(synthetic.SEED_X0 + 17 * it + r, count) for r in range(n)]).astype(np.float64)
        G = np.stack([synthetic.uniform(synthetic.grad_seed(it, r), count, scale=2.0 ** -7)
                      for r in range(n)]).astype(np.float64)
        x = torch.from_numpy(X[rows].astype(np.float32)).cuda()
        g = torch.from_numpy(G[rows].astype(np.float32)).cuda()
        lr = 0.1
        b = np.abs(W) @ (np.abs(X) + lr * np.abs(G))
        tol = 1e-6
        if op == "nar":
            y = ctx.neighbor_allreduce(x)
            ref = ora.mix(W, X)
        elif op in ("atc", "atc_bf16"):
            wire = torch.bfloat16 if op == "atc_bf16" else torch.float32
            ctx.atc_step(x, g, lr, wire=wire)
            y = x
            ref = ora.atc(W, X, G, lr, wire_bf16=(op == "atc_bf16"))
            tol = 1e-2 if op == "atc_bf16" else 1e-6
        elif op == "awc":
            ctx.awc_step(x, g, lr)
            y = x
            ref = ora.awc(W, X, G, lr)
            b = np.abs(W) @ np.abs(X) + lr * np.abs(G)
        else:
            P = np.stack([synthetic.uniform(synthetic.grad_seed(it + 99, r), count) for r in range(n)]).astype(np.float64)
            psi = torch.from_numpy(P[rows].astype(np.float32)).cuda()
            ctx.exact_diffusion_step(x, g, psi, lr)
            y = x
            ref, _ = ora.exact_diffusion(W, X, G, P, lr)
            b = np.abs(W) @ (2 * np.abs(X) + lr * np.abs(G) + np.abs(P))
        torch.cuda.synchronize()
        err = np.abs(y.cpu().numpy().astype(np.float64) - ref[rows]) / (b[rows] + 1e-30)
        e = float(err.max())
        worst[op] = max(worst.get(op, 0.0), e)
        if e > tol:
            bad += 1
            print(f"rank {rank} it {it} {op} {topo} count {count}: rel err {e:.3e} > {tol}", flush=True)
    ctx.poll_error()
    dist.barrier()
    print(f"rank {rank} K={k} iters={iters} failures={bad} worst=" +
          " ".join(f"{kk}:{vv:.2e}" for kk, vv in sorted(worst.items())), flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
