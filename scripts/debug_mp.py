"""Focused multi-process ATC check: every (round, wire) combination, with the
location of the worst element (debug aid, run under torchrun)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as ora  # noqa: E402
import paper_2111_04287_b200 as bfp  # noqa: E402
import synthetic  # noqa: E402

world = int(os.environ["WORLD_SIZE"]); rank = int(os.environ["RANK"]); local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
count = int(sys.argv[2]) if len(sys.argv) > 2 else 123457
ctx = bfp.Context(agents_per_proc=k, heap_bytes=1 << 28, device=local)
n = ctx.n
rows = list(range(rank * k, rank * k + k))
for wire in (torch.float32, torch.bfloat16):
    for kk in range(3):
        ctx.set_dynamic_schedule("one_peer_exp2", kk)
        X = synthetic.agents_x0(n, count).astype(np.float64)
        G = np.stack([synthetic.uniform(synthetic.grad_seed(1, r), count, scale=2.0 ** -7) for r in range(n)])
        x = torch.from_numpy(X[rows].astype(np.float32)).cuda()
        g = torch.from_numpy(G[rows].copy()).cuda()
        print(f"rank {rank} round={kk} x ptr {hex(x.data_ptr())} g ptr {hex(g.data_ptr())}", flush=True)
        ctx.atc_step(x, g, 0.1, wire=wire)
        torch.cuda.synchronize()
        Wk = ora.one_peer_exp2(n, kk)
        ref = ora.atc(Wk, X, G.astype(np.float64), 0.1, wire_bf16=wire == torch.bfloat16)[rows]
        got = x.cpu().numpy().astype(np.float64)
        b = (np.abs(Wk) @ (np.abs(X) + 0.1 * np.abs(G)))[rows]
        rel = np.abs(got - ref) / b
        bad = np.argwhere(rel > (1e-6 if wire == torch.float32 else 1e-2))
        if len(bad):   # which wrong result is it?
            Xh = X - np.float32(0.1) * G
            hyps = {"self_only": 0.5 * Xh[rows], "zero": 0 * Xh[rows], "input": X[rows]}
            for j in range(n):
                hyps[f"self+src{j}"] = 0.5 * Xh[rows] + 0.5 * Xh[j]
            for name, h in hyps.items():
                e = np.abs(got - h) / b
                print(f"rank {rank} round={kk} hypothesis {name}: max rel {e.max():.3e} agent0 {e[0].max():.2e} agent1 {e[-1].max():.2e}", flush=True)
        print(f"rank {rank} k={k} wire={wire} round={kk}: max rel {rel.max():.3e} bad {len(bad)}"
              + (f" first {bad[:3].tolist()} last {bad[-3:].tolist()} sub-items {sorted(set((bad[:, 1] // 1024).tolist()))[:12]}" if len(bad) else ""),
              flush=True)
        dist.barrier()
ctx.close()
dist.destroy_process_group()
