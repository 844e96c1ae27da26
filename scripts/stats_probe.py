#!/usr/bin/env python
"""Per-round diagnostics of the fused exchange kernel (needs a -DBF_STATS=1
library via BF_LIB_PATH and BF_STATS=1).  Same workload as bench.py (C4).

  BF_STATS=1 BF_LIB_PATH=variants/lib_stats.so torchrun --nproc-per-node N scripts/stats_probe.py
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_04287_b200 as bfp  # noqa: E402
import synthetic  # noqa: E402


def main():
    topo = sys.argv[1] if len(sys.argv) > 1 else "one_peer"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    agents = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    count = 25_600_000
    k = agents // world
    ctx = bfp.Context(agents_per_proc=k, heap_bytes=(k + agents) * 2 * count * 4 + (64 << 20), device=local)
    n = ctx.n
    if topo == "one_peer":
        ctx.set_dynamic_schedule("one_peer_exp2", 0)
    else:
        ctx.set_topology(bfp.topology_matrix("exp2", n))
    x = torch.empty(k, count, device="cuda")
    g = torch.empty(k, count, device="cuda")
    for la in range(k):
        bfp.Context.fill_uniform(x[la], synthetic.SEED_X0 + ctx.rank + la)
        bfp.Context.fill_uniform(g[la], synthetic.grad_seed(0, ctx.rank + la), scale=2.0 ** -7)
    for _ in range(6):
        ctx.atc_step(x, g, 0.1)
    torch.cuda.synchronize()
    ctx.exchange_stats(reset=True)
    tau = max(1, (n - 1).bit_length()) if topo == "one_peer" else 1
    names = ["kernel", "cons_wait", "comm_wait_peer", "comm_wait_slot", "fence", "fences", "polls", "prologue"]
    if os.environ.get("BF_XFER", "push") != "pull" and (k <= 2 or os.environ.get("BF_XFER") == "push_all") and world > 1:   # exchange_push.cuh slots
        names = ["kernel", "cons_wait", "first_ready", "loop_end", "fence", "fences", "polls", "prologue"]
    rows = {r: [] for r in range(tau)}
    for s in range(6 * tau):
        if world > 1:
            dist.barrier()
        ctx.atc_step(x, g, 0.1)
        torch.cuda.synchronize()
        st = ctx.exchange_stats(reset=True).astype(np.float64)
        used = st[:, 0] > 0
        rows[(6 + s) % tau].append(st[used])
    if world > 1:
        dist.barrier()
    for r in range(tau):
        st = np.concatenate(rows[r])
        med = np.median(st, axis=0)
        mx = st.max(axis=0)
        txt = " ".join(f"{nm}={med[i] / (1 if nm in ('fences', 'polls') else 1e3):.1f}/{mx[i] / (1 if nm in ('fences', 'polls') else 1e3):.1f}"
                       for i, nm in enumerate(names))
        print(f"rank {rank} round {r} CTAs {st.shape[0] // 6}: median/max us: {txt}", flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
