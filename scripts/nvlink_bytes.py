#!/usr/bin/env python
"""NVLink bytes per step of the cross-GPU fused ATC step, from the GPUs' own
NVLink data counters (`nvidia-smi nvlink -gt d`, per-link Tx/Rx KiB), read
around a fixed number of steps -- a hardware count of what crossed the links,
without profiling a multi-rank run under ncu.

  torchrun --nproc-per-node N scripts/nvlink_bytes.py [one_peer|exp2] [agents] [steps]
"""
import json
import os
import re
import subprocess
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_04287_b200 as bfp  # noqa: E402
import synthetic  # noqa: E402

PAT = re.compile(r"Link\s+(\d+):\s+Data\s+(Tx|Rx):\s+(\d+)\s*KiB")


def counters():
    """{gpu: {"tx": bytes, "rx": bytes}} summed over links, or the raw text on failure."""
    out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d"], capture_output=True, text=True).stdout
    res, gpu = {}, None
    for line in out.splitlines():
        m = re.match(r"GPU\s+(\d+):", line.strip())
        if m:
            gpu = int(m.group(1))
            res[gpu] = {"tx": 0, "rx": 0}
            continue
        m = PAT.search(line)
        if m and gpu is not None:
            res[gpu]["tx" if m.group(2) == "Tx" else "rx"] += int(m.group(3)) * 1024
    return res, out


def main():
    topo = sys.argv[1] if len(sys.argv) > 1 else "one_peer"
    agents = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    k = agents // world
    count = 25_600_000
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
    dist.barrier()
    c0, raw0 = counters() if rank == 0 else ({}, "")
    dist.barrier()
    for _ in range(steps):
        ctx.atc_step(x, g, 0.1)
    torch.cuda.synchronize()
    dist.barrier()
    c1, raw1 = counters() if rank == 0 else ({}, "")
    if rank == 0:
        tau = max(1, (n - 1).bit_length())
        # algorithmic: distinct remote source agents of each GPU's agents x M (fp32)
        def sources(i, r):
            if topo == "one_peer":
                return [(i - (1 << (r % tau))) % n]
            d, off, out = 0, 1, []
            while off <= n - 1:
                out.append((i - off) % n)
                off *= 2
            return out
        alg = []
        for q in range(world):
            tot = 0
            for r in range(6, 6 + steps):
                tot += len({j for a in range(k) for j in sources(q * k + a, r) if j // k != q}) * count * 4
            alg.append(tot / steps)
        res = {"topology": topo, "agents": agents, "gpus": world, "steps": steps,
               "xfer": os.environ.get("BF_XFER", "push"),
               "algorithmic_nvlink_in_bytes_per_step": alg, "per_gpu": {}}
        for gq in sorted(c1):
            if gq in c0 and gq < world:
                res["per_gpu"][gq] = {"tx_bytes_per_step": (c1[gq]["tx"] - c0[gq]["tx"]) / steps,
                                      "rx_bytes_per_step": (c1[gq]["rx"] - c0[gq]["rx"]) / steps}
        if not res["per_gpu"]:
            res["raw"] = raw1[-2000:]
        print(json.dumps(res), flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
