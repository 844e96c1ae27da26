"""One neighbor_allreduce of 8 virtual agents (exp-2) on one GPU, fp32 and bf16, for ncu."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_04287_b200 as bfp, synthetic
n, nbytes = 8, 64 << 20
ctx = bfp.Context(agents_per_proc=n, heap_bytes=n * 2 * nbytes + (256 << 20), device=0)
ctx.set_topology(bfp.topology_matrix("exp2", n))
for dtype, es in ((torch.float32, 4), (torch.bfloat16, 2)):
    x = torch.empty(n, nbytes // es, device="cuda", dtype=dtype)
    for a in range(n):
        bfp.Context.fill_uniform(x[a], synthetic.SEED_X0 + a)
    y = torch.empty_like(x)
    for _ in range(3):
        ctx.neighbor_allreduce(x, out=y)
    torch.cuda.synchronize()
ctx.close()
print("ok")
