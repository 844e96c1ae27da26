"""One push-sum gradient-tracking round (gt_uv_step + gt_y_step) of 8 virtual agents x 25.6M fp32, for ncu."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_04287_b200 as bfp, synthetic
n, count = 8, 25_600_000
ctx = bfp.Context(agents_per_proc=n, heap_bytes=n * 2 * count * 4 + (256 << 20), device=0)
ctx.set_topology(bfp.topology_matrix("exp2", n))
u, y, g, gp, xo = (torch.empty(n, count, device="cuda") for _ in range(5))
for a in range(n):
    for i, t in enumerate((u, y, g, gp)):
        bfp.Context.fill_uniform(t[a], synthetic.SEED_X0 + 10 * i + a, scale=2.0 ** -7)
v = torch.ones(n, device="cuda")
for r in range(3):
    ctx.gt_uv_step(u, v, y, xo, 1e-3)
    ctx.gt_y_step(y, g, gp)
torch.cuda.synchronize()
ctx.close()
print("ok")
