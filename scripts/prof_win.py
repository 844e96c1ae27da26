"""One push-sum round (win_accumulate + win_update_then_collect) of 8 virtual agents, bf16, for ncu."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_04287_b200 as bfp, synthetic
n, count = 8, 64 << 20
ctx = bfp.Context(agents_per_proc=n, heap_bytes=n * 3 * count * 8 + (1 << 30), device=0)
ctx.set_topology(bfp.topology_matrix("exp2", n))
x = torch.empty(n, count, device="cuda", dtype=torch.bfloat16)
for a in range(n):
    bfp.Context.fill_uniform(x[a], synthetic.SEED_X0 + a)
ctx.win_create(x, "ext", zero_init=True, with_p=True)
for r in range(4):
    dst = [{bfp.one_peer_exp2(n, a, r)[1]: 0.5} for a in range(n)]
    ctx.win_accumulate("ext", self_weight=[0.5] * n, dst_weights=dst)
    ctx.win_update_then_collect("ext")
torch.cuda.synchronize()
ctx.close()
print("ok")
