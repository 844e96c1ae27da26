"""N = 1 C4 step: eager launches vs the same steps captured in one CUDA graph (diagnostic)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_04287_b200 as bfp, synthetic
n, count = 8, 25_600_000
ctx = bfp.Context(agents_per_proc=n, heap_bytes=n * 2 * count * 4 + (64 << 20), device=0)
ctx.set_dynamic_schedule("one_peer_exp2", 0)
x = torch.empty(n, count, device="cuda")
gs = [torch.empty(n, count, device="cuda") for _ in range(2)]
for a in range(n):
    bfp.Context.fill_uniform(x[a], synthetic.SEED_X0 + a)
    for s, g in enumerate(gs):
        bfp.Context.fill_uniform(g[a], synthetic.grad_seed(s, a), scale=2.0 ** -7)
def steps(k):
    for s in range(k):
        ctx.atc_step(x, gs[s % 2], 0.1)
for _ in range(3):
    steps(6)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); steps(60); e1.record(); torch.cuda.synchronize()
print("eager ms/step", e0.elapsed_time(e1) / 60)
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st):
    steps(6)
torch.cuda.current_stream().wait_stream(st)
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr):
    steps(60)
gr.replay(); torch.cuda.synchronize()
e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
print("graph ms/step", e0.elapsed_time(e1) / 60)
ctx.close()
