import os, sys
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_04287_b200 as bfp, synthetic
world = int(os.environ["WORLD_SIZE"]); rank = int(os.environ["RANK"]); local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
k, count = 2, 1048576
ctx = bfp.Context(agents_per_proc=k, heap_bytes=1 << 28, device=local)
for kk in range(3):
    ctx.set_dynamic_schedule("one_peer_exp2", kk)
    x = torch.ones(k, count, device="cuda"); g = torch.zeros(k, count, device="cuda")
    ctx.exchange_stats(reset=True)
    ctx.atc_step(x, g, 0.1)
    torch.cuda.synchronize()
    st = ctx.exchange_stats(reset=True)
    e = st[0, 3] >> 24
    print(f"rank {rank} round {kk}: epoch {e} CTA0 seen {st[0,2]>>24}:{st[0,2]&0xffffff} need {st[0,3]>>24}:{st[0,3]&0xffffff} remote-now {st[0,6]>>24}:{st[0,6]&0xffffff}; x mean {x.mean().item():.4f}", flush=True)
    dist.barrier()
