"""Host-side cost of one C-ABI call (tiny neighbor_allreduce, 4 agents x 1024 fp32):
Python wrapper vs a raw ctypes call with pre-built arguments."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_04287_b200 as bfp  # noqa: E402

ctx = bfp.Context(agents_per_proc=4, heap_bytes=1 << 26, device=0)
ctx.set_topology(bfp.topology_matrix("ring", 4))
x = torch.ones(4, 1024, device="cuda")
y = torch.empty_like(x)
for _ in range(100):
    ctx.neighbor_allreduce(x, out=y)
torch.cuda.synchronize()
n = 3000
t0 = time.perf_counter()
for _ in range(n):
    ctx.neighbor_allreduce(x, out=y)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
lib = ctx.lib
xs, ys, st = C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream)
t3 = time.perf_counter()
for _ in range(n):
    lib.bf_neighbor_allreduce(ctx.h, xs, ys, 1024, 0, None, st)
t4 = time.perf_counter()
torch.cuda.synchronize()
t5 = time.perf_counter()
t6 = time.perf_counter()
for _ in range(n):
    torch.cuda.current_stream()
t7 = time.perf_counter()
print(f"python wrapper: {(t1 - t0) / n * 1e6:.2f} us/call issue, {(t2 - t0) / n * 1e6:.2f} us/call incl. drain")
print(f"raw ctypes:     {(t4 - t3) / n * 1e6:.2f} us/call issue, {(t5 - t3) / n * 1e6:.2f} us/call incl. drain")
print(f"torch.cuda.current_stream(): {(t7 - t6) / n * 1e6:.2f} us")
ctx.close()
