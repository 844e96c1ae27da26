#!/usr/bin/env python
"""Measurement suite for the BASELINE.json configs beyond bench.py's C4 line.

  C1  consensus, ring-4, fp32[4096], 20 iterations: microseconds per iteration
  C2  ATC-DSGD on synthetic least squares (d=10k, 8 agents, m=2000 rows each):
      iterations/s and distance to the oracle's x* (gradients by torch GEMV --
      workload plumbing, not the hot path)
  C3  neighbor_allreduce sweep 1 KB .. 1 GB per agent, fp32/bf16, static exp-2
      vs one-peer: exchange GB/s per GPU and HBM fraction
  C5  push-sum through win_accumulate / win_update_then_collect, 340M bf16 per
      agent, one-peer destinations inside the static exp-2 window topology
  H   hierarchical_neighbor_allreduce, 25.6M fp32, L = 2, 4
  O   ATC optimizer wrapper over ResNet-50's 161 parameter tensors (tensor
      fusion into buckets, one fused kernel per bucket)
  E   Exact-Diffusion step (appendix ed-1..ed-3), 8 agents x 25.6M fp32; and
      in C2, Exact-Diffusion vs ATC distance to the exact minimiser x*

One JSON object per line.  N = 1: the 8 agents are virtual agents of one GPU;
under torchrun, 8/N agents per GPU.  Every number is CUDA-event time on the
launching stream, after warm-up, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c3,c5,h,io,o,e,gt,c2,oracle")
    ap.add_argument("--agents", type=int, default=8)
    ap.add_argument("--max-bytes", type=int, default=1 << 30)
    ap.add_argument("--out", default=None)
    return ap.parse_args()


def main():
    a = parse()
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2111_04287_b200 as bfp
    import synthetic

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    out = open(a.out, "a") if (a.out and rank == 0) else None
    stream = torch.cuda.current_stream()

    def emit(d):
        d["n_gpus"] = world
        if rank == 0:
            line = json.dumps(d)
            print(line, flush=True)
            if out:
                out.write(line + "\n")
                out.flush()

    def timed(fn, iters, warm=3):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / iters], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms)

    only = set(a.only.split(","))

    def fresh():
        # every config starts from fresh allocations: carving its buffers out of the
        # previous config's freed blocks measurably changed the HBM-bound lines (e.g. the
        # Exact-Diffusion step after C5 0.684 -> 0.786 ms at N = 1, profiles/r02c_suite_order_n1.txt)
        import gc
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()

    def xheap(k, n, bytes_per_agent, extra):
        # exchange slots (k agents x 2 parities) + across GPUs the push inboxes (n x 2)
        # and the tagged-word inboxes (n x 2 x BF_LL_CAP x 8 B)
        ll = n * 2 * int(os.environ.get("BF_LL_CAP", "262144")) * 8 if world > 1 else 0
        return (k + (n if world > 1 else 0)) * 2 * bytes_per_agent + extra + ll

    # ---------------------------------------------------------------- C1 ----
    if "c1" in only:
        n = 4
        if n % world == 0:
            k = n // world
            ctx = bfp.Context(agents_per_proc=k, heap_bytes=64 << 20, device=local)
            ctx.set_topology(bfp.topology_matrix("ring", n))
            x = torch.empty(k, 4096, device="cuda")
            for la in range(k):
                bfp.Context.fill_uniform(x[la], synthetic.SEED_X0 + ctx.rank + la)
            y = torch.empty_like(x)

            def c1():
                for _ in range(10):
                    ctx.neighbor_allreduce(x, out=y)
                    ctx.neighbor_allreduce(y, out=x)
            ms = timed(c1, 5)
            emit({"config": "C1 consensus ring-4 fp32[4096] x 20 iterations", "us_per_iteration": ms * 1e3 / 20,
                  "ms_20_iterations": ms, "launch": "eager (one C-ABI call per iteration)"})
            # the same 20 iterations captured once in a CUDA graph (epochs live in device memory)
            gs = torch.cuda.Stream()
            gs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(gs):
                c1()
            torch.cuda.current_stream().wait_stream(gs)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                c1()
            ms = timed(graph.replay, 5)
            emit({"config": "C1 consensus ring-4 fp32[4096] x 20 iterations", "us_per_iteration": ms * 1e3 / 20,
                  "ms_20_iterations": ms, "launch": "CUDA graph of the 20 iterations"})
            ctx.close()

    # ---------------------------------------------------------------- C3 ----
    if "c3" in only:
        x = g = y = psi = u = gp = xo = None   # the previous config's buffers
        fresh()
        n = a.agents
        k = n // world
        maxb = a.max_bytes
        # + room for the registered (bf_alloc) fp32 input of the largest size
        ctx = bfp.Context(agents_per_proc=k, heap_bytes=xheap(k, n, maxb, k * maxb + (256 << 20)), device=local)
        ctx.reserve(maxb)
        W = bfp.topology_matrix("exp2", n)
        for dtype, es in ((torch.float32, 4), (torch.bfloat16, 2)):
            nb = 1024
            while nb <= maxb:
                count = nb // es
                x = torch.empty(k, count, device="cuda", dtype=dtype)
                for la in range(k):
                    bfp.Context.fill_uniform(x[la], synthetic.SEED_X0 + ctx.rank + la)
                y = torch.empty_like(x)
                for topo in ("exp2", "one_peer"):
                    if topo == "exp2":
                        ctx.set_topology(W)
                        d = 3 if n == 8 else int(np.count_nonzero(W[0])) - 1
                    else:
                        ctx.set_dynamic_schedule("one_peer_exp2", 0)
                        d = 1
                    iters = max(3, min(200, int(2e8 // max(nb, 1))))
                    ms = timed(lambda: ctx.neighbor_allreduce(x, out=y), iters)
                    ctx.set_dynamic_schedule("none")
                    gbs = k * d * nb / (ms * 1e-3) / 1e9
                    # fused kernel: read x + write y per agent; the wire copy is published only
                    # by agents read from another GPU (none at N = 1)
                    pubs = 0 if world == 1 else k
                    hbm = (k * 2 + pubs) * nb / (ms * 1e-3) / 1e9
                    emit({"config": "C3 neighbor_allreduce sweep", "bytes_per_agent": nb,
                          "dtype": str(dtype).split(".")[-1], "topology": topo, "agents": n, "agents_per_gpu": k,
                          "input": "torch tensor (unregistered)",
                          "us": ms * 1e3, "exchange_gbs_per_gpu": gbs, "hbm_gbs": hbm, "hbm_frac": hbm / peak})
                del x, y
                nb *= 4
        # the same call on a registered input (bf_alloc: the tensor lives in the symmetric heap).
        # Nothing to save here: across GPUs the writer stores its wire copy into the readers'
        # inboxes straight from registers, and on one GPU nothing is published -- there is no
        # publish copy that registration could avoid (SURVEY C3 asks for both lines)
        nb = maxb
        count = nb // 4
        x = ctx.alloc((k, count))
        for la in range(k):
            bfp.Context.fill_uniform(x[la], synthetic.SEED_X0 + ctx.rank + la)
        y = torch.empty_like(x)
        for topo in ("exp2", "one_peer"):
            if topo == "exp2":
                ctx.set_topology(W)
                d = 3 if n == 8 else int(np.count_nonzero(W[0])) - 1
            else:
                ctx.set_dynamic_schedule("one_peer_exp2", 0)
                d = 1
            ms = timed(lambda: ctx.neighbor_allreduce(x, out=y), 3)
            ctx.set_dynamic_schedule("none")
            gbs = k * d * nb / (ms * 1e-3) / 1e9
            hbm = (k * 2 + (0 if world == 1 else k)) * nb / (ms * 1e-3) / 1e9
            emit({"config": "C3 neighbor_allreduce sweep", "bytes_per_agent": nb, "dtype": "float32", "topology": topo,
                  "agents": n, "agents_per_gpu": k, "input": "registered (bf_alloc, symmetric heap)",
                  "us": ms * 1e3, "exchange_gbs_per_gpu": gbs, "hbm_gbs": hbm, "hbm_frac": hbm / peak})
        del x, y
        ctx.close()

    # ----------------------------------------------------------------- H ----
    if "h" in only:
        x = g = y = psi = u = gp = xo = None   # the previous config's buffers
        fresh()
        hier_env = os.environ.get("BF_HIER", "")
        hier_fused = (world == 1 and hier_env != "staged") or hier_env == "fused"
        n = a.agents
        k = n // world
        count = 25_600_000
        ctx = bfp.Context(agents_per_proc=k, heap_bytes=xheap(k, n, count * 4, 6 * k * count * 4 + (1 << 30)),
                          device=local)
        x = torch.empty(k, count, device="cuda")
        for la in range(k):
            bfp.Context.fill_uniform(x[la], synthetic.SEED_X0 + ctx.rank + la)
        y = torch.empty_like(x)
        for L in (2, 4):
            nm = n // L
            ctx.set_machine_topology(bfp.topology_matrix("exp2", nm), L)
            nvls = False
            if world > 1 and L > k and L % k == 0 and os.environ.get("BF_NVLS", "1") != "0":
                nvls = ctx.enable_nvls(L, count)     # machines span GPUs: average in the switch
                nvls = nvls and L // k >= int(os.environ.get("BF_NVLS_MIN_P", "4"))   # the library's threshold
            ms = timed(lambda: ctx.hierarchical_neighbor_allreduce(x, out=y), 20)
            dm = 1 if nm == 2 else (2 if nm in (3, 4) else 3)
            if world > 1 and not hier_fused:
                path = ("NVLS machine average (multimem.ld_reduce) + push machine exchange" if nvls else
                        "push hierarchical mode (machine average in registers / per-process partials)"
                        if (L <= k and k % L == 0) or L % k == 0 else "staged kernel")
            if hier_fused:
                # one GPU: the Kronecker mix W_M (x) J/L in the fused kernel -- read x, write y
                per_agent, path = 2 * count * 4, "fused kernel, W = W_M (x) J_L/L (read x + write y)"
            else:
                per_agent = (2 * (L - 1) + dm) * count * 4 / L + 3 * count * 4
            emit({"config": f"H hierarchical_neighbor_allreduce 25.6M fp32, {nm} machines x {L}", "ms": ms,
                  "path": path, "gbs_per_gpu": k * per_agent / (ms * 1e-3) / 1e9,
                  "hbm_frac": k * per_agent / (ms * 1e-3) / 1e9 / peak if world == 1 else None})
        # H-ATC / H-AWC (caption P:869): the step of Table, in place on x
        g = torch.empty_like(x)
        for la in range(k):
            bfp.Context.fill_uniform(g[la], synthetic.grad_seed(0, ctx.rank + la), 2.0 ** -7)
        for L in (2, 4):
            nm = n // L
            ctx.set_machine_topology(bfp.topology_matrix("exp2", nm), L)
            nvls = False
            if world > 1 and L > k and L % k == 0 and os.environ.get("BF_NVLS", "1") != "0":
                nvls = ctx.enable_nvls(L, count) and L // k >= int(os.environ.get("BF_NVLS_MIN_P", "4"))
            for style, fn in (("H-ATC", ctx.hierarchical_atc_step), ("H-AWC", ctx.hierarchical_awc_step)):
                ms = timed(lambda: fn(x, g, 1e-3), 20)
                dm = 1 if nm == 2 else (2 if nm in (3, 4) else 3)
                if hier_fused:
                    per_agent, path = 3 * count * 4, "fused kernel, W = W_M (x) J_L/L (read x, g + write x)"
                else:
                    per_agent = (2 * (L - 1) + dm) * count * 4 / L + 4 * count * 4
                    path = ("NVLS machine average + push machine exchange" if nvls else
                            "push hierarchical mode" if (L <= k and k % L == 0) or L % k == 0 else "staged kernel")
                emit({"config": f"{style} step 25.6M fp32, {nm} machines x {L}", "ms": ms, "path": path,
                      "gbs_per_gpu": k * per_agent / (ms * 1e-3) / 1e9,
                      "hbm_frac": k * per_agent / (ms * 1e-3) / 1e9 / peak if world == 1 else None})
        ctx.close()

    # ------------------------------------------- inner-outer exp-2 schedule ----
    if "io" in only:
        x = g = y = psi = u = gp = xo = None   # the previous config's buffers
        fresh()
        n = a.agents
        k = n // world
        count = 25_600_000
        ctx = bfp.Context(agents_per_proc=k, heap_bytes=xheap(k, n, count * 4, 6 * k * count * 4 + (1 << 30)),
                          device=local)
        x = torch.empty(k, count, device="cuda")
        g = torch.empty_like(x)
        for la in range(k):
            bfp.Context.fill_uniform(x[la], synthetic.SEED_X0 + ctx.rank + la)
            bfp.Context.fill_uniform(g[la], synthetic.grad_seed(0, ctx.rank + la), 2.0 ** -7)
        for L in (2, 4):
            ctx.set_machine_topology(bfp.topology_matrix("exp2", n // L), L)
            ctx.set_dynamic_schedule("inner_outer_exp2", 0)
            ms = timed(lambda: ctx.atc_step(x, g, 1e-3), 4 * L)   # whole periods of the outer rotation
            emit({"config": f"ATC step, inner-outer exp-2 schedule (P:828, R27), 25.6M fp32 x {n}, machines of {L}",
                  "ms": ms, "gbs_per_gpu": k * 12 * count / (ms * 1e-3) / 1e9,
                  "hbm_frac": k * 12 * count / (ms * 1e-3) / 1e9 / peak if world == 1 else None})
        ctx.set_dynamic_schedule("none")
        ctx.close()

    # ---------------------------------------------------------------- C5 ----
    if "c5" in only:
        x = g = y = psi = u = gp = xo = None   # the previous config's buffers
        fresh()
        n = a.agents
        k = n // world
        count = 340_000_000
        try:
            ctx = bfp.Context(agents_per_proc=k, heap_bytes=k * 3 * count * (2 * 2 + 4) + (1 << 30), device=local)
            ctx.set_topology(bfp.topology_matrix("exp2", n))
            x = torch.empty(k, count, device="cuda", dtype=torch.bfloat16)
            for la in range(k):
                bfp.Context.fill_uniform(x[la], synthetic.SEED_X0 + ctx.rank + la)
            ctx.win_create(x, "ext", zero_init=True, with_p=True)
            r = [0]

            def c5():
                ks = r[0]
                dst = []
                for la in range(k):
                    _, d_ = bfp.one_peer_exp2(n, ctx.rank + la, ks)
                    dst.append({d_: 0.5})
                ctx.win_accumulate("ext", self_weight=[0.5] * k, dst_weights=dst)
                ctx.win_update_then_collect("ext")
                r[0] += 1
            ms = timed(c5, 10)
            # drain (untimed): every process collects what it was sent, then pushes what its
            # outboxes still owe and collects again -- only then is sum_i p_i = n exact
            def sync():
                torch.cuda.synchronize()
                if world > 1:
                    dist.barrier()
            sync()
            ctx.win_update_then_collect("ext")       # everything already delivered
            sync()
            flush = [{j: 0.0 for j in ctx.out_neighbor_ranks(ctx.rank + la)} for la in range(k)]
            ctx.win_accumulate("ext", self_weight=[1.0] * k, dst_weights=flush)   # owed outboxes only
            sync()
            if world > 1:
                dist.barrier()
            ctx.win_update_then_collect("ext")
            torch.cuda.synchronize()
            p = ctx.win_p("ext")
            tot = torch.tensor([float(p.sum())], device="cuda", dtype=torch.float64)
            if world > 1:
                dist.all_reduce(tot)
            nvl = k * count * 2                      # one payload per agent per round
            emit({"config": "C5 push-sum round (win_accumulate + win_update_then_collect), 340M bf16/agent, "
                            "one-peer dst in exp-2 window", "ms_per_round": ms, "rounds_per_s": 1e3 / ms,
                  "payload_gbs_per_gpu": nvl / (ms * 1e-3) / 1e9, "sum_p": float(tot), "expected_sum_p": n})
            ctx.win_free("ext")
            ctx.close()
        except Exception as ex:  # noqa: BLE001
            emit({"config": "C5", "error": repr(ex)[:300]})

    # ----------------------------------------------------------------- E ----
    # Exact-Diffusion step (appendix ed-1..ed-3) fused like ATC, C4-sized vectors
    if "e" in only:
        x = g = y = psi = u = gp = xo = None   # the previous config's buffers
        fresh()
        n = a.agents
        k = n // world
        count = 25_600_000
        ctx = bfp.Context(agents_per_proc=k, heap_bytes=xheap(k, n, count * 4, 256 << 20), device=local)
        ctx.set_topology(bfp.topology_matrix("exp2", n))
        x = torch.empty(k, count, device="cuda")
        g = torch.empty(k, count, device="cuda")
        psi = torch.empty(k, count, device="cuda")
        for la in range(k):
            bfp.Context.fill_uniform(x[la], synthetic.SEED_X0 + ctx.rank + la)
            bfp.Context.fill_uniform(g[la], synthetic.grad_seed(0, ctx.rank + la), scale=2.0 ** -7)
        psi.copy_(x)
        ms = timed(lambda: ctx.exact_diffusion_step(x, g, psi, 0.1), 20)
        hbm = k * 20 * count / (ms * 1e-3) / 1e9     # x, g, psi read + psi, x write
        emit({"config": f"E Exact-Diffusion step, {n} agents x {count} fp32, static exp-2", "ms_per_step": ms,
              "iters_per_s": 1e3 / ms, "hbm_gbs": hbm if world == 1 else None,
              "hbm_frac": hbm / peak if world == 1 else None})
        ctx.close()

    # ---------------------------------------------------------------- GT ----
    # push-sum gradient tracking round (appendix): the two fused
    # launches (gt_uv_step, gt_y_step) over C4-sized vectors, static exp-2
    if "gt" in only:
        x = g = y = psi = u = gp = xo = None   # the previous config's buffers
        fresh()
        n = a.agents
        k = n // world
        count = 25_600_000
        ctx = bfp.Context(agents_per_proc=k, heap_bytes=xheap(k, n, count * 4, 256 << 20), device=local)
        ctx.set_topology(bfp.topology_matrix("exp2", n))
        u, y, g, gp, xo = (torch.empty(k, count, device="cuda") for _ in range(5))
        for la in range(k):
            for i, t in enumerate((u, y, g, gp)):
                bfp.Context.fill_uniform(t[la], synthetic.SEED_X0 + 10 * i + ctx.rank + la, scale=2.0 ** -7)
        v = torch.ones(k, device="cuda")

        def gt_round():
            ctx.gt_uv_step(u, v, y, xo, 1e-3)
            ctx.gt_y_step(y, g, gp)
        ms = timed(gt_round, 20)
        hbm = k * 32 * count        # uv: u, y read + u, x write; y: y, g, g_prev read + y write
        emit({"config": f"GT push-sum gradient-tracking round (2 fused launches), {n} agents x {count} fp32, "
                        "static exp-2", "ms_per_round": ms, "rounds_per_s": 1e3 / ms,
              "hbm_gbs": hbm / (ms * 1e-3) / 1e9 if world == 1 else None,
              "hbm_frac": hbm / (ms * 1e-3) / 1e9 / peak if world == 1 else None})
        ctx.close()

    # ----------------------------------------------------------------- O ----
    # ATC optimizer over ResNet-50's 161 parameter tensors (tensor fusion into
    # buckets, one fused kernel per bucket), synthetic gradients (§8(f) rank 3)
    if "o" in only:
        x = g = y = psi = u = gp = xo = None   # the previous config's buffers
        fresh()
        import math
        from paper_2111_04287_b200.optim import DistributedAdaptThenCombineOptimizer, resnet50_param_shapes
        n = a.agents
        k = n // world
        shapes = resnet50_param_shapes()
        total = sum(math.prod(sh) for sh in shapes)
        ctx = bfp.Context(agents_per_proc=k, heap_bytes=xheap(k, n, total * 4, 256 << 20), device=local)
        ctx.set_dynamic_schedule("one_peer_exp2", 0)
        for bucket_mb in (4, 25, 128):
            params = [torch.nn.Parameter(torch.zeros(k, *sh, device="cuda")) for sh in shapes]
            opt = DistributedAdaptThenCombineOptimizer(ctx, params, 0.1, bucket_bytes=bucket_mb << 20)
            for bi, bkt in enumerate(opt.buckets):
                for la in range(k):
                    bfp.Context.fill_uniform(bkt.x[la], synthetic.SEED_X0 + ctx.rank + la, offset=bi << 28)
                    bfp.Context.fill_uniform(bkt.g[la], synthetic.grad_seed(0, ctx.rank + la), offset=bi << 28,
                                             scale=2.0 ** -7)
            ms = timed(opt.step, 20)
            emit({"config": f"O ATC optimizer, ResNet-50 parameter list (161 tensors, {total} elements) x "
                            f"{n} agents, one-peer, {bucket_mb} MB buckets", "buckets": len(opt.buckets),
                  "ms_per_step": ms, "iters_per_s": 1e3 / ms,
                  "hbm_gbs": k * 12 * total / (ms * 1e-3) / 1e9 if world == 1 else None})
            del opt, params
        ctx.close()

    # ---------------------------------------------------------------- C2 ----
    # ------------------------------------------------------ oracle timings ----
    # the CPU oracle (oracle/bf_oracle.c, single thread, as it stands) on the C1, C3
    # and C5 workloads -- a reported baseline (SURVEY 8(d) oracle timing protocol)
    if "oracle" in only and world == 1 and rank == 0:
        import time
        import oracle as ora

        def clock(fn, reps=3):
            fn()
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - t0)
            return sorted(ts)[len(ts) // 2]
        ncpu = len(os.sched_getaffinity(0))
        X1 = synthetic.agents_x0(4, 4096).astype(np.float64)
        W1 = ora.ring(4)

        def c1o():
            X = X1
            for _ in range(20):
                X = ora.mix(W1, X)
        t = clock(c1o)
        emit({"config": "oracle C1 ring-4 fp32[4096] x 20 iterations (fp64, 1 thread)", "s": t,
              "us_per_iteration": t / 20 * 1e6, "cores": 1, "nproc": ncpu})
        W8 = ora.exp2(8)
        for nb in (1 << 20, 1 << 26):
            X3 = synthetic.agents_x0(8, nb // 4).astype(np.float64)
            t = clock(lambda: ora.mix(W8, X3), reps=1 if nb > (1 << 22) else 3)
            emit({"config": f"oracle C3 neighbor_allreduce exp-2, 8 agents x {nb} B fp32 (fp64, 1 thread)", "s": t,
                  "gbs_per_agent": nb / t / 1e9, "cores": 1, "nproc": ncpu})
        pre = 1 << 20
        X5 = np.concatenate([synthetic.agents_x0(8, pre).astype(np.float64), np.ones((8, 1))], axis=1)
        win = ora.Window(W8, X5, zero_init=True)
        rnd = [0]

        def c5o():
            k_ = rnd[0]
            for i in range(8):
                _, dst = ora.one_peer_exp2_peers(8, k_, i)
                win.accumulate(i, 0.5, {dst: 0.5})
            for i in range(8):
                win.collect(i)
            rnd[0] += 1
        t = clock(c5o)
        emit({"config": f"oracle C5 push-sum round (event model), 8 agents x {pre}-element prefix of 340M "
                        "(fp64, 1 thread)", "s": t, "s_per_round_extrapolated_to_340M": t * 340_000_000 / pre,
              "cores": 1, "nproc": ncpu})

    if "c2" in only and world == 1:
        import oracle as ora
        n, m, d = a.agents, 2000, 10_000
        As = torch.stack([torch.from_numpy(synthetic.uniform(synthetic.SEED_A + r, m * d,
                                                             scale=1.0 / np.sqrt(m)).reshape(m, d))
                          for r in range(n)]).cuda()
        xnat = torch.from_numpy(synthetic.uniform(synthetic.SEED_XNAT, d)).cuda()
        bs = torch.stack([As[r] @ xnat + torch.from_numpy(synthetic.uniform(synthetic.SEED_NOISE + r, m,
                                                                            scale=0.01)).cuda()
                          for r in range(n)])
        L = max(float(torch.linalg.matrix_norm(As[r], ord=2) ** 2) for r in range(n))
        lr = 1.0 / L
        ctx = bfp.Context(agents_per_proc=n, heap_bytes=64 << 20, device=local)
        x = torch.zeros(n, d, device="cuda")
        g = torch.empty_like(x)
        # Exact-Diffusion on the ring (the paper's Listing ED-static; ED assumes a symmetric W --
        # on the directed exp-2 graph it diverges)
        for topo in ("exp2", "one_peer", "ring_exact_diffusion"):
            x.zero_()
            ed = topo == "exp2_exact_diffusion"
            psi = torch.zeros_like(x) if ed else None
            if topo == "ring_exact_diffusion":
                ctx.set_topology(bfp.topology_matrix("ring", n))
            elif topo == "exp2":
                ctx.set_topology(bfp.topology_matrix("exp2", n))
            else:
                ctx.set_dynamic_schedule("one_peer_exp2", 0)

            def step():
                r_ = torch.bmm(As, x.unsqueeze(2)).squeeze(2) - bs
                torch.bmm(As.transpose(1, 2), r_.unsqueeze(2), out=g.unsqueeze(2))
                if ed:
                    ctx.exact_diffusion_step(x, g, psi, lr)
                else:
                    ctx.atc_step(x, g, lr)
            ms = timed(step, 200, warm=0)
            ctx.set_dynamic_schedule("none")
            xs, _ = ora.lsq_solve(As.double().cpu().numpy(), bs.double().cpu().numpy(), tol=1e-10, max_iter=500)
            xbar = x.double().mean(0).cpu().numpy()
            emit({"config": f"C2 ATC-DSGD least squares d=10k m=2000 x 8 agents, {topo}", "ms_per_iter": ms,
                  "iters_per_s": 1e3 / ms, "rel_dist_to_xstar_after_203_iters":
                      float(np.linalg.norm(xbar - xs) / np.linalg.norm(xs)),
                  "consensus_residual": float((x.double() - x.double().mean(0)).abs().max())})
        ctx.close()

    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
