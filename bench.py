#!/usr/bin/env python
"""Benchmark of the BlueFog hot path on B200 (one JSON line on rank 0).

Workload (BASELINE.json configs[3], "C4"): one fused ATC-DSGD step
(Eq. 4-5 + Eq. 17) of n = 8 agents, each holding a 25.6M-element fp32
parameter vector (ResNet-50-sized), synthetic gradients, dynamic one-peer
exponential-2 topology.  A "step" = one pass of the whole hot path:
weight/schedule resolution, adapt, publish, neighbour exchange, weighted
combine, store -- one kernel launch per step.

  N = 1 : the 8 agents run as virtual agents on one GPU (HBM-bound)
  N > 1 : 8/N agents per GPU, neighbours on other GPUs read over NVLink
          through CUDA-IPC peer pointers (strong scaling: total work fixed)

Launch:  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
         (N > 1 through torch.distributed.run, one rank per GPU)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "neighbor_allreduce GB/s/GPU + ATC-DSGD iters/s at 1/2/4/8 B200, % of roofline"
NVLINK_PEAK_GBS = 770.0      # B200_PROFILING.md: measured peer copy per direction (the roofline denominator)
NVLINK_NOMINAL_GBS = 900.0   # north_star / B200_PROFILING.md nominal per direction (context)
NVLINK_BIDIR_GBS = 680.0     # profiles/r01_nvlink_calibration.md: per-GPU pull/push with both directions busy (context)
HBM_FALLBACK_GBS = 6650.0    # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--agents", type=int, default=8)
    ap.add_argument("--count", type=int, default=25_600_000)
    ap.add_argument("--topology", choices=["one_peer", "exp2", "self"], default="one_peer")
    ap.add_argument("--wire", choices=["fp32", "bf16"], default="fp32")
    ap.add_argument("--lr", type=float, default=0.1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-nar", action="store_true", help="skip the C3 1 GiB neighbor_allreduce line")
    ap.add_argument("--nar-bytes", type=int, default=1 << 30, help="bytes per agent of the C3 call")
    return ap.parse_args()


def host_cpu():
    """(model name, logical CPUs usable by this process) of the box's host."""
    model = "unknown"
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        ncpu = len(os.sched_getaffinity(0))
    except Exception:
        ncpu = os.cpu_count() or 1
    return model, ncpu


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


def degree(topology, n):
    if n == 1 or topology == "self":
        return 0
    if topology == "one_peer":
        return 1
    d, off = 0, 1
    while off <= n - 1:
        d += 1
        off *= 2
    return d


def workload_name(a):
    return (f"C4: ATC-DSGD step (fused adapt+exchange+combine), {a.agents} agents x {a.count} fp32 "
            f"(ResNet-50-sized), {'dynamic one-peer exp-2' if a.topology == 'one_peer' else 'static exp-2'} "
            f"topology, {a.wire} wire, synthetic gradients")


# ---------------------------------------------------------------- clocks ----
class Clocks:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", delete=False, suffix=".csv")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", "--query-gpu=" + ",".join(self.FIELDS),
                                       "--format=csv,noheader,nounits", "-lms", "20"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.05)
        self.p.terminate()
        try:
            self.p.wait(5)
        except Exception:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        for line in self.f.read().splitlines():
            parts = [s.strip() for s in line.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        os.unlink(self.f.name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ CPU oracle ----
def oracle_step_rate(a, budget_s=12.0, prefix=1 << 20, threads=1):
    """Time the oracle (oracle/bf_oracle.c, as it stands) on a bounded prefix
    sample of the same workload.  threads > 1: the prefix is split into column
    slices, one thread per slice, each calling the same single-threaded oracle
    function (the step is column-wise; ctypes releases the GIL), so `threads`
    host cores work.  Returns (iters/s extrapolated to the full count, sample
    description, seconds spent, measured seconds per prefix step, factor)."""
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    import oracle as ora
    import synthetic
    n = a.agents
    X = synthetic.agents_x0(n, prefix).astype(np.float64)
    G = synthetic.agents_grad(n, prefix, 0).astype(np.float64)
    Wk = [ora.one_peer_exp2(n, k) if a.topology == "one_peer" else ora.exp2(n) for k in range(3)]
    bounds = np.linspace(0, prefix, threads + 1).astype(int)
    Xs = [np.ascontiguousarray(X[:, lo:hi]) for lo, hi in zip(bounds[:-1], bounds[1:])]
    Gs = [np.ascontiguousarray(G[:, lo:hi]) for lo, hi in zip(bounds[:-1], bounds[1:])]
    pool = ThreadPoolExecutor(threads) if threads > 1 else None
    t0 = time.perf_counter()
    steps = 0
    while True:
        W = Wk[steps % 3]
        f = lambda i: ora.atc(W, Xs[i], Gs[i], a.lr, wire_bf16=(a.wire == "bf16"))
        Xs = list(pool.map(f, range(threads))) if pool else [f(0)]
        steps += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    if pool:
        pool.shutdown()
    per_prefix = el / steps
    factor = a.count / prefix
    sample = (f"{steps} oracle ATC steps on a {prefix}-element prefix of each of the {n} agents "
              f"({el:.1f} s, {per_prefix * 1e3:.1f} ms per prefix step, {threads} thread(s) on column slices), "
              f"time scaled linearly by {factor:.2f} to {a.count} elements")
    return 1.0 / (per_prefix * factor), sample, el, per_prefix, factor


def run_reference(a):
    """--impl reference: the oracle (CPU) as it stands, same metric/unit."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np

    import oracle as ora
    import synthetic
    n, prefix = a.agents, 1 << 19
    X = synthetic.agents_x0(n, prefix).astype(np.float64)
    G = synthetic.agents_grad(n, prefix, 0).astype(np.float64)
    Wk = [ora.one_peer_exp2(n, k) if a.topology == "one_peer" else ora.exp2(n) for k in range(3)]
    for s in range(a.warmup):
        X = ora.atc(Wk[s % 3], X, G, a.lr, wire_bf16=(a.wire == "bf16"))
    t0 = time.perf_counter()
    for s in range(a.steps):
        X = ora.atc(Wk[s % 3], X, G, a.lr, wire_bf16=(a.wire == "bf16"))
    el = time.perf_counter() - t0
    factor = a.count / prefix
    ms_prefix = el / a.steps * 1e3
    ms_full = ms_prefix * factor
    value = 1e3 / ms_full
    model, ncpu = host_cpu()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_full, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(a), "agents": n, "count": a.count, "topology": a.topology,
                   "wire": a.wire},
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": 1, "kind": "oracle",
                         "cpu_model": model, "nproc": ncpu,
                         "sample": f"each step = one oracle ATC step on a {prefix}-element prefix of each agent, "
                                   f"time scaled linearly to {a.count} elements",
                         "measured_ms_per_prefix_step": ms_prefix, "extrapolation_factor": factor},
        "timing": "ms_per_step is the measured prefix time x extrapolation_factor (not timed at full size)",
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def nar_line(a, ctx, k, world, nar_count, ms, nsteps, rounds, peak_hbm, peak_kind, sources, dests):
    """C3 neighbor_allreduce GB/s/GPU: algorithmic NVLink-in bytes
    d_in_remote x M per second at N > 1; at N = 1 (every neighbour on the same GPU,
    combined in registers) the algorithmic HBM bytes (read x + write y) per second."""
    M = nar_count * 4
    rounds = rounds if a.topology == "one_peer" else [0]
    rem = statistics.mean(len({j for la in range(k) for j in sources(ctx.rank + la, r) if j // k != ctx.proc})
                          for r in rounds)
    pub = statistics.mean(sum(1 for la in range(k) if any(j // k != ctx.proc for j in dests(ctx.rank + la, r)))
                          for r in rounds)
    hbm = k * 2 * M + pub * M
    nvl = rem * M
    t = ms * 1e-3
    out = {"bytes_per_agent": M, "dtype": "fp32", "topology": a.topology, "ms_per_call": ms, "calls": nsteps,
           "hbm_gbs": hbm / t / 1e9, "nvlink_in_gbs_per_gpu": nvl / t / 1e9}
    if world == 1 or nvl == 0:
        out["gbs_per_gpu"] = out["hbm_gbs"]
        out["gbs_definition"] = "N = 1: algorithmic HBM bytes (read x + write y) per second"
        out["frac_of_hbm_peak"] = out["hbm_gbs"] / peak_hbm
        out["peak"] = f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"
    else:
        out["gbs_per_gpu"] = out["nvlink_in_gbs_per_gpu"]
        out["gbs_definition"] = "algorithmic NVLink-in bytes (distinct remote in-neighbours of the local agents x M) per second"
        out["frac_of_nvlink_770"] = out["gbs_per_gpu"] / NVLINK_PEAK_GBS
        out["frac_of_nominal_900"] = out["gbs_per_gpu"] / NVLINK_NOMINAL_GBS
        out["frac_of_bidir_680"] = out["gbs_per_gpu"] / NVLINK_BIDIR_GBS
    return out


# ----------------------------------------------------------------- ours -----
def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BF_BENCH_SHARE_GPUS=G (diagnostic, never a bench number): rank r on GPU r mod G with a
    # gloo bootstrap -- runs the N-process flow (e.g. N = 8) on a box with fewer GPUs
    share = int(os.environ.get("BF_BENCH_SHARE_GPUS", "0"))
    if share:
        local = local % share
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if a.agents % world:
        raise SystemExit(f"{a.agents} agents do not split over {world} GPUs")
    k = a.agents // world
    import paper_2111_04287_b200 as bfp
    import synthetic

    count = a.count
    wire_dt = torch.float32 if a.wire == "fp32" else torch.bfloat16
    wire_b = 4 if a.wire == "fp32" else 2
    # exchange slots (k agents x 2 parities) + across GPUs the push inboxes (n agents x 2 parities)
    nar_count = 0 if a.no_nar else a.nar_bytes // 4
    heap = (k + (a.agents if world > 1 else 0)) * 2 * max(count * wire_b, nar_count * 4) + (64 << 20)
    ctx = bfp.Context(agents_per_proc=k, heap_bytes=heap, device=local)
    n = ctx.n
    if a.topology == "one_peer":
        ctx.set_dynamic_schedule("one_peer_exp2", 0)
    elif a.topology == "self":      # diagnostic: W = I, no neighbour traffic
        import numpy as np
        ctx.set_topology(np.eye(n))
    else:
        ctx.set_topology(bfp.topology_matrix("exp2", n))
    ctx.reserve(count * wire_b)

    x = torch.empty(k, count, device="cuda")
    gs = [torch.empty(k, count, device="cuda") for _ in range(2)]
    for la in range(k):
        gid = ctx.rank + la
        bfp.Context.fill_uniform(x[la], synthetic.SEED_X0 + gid)
        for s, g in enumerate(gs):
            bfp.Context.fill_uniform(g[la], synthetic.grad_seed(s, gid), scale=2.0 ** -7)
    torch.cuda.synchronize()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = Clocks(local)
    for s in range(a.warmup):
        ctx.atc_step(x, gs[s % 2], a.lr, wire=wire_dt)
    barrier()
    stream = torch.cuda.current_stream()
    l0 = ctx.kernel_launches()
    t_begin = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    # the timed region: K back-to-back steps, no event between them
    t_begin.record(stream)
    for s in range(a.steps):
        ctx.atc_step(x, gs[s % 2], a.lr, wire=wire_dt)
    t_end.record(stream)
    barrier()
    launches = ctx.kernel_launches() - l0
    total_ms = t_begin.elapsed_time(t_end)
    kern_ms = total_ms / a.steps   # one launch per step: the kernel's average launch duration
    # per-round detail (diagnostic, after the timed region): one-peer rotates through
    # tau = ceil(log2 n) graphs; each step bracketed by its own events
    tau_r = max(1, (ctx.n - 1).bit_length()) if a.topology == "one_peer" else 1
    n_diag = max(tau_r * 3, min(a.steps, 48) // tau_r * tau_r, 3)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(n_diag)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(n_diag)]
    for s in range(n_diag):
        starts[s].record(stream)
        ctx.atc_step(x, gs[s % 2], a.lr, wire=wire_dt)
        ends[s].record(stream)
    barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    srt = sorted(step_ms)
    step_stats = [statistics.median(step_ms), srt[0], srt[min(len(srt) - 1, int(0.9 * len(srt)))]]
    r_diag0 = a.warmup + a.steps
    by_round = [statistics.mean(step_ms[i] for i in range(n_diag) if (r_diag0 + i) % tau_r == r)
                for r in range(tau_r)]
    ctx.poll_error()

    # ---- end to end through the public API: host gradients in, sample out ----
    e2e = None
    if not a.no_e2e:
        gh = [g.cpu().pin_memory() for g in gs]
        sample = torch.empty(k, 1024, dtype=torch.float32).pin_memory()
        for s in range(2):
            ctx.atc_step(x, gh[s % 2], a.lr, wire=wire_dt)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(a.steps):
            ctx.atc_step(x, gh[s % 2], a.lr, wire=wire_dt)
            sample.copy_(x[:, :1024], non_blocking=True)
        e1.record(stream)
        barrier()
        e2e_ms = e0.elapsed_time(e1) / a.steps
        e2e = {"ms": e2e_ms, "h2d": k * count * 4, "d2h": k * 1024 * 4}
    # ---- C3 (BASELINE.json configs[2]): one neighbor_allreduce call at 1 GiB fp32 per
    # agent on the same topology, timed on the device like the step ----
    nar = None
    if nar_count:
        del gs
        xn = torch.empty(k, nar_count, device="cuda")
        for la in range(k):
            bfp.Context.fill_uniform(xn[la], synthetic.SEED_X0 + 100 + ctx.rank + la)
        yn = torch.empty_like(xn)
        nsteps = max(3, min(a.steps, 20))
        for _ in range(3):
            ctx.neighbor_allreduce(xn, out=yn)
        barrier()
        n0 = torch.cuda.Event(enable_timing=True)
        n1 = torch.cuda.Event(enable_timing=True)
        n0.record(stream)
        for _ in range(nsteps):
            ctx.neighbor_allreduce(xn, out=yn)
        n1.record(stream)
        barrier()
        # schedule rounds of the timed calls (every schedule-mode call advances the round)
        r0 = a.warmup + a.steps + n_diag + (0 if a.no_e2e else 2 + a.steps) + 3
        nar = {"ms": n0.elapsed_time(n1) / nsteps, "steps": nsteps, "rounds": range(r0, r0 + nsteps)}
        del xn, yn
    clk = clocks.stop()
    ctx.poll_error()

    # ---- max over ranks ----
    vals = torch.tensor([total_ms / a.steps, kern_ms, e2e["ms"] if e2e else 0.0, nar["ms"] if nar else 0.0]
                        + step_stats + by_round, dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    vals = [float(v) for v in vals.cpu()]
    ms_step, ms_kern, ms_e2e, ms_nar = vals[:4]
    ms_med, ms_min, ms_p90 = vals[4:7]
    ms_by_round = vals[7:]

    if rank == 0:
        d = degree(a.topology, n)
        # algorithmic bytes per launch on this GPU, for the
        # default local-agent fused kernel: every local agent reads x and g and
        # writes x (12 B per element); an agent whose x_half is read by another
        # process also publishes its wire copy (w B per element).  Local sources
        # are combined in registers, remote sources cross NVLink (d_in remote x w).
        tau = max(1, (n - 1).bit_length())
        rounds = range(a.warmup, a.warmup + a.steps)   # the schedule rounds of the timed steps

        def sources(gid, r):
            if n == 1 or a.topology == "self":
                return []
            if a.topology == "one_peer":
                return [(gid - (1 << (r % tau))) % n]
            return [(gid - (1 << j)) % n for j in range(d)]

        def dests(gid, r):
            if n == 1 or a.topology == "self":
                return []
            if a.topology == "one_peer":
                return [(gid + (1 << (r % tau))) % n]
            return [(gid + (1 << j)) % n for j in range(d)]

        peak_hbm, peak_kind = hbm_peak()
        remote, publishers, t_roof = 0.0, 0.0, 0.0
        roof_by_round = {}
        for r in rounds:
            # distinct remote source agents: one copy per GPU is what the method must move
            rem_r = len({sidx for la in range(k) for sidx in sources(ctx.rank + la, r) if sidx // k != ctx.proc})
            pub_r = sum(1 for la in range(k) if any(didx // k != ctx.proc for didx in dests(ctx.rank + la, r)))
            remote += rem_r / len(rounds)
            publishers += pub_r / len(rounds)
            # per-round roofline time: the slower of HBM and NVLink-in for this round's graph
            t_r = max((k * 12 + pub_r * wire_b) * count / (peak_hbm * 1e9),
                      rem_r * count * wire_b / (NVLINK_PEAK_GBS * 1e9))
            t_roof += t_r / len(rounds)
            roof_by_round[r % tau_r] = t_r
        hbm_bytes = k * count * (4 + 4 + 4) + publishers * count * wire_b
        nvl_bytes = remote * count * wire_b
        t_hbm = hbm_bytes / (peak_hbm * 1e9)
        t_nvl = nvl_bytes / (NVLINK_PEAK_GBS * 1e9)
        if t_nvl > t_hbm:
            roof = {"bound": "nvlink", "achieved": nvl_bytes / (ms_kern * 1e-3) / 1e9, "peak": NVLINK_PEAK_GBS,
                    "unit": "GB/s", "peak_source": "B200_PROFILING.md measured peer copy per direction"}
        else:
            roof = {"bound": "hbm", "achieved": hbm_bytes / (ms_kern * 1e-3) / 1e9, "peak": peak_hbm,
                    "unit": "GB/s", "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"}
        roof["frac"] = roof["achieved"] / roof["peak"]
        # one-peer rounds alternate between HBM- and NVLink-bound on N > 1: the
        # mean over rounds of max(HBM time, NVLink time) at the peaks, / measured
        roof["t_roof_ms"] = t_roof * 1e3
        roof["frac_per_round_bound"] = t_roof * 1e3 / ms_kern
        roof["by_round"] = [{"ms": m, "t_roof_ms": roof_by_round.get(r, 0.0) * 1e3,
                             "frac": roof_by_round.get(r, 0.0) * 1e3 / m if m > 0 else None}
                            for r, m in enumerate(ms_by_round)]
        roof["by_round_note"] = "per-round times from separate event-bracketed steps after the timed region"
        roof["step_ms_event_bracketed"] = {"median": ms_med, "min": ms_min, "p90": ms_p90, "steps": n_diag}
        # every schedule round of the timed steps is one roofline class: one-peer with
        # tau graphs needs steps >= tau for every class to be present
        roof["traffic"] = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            try:
                with open(tp) as f:
                    tj = json.load(f)
                # ncu DRAM bytes per launch: N = 1 from a --set full capture, N > 1 from the
                # one-rank capture of scripts/ncu_nvlink.py (profiles/r02_ncu_multirank_n2.md)
                key = f"{a.topology}_{a.wire}_n{world}"
                roof["traffic"] = tj.get(f"{key}_a{n}", tj.get(key))
            except Exception:
                pass
        roof["algorithmic_bytes_per_launch"] = hbm_bytes if roof["bound"] == "hbm" else nvl_bytes
        if world == 1:
            roof["kernel"] = "bf::exchange_fused_kernel (ATC adapt + combine of the 8 local agents in registers)"
        elif k <= 2 or a.topology != "one_peer":
            roof["kernel"] = ("bf::exchange_push_kernel (ATC adapt, wire copies stored into the readers' inboxes "
                              "over NVLink, local part parked in shared memory, remote terms from the local inbox)")
        else:
            roof["kernel"] = ("bf::exchange_fused_kernel, pull path (publish into the own slot, TMA pulls of the "
                              "remote sources over NVLink; K = 4 schedules)")
        value = 1e3 / ms_step
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(a), "agents": n, "agents_per_gpu": k, "count": count,
                       "topology": a.topology, "wire": a.wire, "lr": a.lr,
                       "l2": "inputs larger than L2 (x, 2 rotating gradient sets: "
                             f"{3 * n * count * 4 / 1e9:.2f} GB)"},
            "gpu_launches": launches,
            "roofline": roof,
            **({"diagnostic": f"BF_BENCH_SHARE_GPUS={share}: {world} processes time-share {share} GPUs; "
                              "not a measurement"} if share else {}),
            "clocks": clk,
        }
        if e2e:
            line["e2e"] = {"value": 1e3 / ms_e2e, "unit": "iters/s", "h2d_bytes_per_step": e2e["h2d"] * world,
                           "d2h_bytes_per_step": e2e["d2h"] * world,
                           "path": "Context.atc_step with pinned host gradients (H2D inside the C-ABI call) "
                                   "+ D2H of 1024 elements per agent"}
        if nar:
            line["neighbor_allreduce"] = nar_line(a, ctx, k, world, nar_count, ms_nar, nar["steps"], nar["rounds"],
                                                  peak_hbm, peak_kind, sources, dests)
            line["neighbor_allreduce_gbs_per_gpu"] = line["neighbor_allreduce"]["gbs_per_gpu"]
        if world > 1:
            roof["frac_of_nominal_900"] = (roof["achieved"] / NVLINK_NOMINAL_GBS if roof["bound"] == "nvlink"
                                           else None)
            roof["frac_of_bidir_680"] = (roof["achieved"] / NVLINK_BIDIR_GBS if roof["bound"] == "nvlink"
                                         else None)
        if world == 1 and not a.no_cpu:
            model, ncpu = host_cpu()
            v, sample, el, per_prefix, factor = oracle_step_rate(a)
            line["cpu_baseline"] = {"value": v, "unit": "iters/s", "cores": 1, "kind": "oracle", "sample": sample,
                                    "cpu_model": model, "nproc": ncpu,
                                    "measured_ms_per_prefix_step": per_prefix * 1e3, "extrapolation_factor": factor}
            thr = min(a.agents, ncpu)
            if thr > 1:
                v2, sample2, _, pp2, _ = oracle_step_rate(a, budget_s=8.0, threads=thr)
                line["cpu_baseline_threads"] = {"value": v2, "unit": "iters/s", "cores": thr, "kind": "oracle",
                                                "sample": sample2, "measured_ms_per_prefix_step": pp2 * 1e3}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
