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
    """{gpu: {"tx": bytes, "rx": bytes}}: NVML NVLink data-throughput counters
    (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX, cumulative KiB, all links), else
    the per-link `nvidia-smi nvlink -gt d` text; plus a note of the source."""
    res, note = {}, ""
    try:
        import pynvml as nv
        nv.nvmlInit()
        for gi in range(nv.nvmlDeviceGetCount()):
            h = nv.nvmlDeviceGetHandleByIndex(gi)
            tx = rx = 0
            vals = nv.nvmlDeviceGetFieldValues(h, [(nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, 0xFFFFFFFF),
                                                   (nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 0xFFFFFFFF)])
            if all(v.nvmlReturn == 0 for v in vals):
                tx, rx = vals[0].value.ullVal * 1024, vals[1].value.ullVal * 1024
                note = "nvml data throughput, all links"
            else:   # per link
                for link in range(18):
                    v = nv.nvmlDeviceGetFieldValues(h, [(nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, link),
                                                        (nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, link)])
                    if v[0].nvmlReturn == 0:
                        tx += v[0].value.ullVal * 1024
                    if v[1].nvmlReturn == 0:
                        rx += v[1].value.ullVal * 1024
                note = f"nvml data throughput per link (rc {vals[0].nvmlReturn}, {vals[1].nvmlReturn} for all links)"
            res[gi] = {"tx": tx, "rx": rx}
        return res, note
    except Exception as ex:   # noqa: BLE001
        note = f"nvml failed: {ex!r}"
    out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d"], capture_output=True, text=True).stdout
    gpu = None
    for line in out.splitlines():
        m = re.match(r"GPU\s+(\d+):", line.strip())
        if m:
            gpu = int(m.group(1))
            res[gpu] = {"tx": 0, "rx": 0}
            continue
        m = PAT.search(line)
        if m and gpu is not None:
            res[gpu]["tx" if m.group(2) == "Tx" else "rx"] += int(m.group(3)) * 1024
    return res, note + " | nvidia-smi nvlink -gt d"


class Gpm:
    """NVLink RX/TX bytes of every GPU between start() and stop(), from the GPM
    (GPU performance monitoring) counters: NVML_GPM_METRIC_NVLINK_TOTAL_RX/TX_PER_SEC
    (MiB/s averaged between two samples) x the host-timed interval."""

    def __init__(self):
        import pynvml as nv
        nv.nvmlInit()
        self.nv = nv
        self.h = [nv.nvmlDeviceGetHandleByIndex(i) for i in range(nv.nvmlDeviceGetCount())]
        self.s0 = [nv.nvmlGpmSampleAlloc() for _ in self.h]
        self.s1 = [nv.nvmlGpmSampleAlloc() for _ in self.h]

    def start(self):
        import time
        for h, s in zip(self.h, self.s0):
            self.nv.nvmlGpmSampleGet(h, s)
        self.t0 = time.perf_counter()

    def stop(self):
        import time
        for h, s in zip(self.h, self.s1):
            self.nv.nvmlGpmSampleGet(h, s)
        dt = time.perf_counter() - self.t0
        out = {}
        for i, (a, b) in enumerate(zip(self.s0, self.s1)):
            mg = self.nv.c_nvmlGpmMetricsGet_t()
            mg.version = self.nv.NVML_GPM_METRICS_GET_VERSION
            mg.numMetrics = 2
            mg.sample1 = a
            mg.sample2 = b
            mg.metrics[0].metricId = self.nv.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC
            mg.metrics[1].metricId = self.nv.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC
            self.nv.nvmlGpmMetricsGet(mg)
            out[i] = {"rx": mg.metrics[0].value * 2 ** 20 * dt, "tx": mg.metrics[1].value * 2 ** 20 * dt,
                      "rc": [mg.metrics[0].nvmlReturn, mg.metrics[1].nvmlReturn], "seconds": dt}
        return out


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
    gpm = None
    if rank == 0:
        try:
            gpm = Gpm()
            gpm.start()
        except Exception as ex:   # noqa: BLE001
            gpm = repr(ex)
    c0, raw0 = counters() if rank == 0 else ({}, "")
    dist.barrier()
    for _ in range(steps):
        ctx.atc_step(x, g, 0.1)
    torch.cuda.synchronize()
    dist.barrier()
    c1, raw1 = counters() if rank == 0 else ({}, "")
    gres = None
    if rank == 0 and not isinstance(gpm, (str, type(None))):
        try:
            gres = gpm.stop()
        except Exception as ex:   # noqa: BLE001
            gres = repr(ex)
    elif rank == 0:
        gres = gpm
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
        res["counter_source"] = raw1
        if isinstance(gres, dict):
            res["gpm"] = {q: {"rx_bytes_per_step": v["rx"] / steps, "tx_bytes_per_step": v["tx"] / steps,
                              "rc": v["rc"], "interval_s": v["seconds"]} for q, v in gres.items() if q < world}
        else:
            res["gpm"] = gres
        print(json.dumps(res), flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
