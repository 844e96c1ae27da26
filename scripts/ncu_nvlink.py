#!/usr/bin/env python
"""NVLink bytes of the cross-GPU exchange kernel from ncu's own counters
(nvlrx__bytes / nvltx__bytes, per GPU), without wrapping a multi-rank job in ncu.

Only rank 0's process runs under ncu, with a metric list that fits one pass
(no kernel replay: a replayed exchange kernel would wait for peers that have
moved on); the other ranks run plain.  ncu on the gpurun boxes first runs the
profiled command once without ncu, so the plain ranks serve sessions in a loop
(one process-group rendezvous per session on the same port) until rank 0 is
done, then this launcher stops them by PID.

  python scripts/ncu_nvlink.py --gpus 2 --agents 2 --topo one_peer --out gpurun_out/nvl_n2_k1
"""
import argparse
import os
import subprocess
import sys
import time

METRICS = {   # two small sets, each meant to fit one pass
    "nvl": "gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,"
           "nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum",
    "dram": "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum",
    # warp stall counters (why the consumers of the cross-GPU kernels are slower than local streaming):
    # like the NVLink counters they answer UnknownError in the one-rank capture on the gpurun boxes
    "stall1": "gpu__time_duration.sum,smsp__warps_active.sum,smsp__warps_issue_stalled_long_scoreboard.sum,"
              "smsp__warps_issue_stalled_lg_throttle.sum,smsp__warps_issue_stalled_membar.sum,"
              "smsp__warps_issue_stalled_sleeping.sum",
    "stall2": "gpu__time_duration.sum,smsp__warps_issue_stalled_barrier.sum,smsp__warps_issue_stalled_drain.sum,"
              "smsp__warps_issue_stalled_short_scoreboard.sum,smsp__warps_issue_stalled_mio_throttle.sum,"
              "smsp__warps_issue_stalled_wait.sum,smsp__warps_issue_stalled_selected.sum",
}
HERE = os.path.dirname(os.path.abspath(__file__))


def rank_main(a):
    """One rank: `sessions` rendezvous, each W + S fused ATC steps."""
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(HERE))
    import paper_2111_04287_b200 as bfp
    import synthetic
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    for _ in range(a.sessions):
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        world = dist.get_world_size()
        k = a.agents // world
        count = a.count
        heap = (k + a.agents) * 2 * count * 4 + (64 << 20)
        ctx = bfp.Context(agents_per_proc=k, heap_bytes=heap, device=local)
        if a.topo == "one_peer":
            ctx.set_dynamic_schedule("one_peer_exp2", 0)
        else:
            ctx.set_topology(bfp.topology_matrix("exp2", ctx.n))
        x = torch.empty(k, count, device="cuda")
        g = torch.empty(k, count, device="cuda")
        for la in range(k):
            bfp.Context.fill_uniform(x[la], synthetic.SEED_X0 + ctx.rank + la)
            bfp.Context.fill_uniform(g[la], synthetic.grad_seed(0, ctx.rank + la), scale=2.0 ** -7)
        for _ in range(a.warmup + a.steps):
            ctx.atc_step(x, g, 0.1)
        torch.cuda.synchronize()
        dist.barrier()
        ctx.close()
        dist.destroy_process_group()
        print(f"rank {dist_rank()} session done", flush=True)


def dist_rank():
    return int(os.environ.get("RANK", "0"))


def launcher(a):
    base = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(a.port), WORLD_SIZE=str(a.gpus),
                BF_TIMEOUT_MS=str(a.timeout_ms))
    me = [sys.executable, os.path.abspath(__file__), "--rank-main", "--agents", str(a.agents), "--topo", a.topo,
          "--count", str(a.count), "--warmup", str(a.warmup), "--steps", str(a.steps)]
    plain = []
    for r in range(1, a.gpus):
        env = dict(base, RANK=str(r), LOCAL_RANK=str(r))
        plain.append(subprocess.Popen(me + ["--sessions", "2"], env=env,
                                      stdout=open(f"{a.out}_rank{r}.log", "w"), stderr=subprocess.STDOUT))
    env0 = dict(base, RANK="0", LOCAL_RANK="0")
    # launches of the exchange kernel: skip the warm-up ones, profile 3
    cmd = ["ncu", "--metrics", METRICS[a.metrics], "--clock-control", "none", "-k",
           "regex:exchange_(push|fused|ll)_kernel", "-s", str(a.warmup), "-c", "3", "--csv",
           "--log-file", f"{a.out}.csv"] + me + ["--sessions", "1"]
    t0 = time.time()
    try:
        rc = subprocess.run(cmd, env=env0, timeout=a.wall).returncode
    except subprocess.TimeoutExpired:
        rc = 124
    print(f"ncu rank 0 rc={rc} in {time.time() - t0:.1f}s", flush=True)
    for p in plain:
        try:
            p.wait(timeout=60)
        except subprocess.TimeoutExpired:
            p.kill()
            p.wait()
    return rc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--agents", type=int, default=2)
    ap.add_argument("--topo", default="one_peer")
    ap.add_argument("--count", type=int, default=25_600_000)
    ap.add_argument("--warmup", type=int, default=6)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--sessions", type=int, default=1)
    ap.add_argument("--port", type=int, default=29561)
    ap.add_argument("--timeout-ms", type=int, default=30000)
    ap.add_argument("--wall", type=int, default=600)
    ap.add_argument("--out", default="gpurun_out/nvl")
    ap.add_argument("--metrics", default="nvl", choices=sorted(METRICS))
    ap.add_argument("--rank-main", action="store_true")
    a = ap.parse_args()
    if a.rank_main:
        rank_main(a)
    else:
        sys.exit(launcher(a))


if __name__ == "__main__":
    main()
