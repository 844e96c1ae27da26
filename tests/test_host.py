"""CPU tests of the C-ABI library's host side (no GPU compute calls):
exported symbols vs include/*.h, host topology builders and the one-peer
schedule against the oracle, error reporting, and the N>1 bootstrap
plumbing on a world_size-2 gloo group.
"""
import ctypes as C
import glob
import os
import re
import socket

import numpy as np
import pytest
import torch

import oracle as ora
import paper_2111_04287_b200 as bfp
from paper_2111_04287_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(bf_[a-z0-9_]+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol():
    declared = _declared_symbols()
    assert len(declared) >= 30
    lib = C.CDLL(_lib.SO_PATH)
    missing = [n for n in sorted(declared) if not hasattr(lib, n)]
    assert not missing, missing
    # the ctypes binding declares exactly the header's functions
    assert set(_lib._SIGS) == declared


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.SO_PATH} 2>&1").read()
    assert "sm_100a" in out


@pytest.mark.parametrize("kind", ["ring", "exp2", "full"])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8, 16])
def test_host_topologies_match_oracle(kind, n):
    ref = {"ring": ora.ring, "exp2": ora.exp2, "full": ora.full}[kind](n)
    assert np.array_equal(bfp.topology_matrix(kind, n), ref)


@pytest.mark.parametrize("n", [2, 3, 5, 8, 16])
def test_host_one_peer_schedule_matches_oracle(n):
    for k in range(7):
        assert np.array_equal(bfp.topology_matrix("one_peer_exp2", n, k), ora.one_peer_exp2(n, k))
        for i in range(n):
            assert bfp.one_peer_exp2(n, i, k) == ora.one_peer_exp2_peers(n, k, i)


@pytest.mark.parametrize("n,L", [(8, 4), (8, 2), (12, 3), (16, 8), (6, 1), (8, 8)])
def test_host_inner_outer_schedule_matches_oracle(n, L):
    # the library's sched_peers (host side of the device evaluation) vs the oracle (R27)
    for k in range(3 * n):
        for i in range(n):
            assert bfp.inner_outer_exp2(n, L, i, k) == ora.inner_outer_exp2_peers(n, L, k, i)
    for bad_n, bad_L in ((n, 0), (n + 1, 2 * L) if L < n else (n, n + 1)):
        with pytest.raises(bfp.BluefogError):
            bfp.inner_outer_exp2(bad_n, bad_L, 0, 0)


def test_status_strings_and_errors():
    lib = _lib.load()
    assert lib.bf_status_string(3) == b"BF_ERR_TOPOLOGY"
    W = np.zeros(4)
    assert lib.bf_topology_matrix(9, 2, 0, W.ctypes.data_as(C.POINTER(C.c_double))) == 1
    with pytest.raises(_lib.BluefogError) as e:
        _lib.check(1)
    assert e.value.name == "BF_ERR_ARG"


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_init_without_gpu_fails_loudly():
    with pytest.raises(_lib.BluefogError) as e:
        bfp.Context(agents_per_proc=1, heap_bytes=1 << 26)
    assert e.value.name in ("BF_ERR_CUDA", "BF_ERR_UNSUPPORTED")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2111_04287_b200.api import _allgather_bytes
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blob = bytes([rank]) * _lib.load().bf_ipc_blob_size()
    blobs = _allgather_bytes(blob)
    # bench.py's max-over-ranks timing reduction
    t = torch.tensor([1.5 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.destroy_process_group()
    q.put((rank, [b[0] for b in blobs], [len(b) for b in blobs], float(t)))


def test_bootstrap_allgather_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(60)
    size = _lib.load().bf_ipc_blob_size()
    for rank, firsts, lens, tmax in res:
        assert firsts == [0, 1] and lens == [size, size]
        assert tmax == 2.5


# ------------------------------------------------ optimizer wrapper (host logic) ---
def test_plan_buckets_reverse_order_no_split():
    from paper_2111_04287_b200.optim import plan_buckets
    numels = [5, 3, 8, 2, 20, 1]
    b = plan_buckets(numels, 10)
    # reverse registration order (backward produces the last layer first)
    assert [i for bb in b for i in bb] == list(reversed(range(len(numels))))
    for bb in b:   # a bucket only exceeds the target when one tensor alone does
        assert sum(numels[i] for i in bb) <= 10 or len(bb) == 1
    assert b == [[5], [4], [3, 2], [1, 0]]


def test_resnet50_shapes():
    import math
    from paper_2111_04287_b200.optim import resnet50_param_shapes
    s = resnet50_param_shapes()
    # torchvision ResNet-50: 161 parameter tensors, 25 557 032 parameters (the model of P:892)
    assert len(s) == 161 and sum(math.prod(x) for x in s) == 25_557_032


def _run_bench(args, env_extra=None):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, **(env_extra or {}))
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py")] + args, cwd=root, env=env,
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    return [json.loads(l) for l in lines]


def test_bench_reference_arm_contract():
    """--impl reference: one JSON line in the same metric/unit as our arm, oracle timed on the host."""
    (d,) = _run_bench(["--impl", "reference", "--steps", "1", "--warmup", "3"])
    assert d["impl"] == "reference" and d["unit"] == "iters/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "iters/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("C4")


def test_bench_reference_arm_nonzero_rank_is_silent():
    """Under torchrun only rank 0 runs the reference arm; other ranks exit 0 without output."""
    assert _run_bench(["--impl", "reference", "--steps", "1", "--warmup", "3", "--gpus", "2"],
                      {"RANK": "1", "WORLD_SIZE": "2"}) == []
