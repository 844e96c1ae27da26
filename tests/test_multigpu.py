"""Multi-GPU parity: one process per GPU (torchrun), CUDA-IPC peer memory over
NVLink.  Needs >= 2 GPUs; skipped otherwise."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("nproc,k,hier", [(2, 1, "auto"), (2, 2, "auto"), (2, 4, "auto"), (2, 2, "fused"),
                                          (2, 3, "auto"), (4, 1, "auto"), (4, 2, "auto")])
def test_multiprocess_parity(nproc, k, hier):
    # hier="fused": the hierarchical calls take the Kronecker mix in the fused
    # kernel across GPUs (BF_HIER=fused) instead of the staged kernel
    if _ngpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    # BF_NVLS_MIN_P=2: the NVLS path also for machines of 2 processes (parity coverage)
    env = dict(os.environ, BF_TEST_K=str(k), BF_TIMEOUT_MS="8000", BF_HIER=hier, BF_NVLS_MIN_P="2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "mp_worker.py")]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-4000:]
    assert out.count("ALL OK") == nproc, out[-4000:]


@pytest.mark.parametrize("nproc,k", [(2, 1), (2, 2), (4, 1), (4, 2)])
def test_multiprocess_production_shape(nproc, k):
    # 25.6M fp32 per agent (the 8-GPU target's per-GPU shape at k = 1), every fused
    # op over consecutive rounds, windows with more items than CTAs (mp_worker_big.py)
    if _ngpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    env = dict(os.environ, BF_TEST_K=str(k), BF_TIMEOUT_MS="10000")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", "--master-port=29534", os.path.join(ROOT, "tests", "mp_worker_big.py")]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-4000:]
    assert out.count("ALL OK") == nproc, out[-4000:]


def test_eight_processes_time_shared():
    # the 8-GPU setting's process logic (8 processes, one agent each: push inboxes of 8
    # writers, one-peer over 8 agents, tagged words, windows, hierarchical) on the GPUs this
    # box has -- process p on GPU p mod G, time-sliced contexts, gloo bootstrap
    g = _ngpus()
    if g < 1:
        pytest.skip("needs a GPU")
    env = dict(os.environ, BF_TEST_K="1", BF_TIMEOUT_MS="20000", BF_TEST_SHARE_GPUS=str(min(g, 8)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr=127.0.0.1", "--master-port=29535", os.path.join(ROOT, "tests", "mp_worker.py")]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-4000:]
    assert out.count("ALL OK") == 8, out[-4000:]


def test_eight_processes_time_shared_production_shape():
    # the same at 25.6M fp32 per agent (the 8-GPU target's per-GPU shape): mp_worker_big.py
    g = _ngpus()
    if g < 1:
        pytest.skip("needs a GPU")
    env = dict(os.environ, BF_TEST_K="1", BF_TIMEOUT_MS="30000", BF_TEST_SHARE_GPUS=str(min(g, 8)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr=127.0.0.1", "--master-port=29536", os.path.join(ROOT, "tests", "mp_worker_big.py")]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=1200)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-4000:]
    assert out.count("ALL OK") == 8, out[-4000:]
