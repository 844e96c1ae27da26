"""Paper-style Python API over the C ABI (argument marshalling only).

Mirrors BlueFog's primitives: set_topology,
neighbor_allreduce (static, or dynamic with self/src/dst weights),
atc_step (the fused adapt-then-combine DSGD step), hierarchical_neighbor_allreduce,
win_create / win_put / win_accumulate / win_update / win_update_then_collect /
win_free, barrier.  PyTorch is used for device memory, streams and the
torch.distributed bootstrap only; every step of the path runs in the CUDA
kernels of libbluefog_b200.so.

Tensors hold the process's local agents stacked: shape (agents_per_proc, count)
(a 1-D tensor is accepted when agents_per_proc == 1).  Weight arguments follow
the paper: self_weight (float), src_weights / dst_weights ({rank: weight});
with several local agents pass one value per agent (lists).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import BluefogError, bf_weights, check

_DT = {torch.float32: _lib.BF_FLOAT32, torch.bfloat16: _lib.BF_BFLOAT16}


_raw_current_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream_ptr(stream=None, device=None):
    """cudaStream_t of `stream`, else of torch's current stream on `device`
    (the raw-handle query avoids building a Stream object: ~3 us per call)."""
    if stream is not None:
        return C.c_void_p(stream.cuda_stream)
    if _raw_current_stream is not None and device is not None:
        return C.c_void_p(_raw_current_stream(device))
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _allgather_bytes(payload: bytes, group=None) -> list:
    """All-gather one bytes object per process (bootstrap plumbing)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, payload, group=group)
    return out


def topology_matrix(kind: str, n: int, round: int = 0) -> np.ndarray:
    """Built-in topologies of the library: ring, exp2, full, one_peer_exp2."""
    kinds = {"ring": 0, "exp2": 1, "full": 2, "one_peer_exp2": 3}
    W = np.zeros((n, n), np.float64)
    check(_lib.load().bf_topology_matrix(kinds[kind], n, int(round),
                                         W.ctypes.data_as(C.POINTER(C.c_double))))
    return W


def one_peer_exp2(n: int, rank: int, round: int):
    s, d = C.c_int(), C.c_int()
    check(_lib.load().bf_schedule_one_peer_exp2(n, rank, int(round), C.byref(s), C.byref(d)))
    return s.value, d.value


def inner_outer_exp2(n: int, local_size: int, rank: int, round: int):
    """(src, dst) of `rank` at `round` of the inner-outer exp-2 schedule (R27); -1 = none."""
    s, d = C.c_int(), C.c_int()
    check(_lib.load().bf_schedule_inner_outer_exp2(n, local_size, rank, int(round), C.byref(s), C.byref(d)))
    return s.value, d.value


class _Views:
    """Keeps a ctypes bf_weights array (and its backing arrays) alive."""

    def __init__(self, k, self_weight, src_weights, dst_weights):
        def per_agent(v):
            if isinstance(v, (list, tuple)):
                if len(v) != k:
                    raise ValueError(f"expected {k} per-agent values, got {len(v)}")
                return list(v)
            return [v] * k if k == 1 else [v] * k

        sw, srcw, dstw = per_agent(self_weight), per_agent(src_weights), per_agent(dst_weights)
        self.arr = (bf_weights * k)()
        self._keep = []
        for a in range(k):
            w = self.arr[a]
            w.self_weight = float("nan") if sw[a] is None else float(sw[a])
            for kind, spec in (("src", srcw[a]), ("dst", dstw[a])):
                if spec is None:
                    setattr(w, "n_" + kind, -1)
                    continue
                ranks = sorted(int(r) for r in spec)
                ra = (C.c_int * max(1, len(ranks)))(*ranks)
                va = (C.c_double * max(1, len(ranks)))(*[float(spec[r]) for r in ranks])
                self._keep += [ra, va]
                setattr(w, "n_" + kind, len(ranks))
                setattr(w, kind + "_ranks", C.cast(ra, C.POINTER(C.c_int)))
                setattr(w, kind + "_weights", C.cast(va, C.POINTER(C.c_double)))

    def ptr(self):
        return C.cast(self.arr, C.POINTER(bf_weights))


class Context:
    """One process = one GPU hosting `agents_per_proc` agents (virtual agents if > 1)."""

    def __init__(self, agents_per_proc: int = 1, heap_bytes: int = 1 << 30, device: Optional[int] = None,
                 proc_rank: Optional[int] = None, n_procs: Optional[int] = None, group=None):
        self.lib = _lib.load()
        import torch.distributed as dist
        dist_on = dist.is_available() and dist.is_initialized()
        if proc_rank is None:
            proc_rank = dist.get_rank(group) if dist_on else 0
        if n_procs is None:
            n_procs = dist.get_world_size(group) if dist_on else 1
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", torch.cuda.current_device() if torch.cuda.is_available() else 0))
        self.device = device
        self.k = agents_per_proc
        self.proc = proc_rank
        self.nprocs = n_procs
        h = C.c_void_p()
        check(self.lib.bf_init(proc_rank, n_procs, agents_per_proc, device, int(heap_bytes), C.byref(h)))
        self.h = h
        blen = self.lib.bf_ipc_blob_size()
        if n_procs > 1:
            buf = C.create_string_buffer(blen)
            ln = C.c_size_t(blen)
            check(self.lib.bf_get_ipc_blob(h, buf, C.byref(ln)))
            blobs = _allgather_bytes(buf.raw[:ln.value], group)
            allb = b"".join(blobs)
            check(self.lib.bf_connect_peers(h, allb, ln.value))
        else:
            check(self.lib.bf_connect_peers(h, None, 0))
        self.n = self.lib.bf_size(h)
        self.rank = self.lib.bf_rank(h)

    # ---- lifecycle ---------------------------------------------------------
    def close(self):
        if getattr(self, "h", None):
            self.lib.bf_finalize(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- helpers -----------------------------------------------------------
    def _rows(self, t: torch.Tensor) -> int:
        if not t.is_cuda and not t.is_pinned() and t.device.type != "cpu":
            raise ValueError("unsupported tensor device")
        if not t.is_contiguous():
            raise ValueError("tensor must be contiguous")
        if t.numel() % self.k:
            raise ValueError(f"tensor numel {t.numel()} not divisible by agents_per_proc {self.k}")
        return t.numel() // self.k

    def _dev(self, t: torch.Tensor, what: str = "tensor") -> torch.Tensor:
        # device-pointer arguments of the C ABI: a CUDA tensor on this context's GPU
        if not t.is_cuda or t.device.index != self.device:
            raise ValueError(f"{what} must be a CUDA tensor on cuda:{self.device} (got {t.device})")
        return t

    def _like(self, t: torch.Tensor, ref: torch.Tensor, what: str, device: bool = True) -> torch.Tensor:
        # companion tensors (g, psi, out, shadow) are read / written with x's layout
        if t.dtype not in _DT:
            raise ValueError(f"{what}: unsupported dtype {t.dtype}")
        if not t.is_contiguous() or t.numel() != ref.numel():
            raise ValueError(f"{what} must be contiguous with {ref.numel()} elements (the layout of x)")
        if device:
            self._dev(t, what)
        elif t.is_cuda and t.device.index != self.device:
            raise ValueError(f"{what} must be on cuda:{self.device} or in host memory (got {t.device})")
        return t

    def _views(self, self_weight, src_weights, dst_weights):
        if self_weight is None and src_weights is None and dst_weights is None:
            return None
        return _Views(self.k, self_weight, src_weights, dst_weights)

    # ---- topology ------------------------------------------------
    def set_topology(self, W) -> bool:
        W = np.ascontiguousarray(np.asarray(W, np.float64))
        check(self.lib.bf_set_topology(self.h, W.shape[0], W.ctypes.data_as(C.POINTER(C.c_double))))
        return True

    def set_topology_local(self, self_weight, src_weights=None, dst_weights=None) -> bool:
        """Static topology from local views (collective): each process
        gives its agents' self / src / dst weights, the library assembles the global W."""
        v = _Views(self.k, self_weight, src_weights, dst_weights)
        check(self.lib.bf_set_topology_local(self.h, v.ptr()))
        return True

    def set_machine_topology(self, WM, local_size: int) -> bool:
        WM = np.ascontiguousarray(np.asarray(WM, np.float64))
        check(self.lib.bf_set_machine_topology(self.h, local_size, WM.shape[0],
                                               WM.ctypes.data_as(C.POINTER(C.c_double))))
        return True

    def in_neighbor_ranks(self, agent: Optional[int] = None):
        return self._nbrs(self.lib.bf_in_neighbors, agent)

    def out_neighbor_ranks(self, agent: Optional[int] = None):
        return self._nbrs(self.lib.bf_out_neighbors, agent)

    def _nbrs(self, fn, agent):
        agent = self.rank if agent is None else agent
        buf = (C.c_int * _lib.MAX_AGENTS)()
        n = C.c_int()
        check(fn(self.h, agent, buf, _lib.MAX_AGENTS, C.byref(n)))
        return list(buf[:n.value])

    def set_dynamic_schedule(self, kind: str = "one_peer_exp2", round0: int = 0):
        """"none", "one_peer_exp2" or "inner_outer_exp2" (R27;
        machines as set by set_machine_topology)."""
        kinds = {"none": 0, "one_peer_exp2": 1, "inner_outer_exp2": 2}
        check(self.lib.bf_set_dynamic_schedule(self.h, kinds[kind], int(round0)))

    def set_topology_check(self, enable: bool):
        check(self.lib.bf_set_topology_check(self.h, 1 if enable else 0))

    def set_max_ctas(self, ctas: int):
        """Grid cap of the exchange kernels (0 = all SMs); the same on every process."""
        check(self.lib.bf_set_max_ctas(self.h, int(ctas)))

    def reserve(self, bytes_per_agent: int):
        check(self.lib.bf_reserve(self.h, int(bytes_per_agent)))

    # ---- hot path ----------------------------------------------------------
    def neighbor_allreduce(self, tensor: torch.Tensor, self_weight=None, src_weights=None, dst_weights=None,
                           out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """Eq. 5 / Eq. 9 partial averaging."""
        count = self._rows(self._dev(tensor))
        y = torch.empty_like(tensor) if out is None else out
        if y.dtype != tensor.dtype:
            raise ValueError("out must have the dtype of the input")
        self._like(y, tensor, "out")
        v = self._views(self_weight, src_weights, dst_weights)
        check(self.lib.bf_neighbor_allreduce(self.h, C.c_void_p(tensor.data_ptr()), C.c_void_p(y.data_ptr()),
                                             count, _DT[tensor.dtype], v.ptr() if v else None,
                                             _stream_ptr(stream, self.device)))
        return y

    def atc_step(self, x: torch.Tensor, g: torch.Tensor, lr: float, wire: torch.dtype = torch.float32,
                 shadow: Optional[torch.Tensor] = None, self_weight=None, src_weights=None, dst_weights=None,
                 stream=None) -> torch.Tensor:
        """Fused ATC-DSGD step (Eq. 4-5, Eq. 17), in place on the fp32 master x."""
        if x.dtype != torch.float32:
            raise ValueError("x must be the fp32 master copy")
        count = self._rows(x)
        # x and g may be host tensors (end-to-end path, staged inside the call)
        self._like(g, x, "g", device=False)
        if shadow is not None:
            if shadow.dtype != torch.bfloat16:
                raise ValueError("shadow must be bf16")
            self._like(shadow, x, "shadow")
        v = self._views(self_weight, src_weights, dst_weights)
        check(self.lib.bf_atc_step(self.h, C.c_void_p(x.data_ptr()), C.c_void_p(g.data_ptr()), _DT[g.dtype],
                                   count, float(lr), _DT[wire],
                                   C.c_void_p(shadow.data_ptr()) if shadow is not None else None,
                                   v.ptr() if v else None, _stream_ptr(stream, self.device)))
        return x

    def exact_diffusion_step(self, x: torch.Tensor, g: torch.Tensor, psi: torch.Tensor, lr: float,
                             wire: torch.dtype = torch.float32, self_weight=None, src_weights=None,
                             dst_weights=None, stream=None) -> torch.Tensor:
        """Exact-Diffusion (appendix ed-1..ed-3): psi <- x - lr g, x <- W (psi + x - psi_prev),
        fused in one kernel; x and psi (fp32) are updated in place (psi = x^(0) initially)."""
        if x.dtype != torch.float32 or psi.dtype != torch.float32 or psi.shape != x.shape:
            raise ValueError("x and psi must be fp32 tensors of the same shape")
        count = self._rows(self._dev(x, "x"))
        self._like(g, x, "g")
        self._like(psi, x, "psi")
        v = self._views(self_weight, src_weights, dst_weights)
        check(self.lib.bf_exact_diffusion_step(self.h, C.c_void_p(x.data_ptr()), C.c_void_p(g.data_ptr()),
                                               _DT[g.dtype], C.c_void_p(psi.data_ptr()), count, float(lr),
                                               _DT[wire], v.ptr() if v else None, _stream_ptr(stream, self.device)))
        return x

    def gt_uv_step(self, u: torch.Tensor, v: torch.Tensor, y: torch.Tensor, x_out: torch.Tensor, lr: float,
                   wire: torch.dtype = torch.float32, self_weight=None, src_weights=None, dst_weights=None,
                   stream=None) -> torch.Tensor:
        """Push-sum gradient tracking, first half of a round (appendix), one
        fused launch: u <- W(u - lr y), v <- W v (one fp32 weight per agent, shape (K,)),
        x_out = u / v.  u, v updated in place; returns x_out."""
        for t, nm in ((u, "u"), (y, "y"), (x_out, "x_out")):
            if t.dtype != torch.float32:
                raise ValueError(f"{nm} must be fp32")
        count = self._rows(self._dev(u, "u"))
        self._like(y, u, "y")
        self._like(x_out, u, "x_out")
        self._dev(v, "v")
        if v.dtype != torch.float32 or v.numel() != self.k or not v.is_contiguous():
            raise ValueError(f"v must be a contiguous fp32 tensor of {self.k} push-sum weights (one per agent)")
        vw = self._views(self_weight, src_weights, dst_weights)
        check(self.lib.bf_gt_uv_step(self.h, C.c_void_p(u.data_ptr()), C.c_void_p(v.data_ptr()),
                                     C.c_void_p(y.data_ptr()), C.c_void_p(x_out.data_ptr()), count, float(lr),
                                     _DT[wire], vw.ptr() if vw else None, _stream_ptr(stream, self.device)))
        return x_out

    def gt_y_step(self, y: torch.Tensor, g: torch.Tensor, g_prev: torch.Tensor, wire: torch.dtype = torch.float32,
                  self_weight=None, src_weights=None, dst_weights=None, stream=None) -> torch.Tensor:
        """Push-sum gradient tracking, second half (appendix), one fused launch:
        y <- W(y + g - g_prev), in place."""
        for t, nm in ((y, "y"), (g, "g"), (g_prev, "g_prev")):
            if t.dtype != torch.float32:
                raise ValueError(f"{nm} must be fp32")
        count = self._rows(self._dev(y, "y"))
        self._like(g, y, "g")
        self._like(g_prev, y, "g_prev")
        vw = self._views(self_weight, src_weights, dst_weights)
        check(self.lib.bf_gt_y_step(self.h, C.c_void_p(y.data_ptr()), C.c_void_p(g.data_ptr()),
                                    C.c_void_p(g_prev.data_ptr()), count, _DT[wire], vw.ptr() if vw else None,
                                    _stream_ptr(stream, self.device)))
        return y

    def awc_step(self, x: torch.Tensor, g: torch.Tensor, lr: float, self_weight=None, src_weights=None,
                 dst_weights=None, stream=None) -> torch.Tensor:
        """Fused AWC-DSGD step (Eq. 16): x <- W x - lr*g, in place on the fp32 master x."""
        if x.dtype != torch.float32:
            raise ValueError("x must be the fp32 master copy")
        count = self._rows(self._dev(x, "x"))
        self._like(g, x, "g")
        v = self._views(self_weight, src_weights, dst_weights)
        check(self.lib.bf_awc_step(self.h, C.c_void_p(x.data_ptr()), C.c_void_p(g.data_ptr()), _DT[g.dtype],
                                   count, float(lr), v.ptr() if v else None, _stream_ptr(stream, self.device)))
        return x

    # ---- non-blocking form -------------------------------------------
    def neighbor_allreduce_nonblocking(self, tensor: torch.Tensor, self_weight=None, src_weights=None,
                                       dst_weights=None):
        """Launch neighbor_allreduce on the context's side stream and return a
        handle immediately; the caller's stream keeps running
        computation.  `wait(handle)` returns the result."""
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=self.device)
        cur = torch.cuda.current_stream()
        self._side.wait_stream(cur)             # the input is complete before the exchange reads it
        out = torch.empty_like(tensor)
        tensor.record_stream(self._side)
        out.record_stream(self._side)
        self.neighbor_allreduce(tensor, self_weight, src_weights, dst_weights, out=out, stream=self._side)
        ev = torch.cuda.Event()
        ev.record(self._side)
        return (out, ev)

    @staticmethod
    def wait(handle) -> torch.Tensor:
        out, ev = handle
        torch.cuda.current_stream().wait_event(ev)
        return out

    def hierarchical_neighbor_allreduce(self, tensor: torch.Tensor, self_weight=None, src_machine_weights=None,
                                        out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """P:660-675 (machine-level neighbour averaging of machine averages)."""
        count = self._rows(self._dev(tensor))
        y = torch.empty_like(tensor) if out is None else out
        if y.dtype != tensor.dtype:
            raise ValueError("out must have the dtype of the input")
        self._like(y, tensor, "out")
        v = self._views(self_weight, src_machine_weights, None)
        check(self.lib.bf_hierarchical_neighbor_allreduce(self.h, C.c_void_p(tensor.data_ptr()),
                                                          C.c_void_p(y.data_ptr()), count, _DT[tensor.dtype],
                                                          v.ptr() if v else None, _stream_ptr(stream, self.device)))
        return y

    def enable_nvls(self, local_size: int, max_count: int) -> bool:
        """Collective: give every machine that spans processes (local_size agents >
        agents_per_proc) a multicast-backed buffer (torch symmetric memory over the
        machine's process group -- allocation plumbing) so the hierarchical calls
        average the machine in the NVSwitch (multimem.ld_reduce, hier_nvls.cu).
        Returns False (and changes nothing) when the box has no multicast support."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        if local_size <= self.k or local_size % self.k or not dist.is_initialized():
            raise ValueError("NVLS needs machines that span processes (local_size a multiple of agents_per_proc)")
        P = local_size // self.k
        if self.nprocs % P:
            raise ValueError("machines must tile the processes")
        cache = getattr(self, "_machine_groups", None) or {}
        if P not in cache:   # every process creates every machine's group once (collective)
            cache[P] = [dist.new_group(list(range(m * P, (m + 1) * P))) for m in range(self.nprocs // P)]
            self._machine_groups = cache
        groups = cache[P]
        mine = groups[self.proc // P]
        cap = (int(max_count) + 3) // 4 * 4
        t = symm.empty(4 * cap, dtype=torch.float32, device=f"cuda:{self.device}")   # partials + averages, x 2
        h = symm.rendezvous(t, mine)
        mc = int(getattr(h, "multicast_ptr", 0) or 0)
        try:   # static query (device type, index) on current torch; older: a property
            sup = bool(symm._SymmetricMemory.has_multicast_support(torch._C._autograd.DeviceType.CUDA, self.device))
        except Exception:   # noqa: BLE001
            sup = mc != 0
        ok = torch.tensor([1 if (sup and mc) else 0], device=f"cuda:{self.device}")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)   # every process takes the same path
        if not int(ok.item()):
            return False
        check(self.lib.bf_hier_set_multicast(self.h, int(local_size), C.c_void_p(t.data_ptr()), mc, 4 * cap * 4))
        self._nvls = (t, h, groups)   # keep the buffer and its mapping alive
        return True

    def disable_nvls(self):
        check(self.lib.bf_hier_set_multicast(self.h, 0, None, 0, 0))
        self._nvls = None

    def hierarchical_atc_step(self, x: torch.Tensor, g: torch.Tensor, lr: float, self_weight=None,
                              src_machine_weights=None, stream=None) -> torch.Tensor:
        """H-ATC: x <- (W_M kron J_L/L)(x - lr g), in place on the fp32 master x."""
        return self._hier_step(self.lib.bf_hierarchical_atc_step, x, g, lr, self_weight, src_machine_weights, stream)

    def hierarchical_awc_step(self, x: torch.Tensor, g: torch.Tensor, lr: float, self_weight=None,
                              src_machine_weights=None, stream=None) -> torch.Tensor:
        """H-AWC: x <- (W_M kron J_L/L) x - lr g, in place on the fp32 master x."""
        return self._hier_step(self.lib.bf_hierarchical_awc_step, x, g, lr, self_weight, src_machine_weights, stream)

    def _hier_step(self, fn, x, g, lr, self_weight, src_machine_weights, stream):
        if x.dtype != torch.float32:
            raise ValueError("x must be the fp32 master copy")
        count = self._rows(self._dev(x, "x"))
        self._like(g, x, "g")
        v = self._views(self_weight, src_machine_weights, None)
        check(fn(self.h, C.c_void_p(x.data_ptr()), C.c_void_p(g.data_ptr()), _DT[g.dtype], count, float(lr),
                 v.ptr() if v else None, _stream_ptr(stream, self.device)))
        return x

    # ---- windows ---------------------------------------------------
    def win_create(self, tensor: torch.Tensor, name: str, zero_init: bool = True, with_p: bool = False) -> bool:
        count = self._rows(self._dev(tensor))
        if not hasattr(self, "_windows"):
            self._windows = {}
        self._windows[name] = (tensor.dtype, tensor.numel())
        torch.cuda.synchronize(self.device)
        check(self.lib.bf_win_create(self.h, name.encode(), C.c_void_p(tensor.data_ptr()), count,
                                     _DT[tensor.dtype], 1 if zero_init else 0, 1 if with_p else 0))
        return True

    def alloc(self, shape, dtype: torch.dtype = torch.float32) -> torch.Tensor:
        """A tensor in the symmetric heap (collective, bf_alloc): windows created on
        it can be read by the neighbours (win_get)."""
        shape = tuple(int(d) for d in shape)
        nbytes = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        ptr = C.c_void_p()
        check(self.lib.bf_alloc(self.h, nbytes, C.byref(ptr)))

        class _HeapBlock:   # __cuda_array_interface__ view; the heap owns the memory
            pass
        blk = _HeapBlock()
        typestr = {torch.float32: "<f4", torch.bfloat16: "<V2"}[dtype]
        blk.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr.value, False),
                                        "version": 2, "strides": None}
        if dtype == torch.bfloat16:   # no bf16 typestr: wrap as int16 and reinterpret
            blk.__cuda_array_interface__["typestr"] = "<i2"
            t = torch.as_tensor(blk, device=f"cuda:{self.device}").view(torch.bfloat16)
        else:
            t = torch.as_tensor(blk, device=f"cuda:{self.device}")
        return t

    def win_get(self, name: str, src_weights=None, agent_mask: int = 0, stream=None) -> bool:
        """neighbor_win_get: fetch weight * x_j of the selected in-neighbours into
        this agent's slots (the window tensor must come from alloc())."""
        v = None
        if src_weights is not None:
            v = _Views(self.k, [1.0] * self.k, src_weights, None)
        check(self.lib.bf_win_get(self.h, name.encode(), v.ptr() if v else None, int(agent_mask),
                                  _stream_ptr(stream, self.device)))
        return True

    def win_set_error_feedback(self, name: str, enable: bool = True) -> bool:
        """bf16 windows: keep the wire rounding residual in the sender's outbox (R24)."""
        check(self.lib.bf_win_set_error_feedback(self.h, name.encode(), 1 if enable else 0))
        return True

    def win_free(self, name: str) -> bool:
        torch.cuda.synchronize(self.device)
        check(self.lib.bf_win_free(self.h, name.encode()))
        getattr(self, "_windows", {}).pop(name, None)
        return True

    def win_put(self, name: str, self_weight=None, dst_weights=None, agent_mask: int = 0, stream=None) -> bool:
        v = self._views(self_weight, None, dst_weights)
        check(self.lib.bf_win_put(self.h, name.encode(), v.ptr() if v else None, agent_mask, _stream_ptr(stream, self.device)))
        return True

    def win_accumulate(self, name: str, self_weight=None, dst_weights=None, require_mutex: bool = True,
                       agent_mask: int = 0, stream=None) -> bool:
        v = self._views(self_weight, None, dst_weights)
        check(self.lib.bf_win_accumulate(self.h, name.encode(), v.ptr() if v else None,
                                         1 if require_mutex else 0, agent_mask, _stream_ptr(stream, self.device)))
        return True

    def win_accumulate_grad(self, name: str, g: torch.Tensor, lr: float, self_weight=None, dst_weights=None,
                            agent_mask: int = 0, stream=None) -> bool:
        """Gradient-in-window push (SGP-style): x <- x - lr g, then win_accumulate, in one kernel.
        g: device tensor of the window's dtype and shape."""
        self._dev(g, "g")
        win = getattr(self, "_windows", {}).get(name)
        if win is not None and (g.dtype != win[0] or g.numel() != win[1]):
            raise ValueError(f"g must have the window's dtype {win[0]} and {win[1]} elements")
        if not g.is_contiguous():
            raise ValueError("g must be contiguous")
        v = self._views(self_weight, None, dst_weights)
        check(self.lib.bf_win_accumulate_grad(self.h, name.encode(), C.c_void_p(g.data_ptr()), float(lr),
                                              v.ptr() if v else None, agent_mask, _stream_ptr(stream, self.device)))
        return True

    def win_update(self, name: str, self_weight=None, src_weights=None, out: Optional[torch.Tensor] = None,
                   agent_mask: int = 0, stream=None):
        if out is not None:
            self._dev(out, "out")
            if not out.is_contiguous():
                raise ValueError("out must be contiguous")
        v = self._views(self_weight, src_weights, None)
        check(self.lib.bf_win_update(self.h, name.encode(), v.ptr() if v else None,
                                     C.c_void_p(out.data_ptr()) if out is not None else None, agent_mask,
                                     _stream_ptr(stream, self.device)))
        return out

    def win_update_then_collect(self, name: str, agent_mask: int = 0, stream=None) -> bool:
        check(self.lib.bf_win_update_then_collect(self.h, name.encode(), agent_mask, _stream_ptr(stream, self.device)))
        return True

    def win_p(self, name: str, stream=None) -> np.ndarray:
        p = np.zeros(self.k, np.float64)
        check(self.lib.bf_win_get_p(self.h, name.encode(), p.ctypes.data_as(C.POINTER(C.c_double)),
                                    _stream_ptr(stream, self.device)))
        return p

    def win_counters(self, name: str, dst_local: int, src_rank: int):
        v, c = C.c_uint64(), C.c_uint64()
        check(self.lib.bf_win_counters(self.h, name.encode(), dst_local, src_rank, C.byref(v), C.byref(c)))
        return v.value, c.value

    def win_version(self, name: str, src_rank: int) -> int:
        v = C.c_uint64()
        check(self.lib.bf_win_version(self.h, name.encode(), int(src_rank), C.byref(v)))
        return v.value

    def win_slot_offset(self, name: str, agent: int, src_rank: int) -> int:
        return self.lib.bf_win_slot_offset(self.h, name.encode(), agent, src_rank)

    # ---- misc ------------------------------------------------------------------
    def barrier(self, stream=None):
        check(self.lib.bf_barrier(self.h, _stream_ptr(stream, self.device)))

    def poll_error(self):
        check(self.lib.bf_poll_error(self.h))

    def exchange_stats(self, reset: bool = True) -> np.ndarray:
        """Per-CTA diagnostics of the fused exchange kernel, shape (4096, 8)
        (BF_STATS=1 and a -DBF_STATS=1 build; see include/bluefog_b200.h)."""
        buf = (C.c_uint64 * (4096 * 8))()
        check(self.lib.bf_exchange_stats(self.h, buf, 4096 * 8, int(reset)))
        return np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8).copy()

    def kernel_launches(self) -> int:
        return int(self.lib.bf_kernel_launches(self.h))

    @staticmethod
    def fill_uniform(t: torch.Tensor, seed: int, offset: int = 0, scale: float = 1.0, stream=None):
        """Synthetic input generator (same counter-based generator as synthetic/)."""
        check(_lib.load().bf_fill_uniform(C.c_void_p(t.data_ptr()), _DT[t.dtype], t.numel(), int(seed), int(offset),
                                          float(scale), _stream_ptr(stream, t.device.index)))
        return t
