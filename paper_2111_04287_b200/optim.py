"""Optimizer wrappers over the fused hot path.

BlueFog wraps a torch optimizer:

    opt = bf.DistributedAdaptThenCombineOptimizer(optim.SGD(...), model=model)

and runs, per layer, the local SGD step (adapt, Eq. 4) followed by the
neighbour averaging (combine, Eq. 5) -- ATC, Eq. 17 -- overlapping the
communication of one layer with the backward pass of the next,
with small tensors fused into one message (tensor fusion).

Here the adapt and the combine of a whole bucket are ONE kernel
(`bf_atc_step`, or `bf_awc_step` for Eq. 16).  Tensor fusion is done without
copies: the parameters of each bucket are re-homed as views into a flat
buffer of shape (K, n_bucket) -- K = the process's local agents -- and their
gradients into a second flat buffer, so a bucket's step is a single C-ABI call
on two contiguous buffers.  With `overlap=True` a bucket's step is launched
from the post-accumulate-grad hook of its last parameter, i.e. while backward
is still computing the gradients of earlier layers (per-layer ATC).

Parameters are stacked per local agent: every tensor has shape (K, *shape).
Plain Python (bucket planning, hooks, views); every arithmetic step runs in
libbluefog_b200.so.
"""
from __future__ import annotations

from typing import Iterable, List, Optional, Sequence

import torch


def plan_buckets(numels: Sequence[int], bucket_elems: int) -> List[List[int]]:
    """Group parameter indices into buckets of about `bucket_elems` elements,
    in REVERSE registration order (backward produces the last layer's
    gradients first), never splitting a tensor.  A tensor larger than
    the bucket gets a bucket of its own."""
    if bucket_elems <= 0:
        raise ValueError("bucket_elems must be positive")
    buckets: List[List[int]] = []
    cur: List[int] = []
    cur_n = 0
    for i in reversed(range(len(numels))):
        n = int(numels[i])
        if cur and cur_n + n > bucket_elems:
            buckets.append(cur)
            cur, cur_n = [], 0
        cur.append(i)
        cur_n += n
    if cur:
        buckets.append(cur)
    return buckets


class _Bucket:
    def __init__(self, params: List[torch.nn.Parameter], k: int, dtype_g: torch.dtype):
        self.params = params
        self.numels = [p[0].numel() for p in params]   # per agent
        self.n = sum(self.numels)
        dev = params[0].device
        self.x = torch.empty(k, self.n, device=dev, dtype=torch.float32)
        self.g = torch.zeros(k, self.n, device=dev, dtype=dtype_g)
        off = 0
        with torch.no_grad():
            for p, m in zip(params, self.numels):
                self.x[:, off:off + m].copy_(p.detach().reshape(k, m))
                shape = p.shape
                # re-home the parameter and its gradient as views into the flat buffers
                p.data = self.x[:, off:off + m].view(shape)
                p.grad = self.g[:, off:off + m].view(shape)
                off += m
        self.pending = len(params)


class DistributedAdaptThenCombineOptimizer:
    """ATC-DSGD optimizer (Eq. 17; wrapper API of P:601-607).

    ctx:      a Context (its topology / one-peer schedule decides the combine)
    params:   tensors of shape (ctx.k, *shape), fp32 masters
    lr:       SGD step (momentum is out of scope)
    wire:     dtype of the published copy (torch.float32 or torch.bfloat16)
    bucket_bytes: tensor-fusion bucket size (fp32 bytes per agent)
    overlap:  launch each bucket's step from backward hooks, on a side stream, so the
              exchange runs while backward computes the earlier layers
    overlap_ctas: with overlap, the exchange kernels' CTA cap (bf_set_max_ctas) -- the
              exchange leaves the other SMs to backward; 0 keeps the context's setting
    awc:      adapt-WITH-combine (Eq. 16) instead of ATC
    grad_dtype: dtype of the flat gradient buffers (fp32 or bf16)
    """

    def __init__(self, ctx, params: Iterable[torch.Tensor], lr: float, wire: torch.dtype = torch.float32,
                 bucket_bytes: int = 25 << 20, overlap: bool = False, awc: bool = False,
                 grad_dtype: torch.dtype = torch.float32, overlap_ctas: int = 0):
        self.ctx = ctx
        self.lr = float(lr)
        self.wire = wire
        self.awc = awc
        self.overlap = overlap
        params = [p for p in params]
        if not params:
            raise ValueError("no parameters")
        for p in params:
            if p.dim() < 1 or p.shape[0] != ctx.k or p.dtype != torch.float32 or not p.is_cuda:
                raise ValueError("parameters must be fp32 CUDA tensors of shape (agents_per_proc, ...)")
        if awc and wire != torch.float32:
            raise ValueError("AWC publishes the fp32 x (bf_awc_step)")
        plan = plan_buckets([p[0].numel() for p in params], max(1, bucket_bytes // 4))
        self.buckets = [_Bucket([params[i] for i in idx], ctx.k, grad_dtype) for idx in plan]
        self.steps_launched = 0
        self._hooks = []
        self._side = None
        if overlap:
            self._side = torch.cuda.Stream(device=params[0].device)
            if overlap_ctas:
                ctx.set_max_ctas(overlap_ctas)
            for b in self.buckets:
                for p in b.params:
                    self._hooks.append(p.register_post_accumulate_grad_hook(self._make_hook(b)))

    # ---- per-bucket fused step --------------------------------------------------
    def _step_bucket(self, b: _Bucket):
        if self.awc:
            self.ctx.awc_step(b.x, b.g, self.lr)
        else:
            self.ctx.atc_step(b.x, b.g, self.lr, wire=self.wire)
        self.steps_launched += 1

    def _make_hook(self, b: _Bucket):
        def hook(_p):
            b.pending -= 1
            if b.pending == 0:   # every gradient of the bucket is accumulated: step it now, beside backward
                self._side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(self._side):
                    self._step_bucket(b)
        return hook

    def step(self):
        """Without overlap: one fused ATC call per bucket.  With overlap the
        buckets were already stepped by the hooks during backward (side stream);
        step() steps any bucket whose hooks did not all fire, joins the side
        stream into the current one and re-arms the hooks."""
        for b in self.buckets:
            if not self.overlap:
                self._step_bucket(b)
            elif b.pending > 0:
                self._side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(self._side):
                    self._step_bucket(b)
            b.pending = len(b.params)
        if self.overlap:
            torch.cuda.current_stream().wait_stream(self._side)

    def zero_grad(self):
        for b in self.buckets:
            b.g.zero_()

    def flat_params(self) -> List[torch.Tensor]:
        return [b.x for b in self.buckets]

    def remove_hooks(self):
        for h in self._hooks:
            h.remove()
        self._hooks = []


def resnet50_param_shapes() -> List[tuple]:
    """Parameter shapes of ResNet-50 (torchvision layout, 161 tensors, 25 557 032
    elements -- the model the paper's DSGD experiments train)."""
    shapes: List[tuple] = [(64, 3, 7, 7), (64,), (64,)]
    inplanes = 64
    for planes, blocks in ((64, 3), (128, 4), (256, 6), (512, 3)):
        for bidx in range(blocks):
            shapes += [(planes, inplanes, 1, 1), (planes,), (planes,),
                       (planes, planes, 3, 3), (planes,), (planes,),
                       (planes * 4, planes, 1, 1), (planes * 4,), (planes * 4,)]
            if bidx == 0:
                shapes += [(planes * 4, inplanes, 1, 1), (planes * 4,), (planes * 4,)]
            inplanes = planes * 4
    shapes += [(1000, 2048), (1000,)]
    return shapes
