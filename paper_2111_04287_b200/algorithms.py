"""Application examples of the paper's appendix built on the fused primitives.

* Exact-Diffusion (appendix, Eqs. ed-1..ed-3) is a single fused primitive:
  `Context.exact_diffusion_step` (MODE 3 of the fused exchange kernel).
* Push-sum gradient tracking (appendix, "Push-sum gradient tracking",
  PAPER.md lines 1000-1006 and its listing) needs three partial averagings per
  round; here they are the library's fused calls:

      u <- W (u - lr y)            one fused ATC call (adapt = u - lr y)
      v <- W v                     neighbor_allreduce of the push-sum weights
      x  = u / v                   elementwise (application code, as in the listing)
      g' = grad(x)                 the caller's gradient
      y <- W (y + g' - g)          one fused ATC call with lr = 1 and "gradient" g - g'

  The elementwise glue (u / v, g - g') is application code exactly as in the
  paper's listing; every partial averaging runs in libbluefog_b200.so.
"""
from __future__ import annotations

from typing import Callable

import torch


def gradient_tracking_step(ctx, u: torch.Tensor, v: torch.Tensor, y: torch.Tensor, g_prev: torch.Tensor,
                           grad_fn: Callable[[torch.Tensor], torch.Tensor], lr: float):
    """One round of push-sum gradient tracking over the context's current
    topology / one-peer schedule (each fused call advances a one-peer round,
    so all three averagings of a round must use the same W: call with a static
    topology, or with per-call views).  u, y, g_prev: fp32 (K, d); v: fp32
    (K, 1).  Returns (x, u, v, y, g) -- u, v, y updated in place."""
    ctx.atc_step(u, y, lr)                      # u <- W (u - lr y)
    ctx.neighbor_allreduce(v, out=v)            # v <- W v
    x = u / v                                   # x = u / v
    g = grad_fn(x)
    diff = g_prev - g                           # y + g - g_prev = y - 1 * (g_prev - g)
    ctx.atc_step(y, diff.contiguous(), 1.0)     # y <- W (y + g - g_prev)
    return x, u, v, y, g
