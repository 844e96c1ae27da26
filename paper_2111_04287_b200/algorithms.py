"""Application examples of the paper's appendix built on the fused primitives.

* Exact-Diffusion (appendix, Eqs. ed-1..ed-3) is a single fused primitive:
  `Context.exact_diffusion_step` (MODE 3 of the fused exchange kernel).
* Push-sum gradient tracking (appendix, "Push-sum gradient tracking",
  PAPER.md lines 1000-1006 and its listing) needs two partial-averaging passes
  per round around the caller's gradient; each is one fused launch:

      u <- W (u - lr y), v <- W v, x = u / v     Context.gt_uv_step   (MODE 5)
      g' = grad(x)                               the caller's gradient
      y <- W (y + g' - g)                        Context.gt_y_step    (MODE 4)

  v is one push-sum weight per agent (reading R28: v^0 = 1 keeps the entries of
  the paper's vector v equal).  No elementwise glue runs outside the kernels.
"""
from __future__ import annotations

from typing import Callable

import torch


def gradient_tracking_step(ctx, u: torch.Tensor, v: torch.Tensor, y: torch.Tensor, g_prev: torch.Tensor,
                           grad_fn: Callable[[torch.Tensor], torch.Tensor], lr: float, x: torch.Tensor = None,
                           **weights):
    """One round of push-sum gradient tracking over the context's current topology /
    schedule, or per-call views passed as `weights` (self_weight, src_weights,
    dst_weights -- the same W for both passes of the round; with a one-peer schedule
    the two passes take two consecutive rounds of it, so use views or a static W).
    u, y, g_prev: fp32 (K, d); v: fp32 (K,).  Returns (x, u, v, y, g) -- u, v, y
    updated in place, g the new gradient (the caller keeps it as the next g_prev)."""
    if x is None:
        x = torch.empty_like(u)
    ctx.gt_uv_step(u, v, y, x, lr, **weights)     # u <- W(u - lr y); v <- W v; x = u / v
    g = grad_fn(x)
    ctx.gt_y_step(y, g, g_prev, **weights)        # y <- W(y + g - g_prev)
    return x, u, v, y, g
