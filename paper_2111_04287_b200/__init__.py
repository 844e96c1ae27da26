"""B200-native decentralized partial averaging (BlueFog, arXiv 2111.04287).

The hot path lives in libbluefog_b200.so (hand-written sm_100a CUDA behind the
C ABI of include/bluefog_b200.h).  It is loaded on first use (Context,
topology helpers); there is no CPU fallback -- a missing library raises.
"""
from . import _lib
from ._lib import BluefogError
from .api import Context, inner_outer_exp2, one_peer_exp2, topology_matrix

__all__ = ["Context", "BluefogError", "topology_matrix", "one_peer_exp2", "inner_outer_exp2"]
