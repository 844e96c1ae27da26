"""B200-native decentralized partial averaging (BlueFog, arXiv 2111.04287).

The hot path lives in libbluefog_b200.so (hand-written sm_100a CUDA behind the
C ABI of include/bluefog_b200.h).  Importing this package loads it; there is no
CPU fallback.
"""
from . import _lib
from ._lib import BluefogError

_lib.load()   # fail loudly if the CUDA library is missing

from .api import Context, one_peer_exp2, topology_matrix  # noqa: E402

__all__ = ["Context", "BluefogError", "topology_matrix", "one_peer_exp2"]
