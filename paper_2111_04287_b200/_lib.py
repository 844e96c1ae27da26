"""ctypes loader for libbluefog_b200.so (the C ABI of include/bluefog_b200.h).

Argument marshalling only.  There is no CPU fallback: if the shared library
is missing or fails to load, importing the product raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("BF_LIB_PATH") or os.path.join(HERE, "libbluefog_b200.so")

BF_OK = 0
STATUS = {0: "BF_OK", 1: "BF_ERR_ARG", 2: "BF_ERR_STATE", 3: "BF_ERR_TOPOLOGY", 4: "BF_ERR_CUDA",
          5: "BF_ERR_TIMEOUT", 6: "BF_ERR_NOMEM", 7: "BF_ERR_UNSUPPORTED", 8: "BF_ERR_WINDOW"}
BF_FLOAT32 = 0
BF_BFLOAT16 = 1
MAX_AGENTS = 64
MAX_PROCS = 16
MAX_LOCAL_AGENTS = 16
MAX_DEGREE = 16


class BluefogError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class bf_weights(C.Structure):
    _fields_ = [("self_weight", C.c_double),
                ("n_src", C.c_int), ("src_ranks", C.POINTER(C.c_int)), ("src_weights", C.POINTER(C.c_double)),
                ("n_dst", C.c_int), ("dst_ranks", C.POINTER(C.c_int)), ("dst_weights", C.POINTER(C.c_double))]


_vp = C.c_void_p
_i = C.c_int
_sz = C.c_size_t
_u64 = C.c_uint64
_wp = C.POINTER(bf_weights)

_SIGS = {
    "bf_init": (_i, [_i, _i, _i, _i, _sz, C.POINTER(_vp)]),
    "bf_ipc_blob_size": (_sz, []),
    "bf_get_ipc_blob": (_i, [_vp, _vp, C.POINTER(_sz)]),
    "bf_connect_peers": (_i, [_vp, _vp, _sz]),
    "bf_finalize": (_i, [_vp]),
    "bf_size": (_i, [_vp]),
    "bf_rank": (_i, [_vp]),
    "bf_local_agents": (_i, [_vp]),
    "bf_last_error": (C.c_char_p, []),
    "bf_status_string": (C.c_char_p, [_i]),
    "bf_set_topology": (_i, [_vp, _i, C.POINTER(C.c_double)]),
    "bf_set_machine_topology": (_i, [_vp, _i, _i, C.POINTER(C.c_double)]),
    "bf_set_topology_local": (_i, [_vp, _wp]),
    "bf_hier_set_multicast": (_i, [_vp, _i, _vp, _u64, _sz]),
    "bf_win_version": (_i, [_vp, C.c_char_p, _i, C.POINTER(_u64)]),
    "bf_in_neighbors": (_i, [_vp, _i, C.POINTER(_i), _i, C.POINTER(_i)]),
    "bf_out_neighbors": (_i, [_vp, _i, C.POINTER(_i), _i, C.POINTER(_i)]),
    "bf_topology_matrix": (_i, [_i, _i, _u64, C.POINTER(C.c_double)]),
    "bf_schedule_one_peer_exp2": (_i, [_i, _i, _u64, C.POINTER(_i), C.POINTER(_i)]),
    "bf_schedule_inner_outer_exp2": (_i, [_i, _i, _i, _u64, C.POINTER(_i), C.POINTER(_i)]),
    "bf_set_dynamic_schedule": (_i, [_vp, _i, _u64]),
    "bf_set_topology_check": (_i, [_vp, _i]),
    "bf_set_max_ctas": (_i, [_vp, _i]),
    "bf_neighbor_allreduce": (_i, [_vp, _vp, _vp, _sz, _i, _wp, _vp]),
    "bf_atc_step": (_i, [_vp, _vp, _vp, _i, _sz, C.c_float, _i, _vp, _wp, _vp]),
    "bf_awc_step": (_i, [_vp, _vp, _vp, _i, _sz, C.c_float, _wp, _vp]),
    "bf_hierarchical_neighbor_allreduce": (_i, [_vp, _vp, _vp, _sz, _i, _wp, _vp]),
    "bf_hierarchical_atc_step": (_i, [_vp, _vp, _vp, _i, _sz, C.c_float, _wp, _vp]),
    "bf_hierarchical_awc_step": (_i, [_vp, _vp, _vp, _i, _sz, C.c_float, _wp, _vp]),
    "bf_win_create": (_i, [_vp, C.c_char_p, _vp, _sz, _i, _i, _i]),
    "bf_win_free": (_i, [_vp, C.c_char_p]),
    "bf_win_put": (_i, [_vp, C.c_char_p, _wp, _u64, _vp]),
    "bf_win_accumulate": (_i, [_vp, C.c_char_p, _wp, _i, _u64, _vp]),
    "bf_win_accumulate_grad": (_i, [_vp, C.c_char_p, _vp, C.c_float, _wp, _u64, _vp]),
    "bf_win_update": (_i, [_vp, C.c_char_p, _wp, _vp, _u64, _vp]),
    "bf_win_update_then_collect": (_i, [_vp, C.c_char_p, _u64, _vp]),
    "bf_win_get_p": (_i, [_vp, C.c_char_p, C.POINTER(C.c_double), _vp]),
    "bf_win_counters": (_i, [_vp, C.c_char_p, _i, _i, C.POINTER(_u64), C.POINTER(_u64)]),
    "bf_win_slot_offset": (C.c_longlong, [_vp, C.c_char_p, _i, _i]),
    "bf_barrier": (_i, [_vp, _vp]),
    "bf_poll_error": (_i, [_vp]),
    "bf_reserve": (_i, [_vp, _sz]),
    "bf_fill_uniform": (_i, [_vp, _i, _sz, _u64, _u64, C.c_float, _vp]),
    "bf_kernel_launches": (_u64, [_vp]),
    "bf_exchange_stats": (_i, [_vp, C.POINTER(_u64), _sz, _i]),
    "bf_win_set_error_feedback": (_i, [_vp, C.c_char_p, _i]),
    "bf_alloc": (_i, [_vp, _sz, C.POINTER(_vp)]),
    "bf_win_get": (_i, [_vp, C.c_char_p, _wp, _u64, _vp]),
    "bf_exact_diffusion_step": (_i, [_vp, _vp, _vp, _i, _vp, _sz, C.c_float, _i, _wp, _vp]),
    "bf_gt_uv_step": (_i, [_vp, _vp, _vp, _vp, _vp, _sz, C.c_float, _i, _wp, _vp]),
    "bf_gt_y_step": (_i, [_vp, _vp, _vp, _vp, _sz, _i, _wp, _vp]),
}

_lib = None


def load():
    """Load the library (raises if it was not built: no silent fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(f"{SO_PATH} is missing: build it with `python -m paper_2111_04287_b200.build` "
                              "(there is no CPU fallback)")
        lib = C.CDLL(SO_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int) -> None:
    if status != BF_OK:
        msg = load().bf_last_error()
        raise BluefogError(status, msg.decode() if msg else "")
