"""ctypes declarations of include/b200reduce.h (argument marshalling only).

Loads the in-tree ``libb200reduce.so``. There is no fallback: if the library
is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# the in-tree build, always (no environment override: the product path loads
# exactly this library; measurement tools that A/B other builds load those
# .so files themselves, tools/ab_lib.py)
LIB_PATH = os.path.join(_HERE, "libb200reduce.so")

RD_INT32, RD_UINT32, RD_INT64, RD_FLOAT32, RD_FLOAT64 = range(5)
RD_SUM, RD_PROD, RD_MIN, RD_MAX, RD_AND, RD_OR, RD_XOR = range(7)
RD_ARGMIN, RD_ARGMAX, RD_SUM_COMPENSATED, RD_SUM_EXACT = 7, 8, 9, 10
RD_EXACT_MAX_WORDS = 72
RD_OK = 0
STATUS = {0: "RD_OK", 1: "RD_ERR_INVALID_ARG", 2: "RD_ERR_UNSUPPORTED", 3: "RD_ERR_MISALIGNED",
          4: "RD_ERR_CUDA", 5: "RD_ERR_NCCL", 6: "RD_ERR_MISMATCH", 7: "RD_ERR_TIMEOUT"}
RD_VARIANT_AUTO, RD_VARIANT_VECTOR, RD_VARIANT_PAPER, RD_VARIANT_BULK, RD_VARIANT_CLUSTER = 0, 1, 2, 3, 4


class rd_record(ctypes.Structure):
    _fields_ = [("tag", ctypes.c_uint32), ("status", ctypes.c_uint32), ("n", ctypes.c_uint64),
                ("acc", ctypes.c_uint64 * 2)]


class rd_exact_record(ctypes.Structure):
    _fields_ = [("tag", ctypes.c_uint32), ("status", ctypes.c_uint32), ("n", ctypes.c_uint64),
                ("flags", ctypes.c_uint32), ("nwords", ctypes.c_uint32), ("reserved", ctypes.c_uint64),
                ("word", ctypes.c_int64 * RD_EXACT_MAX_WORDS)]


class rd_arg_result(ctypes.Structure):
    _fields_ = [("value", ctypes.c_uint64), ("index", ctypes.c_int64)]


class rd_unique_id(ctypes.Structure):
    _fields_ = [("internal", ctypes.c_char * 128)]


class rd_config(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int32), ("vec_bytes", ctypes.c_int32), ("unroll", ctypes.c_int32),
                ("block", ctypes.c_int32), ("grid", ctypes.c_int32), ("reserved", ctypes.c_int32 * 3)]


class rd_launch_info(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int32), ("vec_bytes", ctypes.c_int32), ("unroll", ctypes.c_int32),
                ("block", ctypes.c_int32), ("grid", ctypes.c_int32), ("regs_per_thread", ctypes.c_int32),
                ("ctas_per_sm", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("head", ctypes.c_uint64), ("nvec", ctypes.c_uint64), ("tail", ctypes.c_uint64)]


# every symbol declared in include/b200reduce.h: name -> (restype, argtypes)
_vp, _sz, _i, _u64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint64
SIGNATURES = {
    "reduce": (_i, [_vp, _sz, _i, _i, _vp, _vp]),
    "reduce_partial": (_i, [_vp, _sz, _i, _i, _vp, _vp]),
    "rd_combine_records": (_i, [_vp, _i, _i, _i, _vp, _vp, _vp, _vp]),
    "reduce_exact_partial": (_i, [_vp, _sz, _i, _vp, _vp]),
    "rd_combine_exact_records": (_i, [_vp, _i, _i, _vp, _vp, _vp, _vp]),
    "reduce_host": (_i, [_vp, _sz, _i, _i, _vp]),
    "rd_get_unique_id": (_i, [ctypes.POINTER(rd_unique_id)]),
    "rd_comm_init": (_i, [ctypes.POINTER(_vp), _i, _i, ctypes.POINTER(rd_unique_id), _i]),
    "rd_comm_destroy": (_i, [_vp]),
    "reduce_multi": (_i, [_vp, _sz, _i, _i, _vp, _vp, _vp]),
    "rd_comm_check": (_i, [_vp, _vp]),
    "rd_shard_range": (_i, [_u64, _i, _i, ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
    "rd_identity": (_i, [_i, _i, _vp]),
    "rd_release_workspaces": (_i, []),
    "rd_status_string": (ctypes.c_char_p, [_i]),
    "rd_last_error": (ctypes.c_char_p, []),
    "rd_reduce_ex": (_i, [_vp, _sz, _i, _i, _vp, _vp, ctypes.POINTER(rd_config),
                          ctypes.POINTER(rd_launch_info)]),
    "rd_fused_create": (_i, [ctypes.POINTER(_vp), _i, _i, _i, _vp]),
    "rd_fused_connect": (_i, [_vp, _vp]),
    "rd_fused_mailbox": (_i, [_vp, ctypes.POINTER(_vp)]),
    "rd_fused_connect_local": (_i, [_vp, ctypes.POINTER(_vp)]),
    "reduce_fused": (_i, [_vp, _sz, _i, _i, _vp, _vp, _vp]),
    "rd_fused_check": (_i, [_vp, _vp]),
    "rd_fused_destroy": (_i, [_vp]),
}

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1710_07358_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class ReduceError(RuntimeError):
    def __init__(self, status: int, where: str):
        detail = lib().rd_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(status, status)}: {detail}")
        self.status = status


def check(status: int, where: str):
    if status != RD_OK:
        raise ReduceError(status, where)
