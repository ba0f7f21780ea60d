"""paper_1710_07358_b200 -- B200-native (sm_100a) parallel reduction.

Python binding of the C ABI in ``include/b200reduce.h`` (argument marshalling
only; every step of the reduction runs in ``libb200reduce.so``). PyTorch is
used for device memory, streams and process groups.

    import torch, paper_1710_07358_b200 as rd
    x = torch.rand(1 << 28, device="cuda")
    s = rd.reduce(x, "sum")          # 0-d tensor on x.device

The operation is x_0 (x) x_1 (x) ... (x) x_{n-1} for
(x) in {sum, prod, min, max, and, or, xor} over int32/uint32/int64/float32/
float64; semantics and tolerances are stated in include/b200reduce.h.
"""
from __future__ import annotations

import contextlib
import ctypes

import numpy as np

from . import _lib
from ._lib import ReduceError, check, lib

__all__ = ["reduce", "reduce_partial", "combine_records", "reduce_exact_partial", "combine_exact_records",
           "reduce_host", "reduce_ex",
           "reduce_multi", "Comm", "FusedComm", "shard_range", "identity", "release_workspaces",
           "ReduceError", "OPS", "RECORD_BYTES", "EXACT_RECORD_BYTES"]

OPS = {"sum": _lib.RD_SUM, "prod": _lib.RD_PROD, "min": _lib.RD_MIN, "max": _lib.RD_MAX,
       "and": _lib.RD_AND, "or": _lib.RD_OR, "xor": _lib.RD_XOR,
       "argmin": _lib.RD_ARGMIN, "argmax": _lib.RD_ARGMAX, "sum_compensated": _lib.RD_SUM_COMPENSATED,
       "sum_exact": _lib.RD_SUM_EXACT}
ARG_OPS = ("argmin", "argmax")
DTYPE_NAMES = {"int32": _lib.RD_INT32, "uint32": _lib.RD_UINT32, "int64": _lib.RD_INT64,
               "float32": _lib.RD_FLOAT32, "float64": _lib.RD_FLOAT64}
RECORD_BYTES = 32
EXACT_RECORD_BYTES = ctypes.sizeof(_lib.rd_exact_record)   # 608
VARIANTS = {"auto": _lib.RD_VARIANT_AUTO, "vector": _lib.RD_VARIANT_VECTOR, "paper": _lib.RD_VARIANT_PAPER,
            "bulk": _lib.RD_VARIANT_BULK, "cluster": _lib.RD_VARIANT_CLUSTER}


def _torch():
    import torch
    return torch


def _dtype_name(dt) -> str:
    s = str(dt)
    return s.replace("torch.", "")


_DT_CACHE = {}


def _dt(t) -> int:
    code = _DT_CACHE.get(t.dtype)
    if code is None:
        name = _dtype_name(t.dtype)
        if name not in DTYPE_NAMES:
            raise TypeError(f"unsupported dtype {t.dtype}")
        code = _DT_CACHE[t.dtype] = DTYPE_NAMES[name]
    return code


def _op(op: str) -> int:
    if op not in OPS:
        raise ValueError(f"unknown op {op!r}; expected one of {sorted(OPS)}")
    return OPS[op]


def _stream(t, stream):
    if stream is None:
        torch = _torch()
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        if raw is not None:
            return raw(t.device.index)
        return torch.cuda.current_stream(t.device).cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _new_out(dtype, device, op):
    """Result buffer: one element, or a 16-byte rd_arg_result for argmin/argmax."""
    torch = _torch()
    if op in ARG_OPS:
        return torch.empty(2, dtype=torch.int64, device=device)
    return torch.empty((), dtype=dtype, device=device)


def _check_out(out, dtype, op):
    """The result buffer must be large enough for what the C call writes."""
    if op in ARG_OPS:
        if out.numel() * out.element_size() < 16 or not out.is_contiguous():
            raise ValueError("argmin/argmax need a 16-byte rd_arg_result buffer (e.g. 2 x int64)")
    elif out.dtype != dtype:
        raise ValueError(f"out has dtype {out.dtype}, expected {dtype}")
    return out


def _arg_view(buf, dtype):
    """rd_arg_result buffer (2 x int64) -> (value 0-d tensor of dtype, index 0-d int64).
    The value's bits are the low sizeof(dtype) bytes of word 0 (little endian), i.e.
    element 0 of the buffer viewed as dtype (two view ops: ~5 us of host time per
    call instead of ~21 us for a byte-slicing view chain)."""
    return buf.view(dtype)[0], buf[1]


def _result(out, dtype, op):
    return _arg_view(out, dtype) if op in ARG_OPS else out


def _dev_guard(t):
    """The C library launches on the CURRENT device: make it t's device."""
    torch = _torch()
    idx = t.device.index
    if idx is None or idx == torch.cuda.current_device():
        return contextlib.nullcontext()
    return torch.cuda.device(idx)


def _check_input(x):
    if not x.is_cuda:
        raise ValueError("x must be a CUDA tensor (use reduce_host for host arrays)")
    if not x.is_contiguous():
        raise ValueError("x must be contiguous")


def reduce(x, op: str, out=None, stream=None):
    """x_0 (x) ... (x) x_{n-1} over all elements of the contiguous CUDA tensor x.
    Returns a 0-d tensor; for "argmin"/"argmax" a (value, index) pair of 0-d
    tensors (views of one 16-byte rd_arg_result; `out` is then 2 x int64)."""
    _check_input(x)
    out = _new_out(x.dtype, x.device, op) if out is None else _check_out(out, x.dtype, op)
    with _dev_guard(x):
        check(lib().reduce(x.data_ptr() if x.numel() else None, x.numel(), _dt(x), _op(op),
                           out.data_ptr(), _stream(x, stream)), "reduce")
    return _result(out, x.dtype, op)


def reduce_partial(x, op: str, rec=None, stream=None):
    """Un-narrowed partial of x as one 32-byte rd_record (uint8 CUDA tensor)."""
    torch = _torch()
    _check_input(x)
    if rec is None:
        rec = torch.empty(RECORD_BYTES, dtype=torch.uint8, device=x.device)
    with _dev_guard(x):
        check(lib().reduce_partial(x.data_ptr() if x.numel() else None, x.numel(), _dt(x), _op(op),
                                   rec.data_ptr(), _stream(x, stream)), "reduce_partial")
    return rec


def combine_records(recs, dtype, op: str, out=None, rec_out=None, status=None, stream=None):
    """Fold k records (a uint8 CUDA tensor of k*32 bytes) in index order."""
    torch = _torch()
    name = _dtype_name(dtype)   # accepts a torch dtype or its name
    tdt = getattr(torch, name)
    if recs.numel() % RECORD_BYTES:
        raise ValueError("recs must hold whole 32-byte records")
    if out is None and rec_out is None:
        out = _new_out(tdt, recs.device, op)
    elif out is not None:
        _check_out(out, tdt, op)
    with _dev_guard(recs):
        check(lib().rd_combine_records(recs.data_ptr() if recs.numel() else None, recs.numel() // RECORD_BYTES,
                                       DTYPE_NAMES[name], _op(op),
                                       out.data_ptr() if out is not None else None,
                                       rec_out.data_ptr() if rec_out is not None else None,
                                       status.data_ptr() if status is not None else None,
                                       _stream(recs, stream)), "rd_combine_records")
    return _result(out, tdt, op) if out is not None else rec_out


def reduce_exact_partial(x, rec=None, stream=None):
    """Exact partial sum of a float CUDA tensor (RD_SUM_EXACT) as one 608-byte
    rd_exact_record (uint8 CUDA tensor)."""
    torch = _torch()
    _check_input(x)
    if rec is None:
        rec = torch.empty(EXACT_RECORD_BYTES, dtype=torch.uint8, device=x.device)
    with _dev_guard(x):
        check(lib().reduce_exact_partial(x.data_ptr() if x.numel() else None, x.numel(), _dt(x),
                                         rec.data_ptr(), _stream(x, stream)), "reduce_exact_partial")
    return rec


def combine_exact_records(recs, dtype, out=None, rec_out=None, status=None, stream=None):
    """Add k exact records (a uint8 CUDA tensor of k*608 bytes) and round once."""
    torch = _torch()
    name = _dtype_name(dtype)
    tdt = getattr(torch, name)
    if recs.numel() % EXACT_RECORD_BYTES:
        raise ValueError("recs must hold whole 608-byte exact records")
    if out is None and rec_out is None:
        out = torch.empty((), dtype=tdt, device=recs.device)
    elif out is not None and out.dtype != tdt:
        raise ValueError(f"out has dtype {out.dtype}, expected {tdt}")
    with _dev_guard(recs):
        check(lib().rd_combine_exact_records(recs.data_ptr() if recs.numel() else None,
                                             recs.numel() // EXACT_RECORD_BYTES, DTYPE_NAMES[name],
                                             out.data_ptr() if out is not None else None,
                                             rec_out.data_ptr() if rec_out is not None else None,
                                             status.data_ptr() if status is not None else None,
                                             _stream(recs, stream)), "rd_combine_exact_records")
    return out if out is not None else rec_out


def reduce_host(x, op: str):
    """End-to-end reduction of a host array (numpy array or CPU tensor; pinned
    memory gives overlapped copies). Returns a numpy scalar ((value, index)
    for argmin / argmax)."""
    if isinstance(x, np.ndarray):
        arr = np.ascontiguousarray(x)
        name, ptr, n = arr.dtype.name, arr.ctypes.data, arr.size
    else:
        if x.is_cuda or not x.is_contiguous():
            raise ValueError("reduce_host takes a contiguous host tensor")
        name, ptr, n = _dtype_name(x.dtype), x.data_ptr(), x.numel()
    if name not in DTYPE_NAMES:
        raise TypeError(f"unsupported dtype {name}")
    if op in ARG_OPS:
        r = _lib.rd_arg_result()
        check(lib().reduce_host(ptr if n else None, n, DTYPE_NAMES[name], _op(op), ctypes.addressof(r)),
              "reduce_host")
        v = np.array([r.value], dtype=np.uint64).view(np.uint8)[:np.dtype(name).itemsize].view(np.dtype(name))[0]
        return v, int(r.index)
    out = np.zeros(1, dtype=np.dtype(name))
    check(lib().reduce_host(ptr if n else None, n, DTYPE_NAMES[name], _op(op), out.ctypes.data),
          "reduce_host")
    return out[0]


def reduce_ex(x, op: str, variant: str = "auto", unroll: int = 0, vec_bytes: int = 0, grid: int = 0,
              out=None, stream=None):
    """reduce with an explicit kernel configuration; returns (out, info dict)."""
    _check_input(x)
    out = _new_out(x.dtype, x.device, op) if out is None else _check_out(out, x.dtype, op)
    cfg = _lib.rd_config(VARIANTS[variant], vec_bytes, unroll, 0, grid)
    info = _lib.rd_launch_info()
    with _dev_guard(x):
        check(lib().rd_reduce_ex(x.data_ptr() if x.numel() else None, x.numel(), _dt(x), _op(op),
                                 out.data_ptr(), _stream(x, stream), ctypes.byref(cfg), ctypes.byref(info)),
              "rd_reduce_ex")
    d = {k: getattr(info, k) for k, _ in _lib.rd_launch_info._fields_ if k != "reserved"}
    d["variant"] = {v: k for k, v in VARIANTS.items()}[d["variant"]]
    return _result(out, x.dtype, op), d


def shard_range(n: int, nranks: int, rank: int):
    """Canonical contiguous split of n elements over nranks: (begin, count)."""
    b, c = ctypes.c_uint64(), ctypes.c_uint64()
    check(lib().rd_shard_range(n, nranks, rank, ctypes.byref(b), ctypes.byref(c)), "rd_shard_range")
    return b.value, c.value


def identity(dtype, op: str):
    """The empty-input result (include/b200reduce.h table) as a numpy scalar;
    (value, -1) for argmin / argmax."""
    name = _dtype_name(dtype)
    if op in ARG_OPS:
        r = _lib.rd_arg_result()
        check(lib().rd_identity(DTYPE_NAMES[name], _op(op), ctypes.addressof(r)), "rd_identity")
        v = np.array([r.value], dtype=np.uint64).view(np.uint8)[:np.dtype(name).itemsize].view(np.dtype(name))[0]
        return v, int(r.index)
    out = np.zeros(1, dtype=np.dtype(name))
    check(lib().rd_identity(DTYPE_NAMES[name], _op(op), out.ctypes.data), "rd_identity")
    return out[0]


def release_workspaces():
    check(lib().rd_release_workspaces(), "rd_release_workspaces")


def broadcast_unique_id(group=None):
    """rank 0 of the process group draws an NCCL unique id (rd_get_unique_id);
    every rank returns the same 128 bytes as an rd_unique_id."""
    import torch.distributed as dist
    uid = _lib.rd_unique_id()
    if dist.get_rank(group) == 0:
        check(lib().rd_get_unique_id(ctypes.byref(uid)), "rd_get_unique_id")
    # the raw 128 bytes (uid.internal would stop at the first NUL)
    obj = [ctypes.string_at(ctypes.addressof(uid), 128) if dist.get_rank(group) == 0 else None]
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(obj, src=src, group=group)
    ctypes.memmove(ctypes.addressof(uid), obj[0], 128)
    return uid


class Comm:
    """One NCCL communicator per process/GPU for reduce_multi."""

    def __init__(self, handle: int, nranks: int, rank: int, device: int):
        self.handle, self.nranks, self.rank, self.device = handle, nranks, rank, device

    @classmethod
    def from_process_group(cls, group=None, device: int | None = None) -> "Comm":
        """Create the communicator: rank 0 draws the NCCL unique id, which is
        broadcast over the torch.distributed process group."""
        torch = _torch()
        import torch.distributed as dist
        rank, nranks = dist.get_rank(group), dist.get_world_size(group)
        dev = torch.cuda.current_device() if device is None else device
        uid = broadcast_unique_id(group)
        h = ctypes.c_void_p()
        check(lib().rd_comm_init(ctypes.byref(h), nranks, rank, ctypes.byref(uid), dev), "rd_comm_init")
        return cls(h.value, nranks, rank, dev)

    def reduce(self, x_local, op: str, out=None, stream=None):
        return reduce_multi(x_local, op, self, out=out, stream=stream)

    def check(self, stream=None):
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        st = st.cuda_stream if hasattr(st, "cuda_stream") else st
        check(lib().rd_comm_check(self.handle, st), "rd_comm_check")

    def destroy(self):
        if self.handle:
            check(lib().rd_comm_destroy(self.handle), "rd_comm_destroy")
            self.handle = None


def reduce_multi(x_local, op: str, comm: Comm, out=None, stream=None):
    """Sharded reduce: every rank passes its contiguous block (rank order);
    every rank receives the bitwise-identical result."""
    _check_input(x_local)
    out = _new_out(x_local.dtype, x_local.device, op) if out is None else _check_out(out, x_local.dtype, op)
    with _dev_guard(x_local):
        check(lib().reduce_multi(x_local.data_ptr() if x_local.numel() else None, x_local.numel(),
                                 _dt(x_local), _op(op), out.data_ptr(), _stream(x_local, stream),
                                 comm.handle), "reduce_multi")
    return _result(out, x_local.dtype, op)


class FusedComm:
    """Multi-GPU reduction with the exchange fused into the reduce kernel
    (include/b200reduce.h reduce_fused): one launch per rank, peer
    stores over NVLink into CUDA-IPC-mapped mailboxes, rank-order fold."""

    def __init__(self, handle: int, nranks: int, rank: int, device: int):
        self.handle, self.nranks, self.rank, self.device = handle, nranks, rank, device

    @classmethod
    def _create(cls, nranks: int, rank: int, device: int, want_ipc: bool):
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(64) if want_ipc else None
        check(lib().rd_fused_create(ctypes.byref(h), nranks, rank, device, buf), "rd_fused_create")
        return cls(h.value, nranks, rank, device), (buf.raw if want_ipc else None)

    @classmethod
    def from_process_group(cls, group=None, device: int | None = None) -> "FusedComm":
        """One process per GPU: exchange the mailboxes' IPC handles over the group.
        Collective: it either succeeds on every rank or raises on every rank
        (a rank that cannot create or map a mailbox never leaves its peers
        waiting in a later exchange)."""
        torch = _torch()
        import torch.distributed as dist
        rank, nranks = dist.get_rank(group), dist.get_world_size(group)
        dev = torch.cuda.current_device() if device is None else device
        comm, mine, err = None, None, None
        try:
            comm, mine = cls._create(nranks, rank, dev, True)
        except ReduceError as e:
            err = e
        handles = [None] * nranks
        dist.all_gather_object(handles, mine, group=group)
        ok = err is None and all(h is not None for h in handles)
        if ok:
            try:
                check(lib().rd_fused_connect(comm.handle, b"".join(handles)), "rd_fused_connect")
            except ReduceError as e:
                err, ok = e, False
        flags = [None] * nranks
        dist.all_gather_object(flags, ok, group=group)
        if not all(flags):
            if comm is not None:
                comm.destroy()
            raise ReduceError(int(err.status) if err is not None else 4,
                              f"FusedComm.from_process_group (rank {rank}: {err}; ranks ok: {flags})")
        return comm

    @classmethod
    def local(cls, nranks: int, device: int = 0, devices=None) -> list:
        """nranks virtual ranks in this process (tests, or several devices driven
        by one process): mailboxes are connected by device pointer; rank r's
        mailbox lives on devices[r] (default: all on `device`)."""
        devs = list(devices) if devices is not None else [device] * nranks
        if len(devs) != nranks:
            raise ValueError("devices must list one device per rank")
        comms = [cls._create(nranks, r, devs[r], False)[0] for r in range(nranks)]
        ptrs = (ctypes.c_void_p * nranks)()
        for r, c in enumerate(comms):
            p = ctypes.c_void_p()
            check(lib().rd_fused_mailbox(c.handle, ctypes.byref(p)), "rd_fused_mailbox")
            ptrs[r] = p
        for c in comms:
            check(lib().rd_fused_connect_local(c.handle, ptrs), "rd_fused_connect_local")
        return comms

    def reduce(self, x_local, op: str, out=None, stream=None):
        _check_input(x_local)
        out = _new_out(x_local.dtype, x_local.device, op) if out is None else _check_out(out, x_local.dtype, op)
        with _dev_guard(x_local):
            check(lib().reduce_fused(x_local.data_ptr() if x_local.numel() else None, x_local.numel(),
                                     _dt(x_local), _op(op), out.data_ptr(), _stream(x_local, stream),
                                     self.handle), "reduce_fused")
        return _result(out, x_local.dtype, op)

    def check(self, stream=None):
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        st = st.cuda_stream if hasattr(st, "cuda_stream") else st
        check(lib().rd_fused_check(self.handle, st), "rd_fused_check")

    def destroy(self):
        if self.handle:
            check(lib().rd_fused_destroy(self.handle), "rd_fused_destroy")
            self.handle = None
