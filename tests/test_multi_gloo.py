"""Multi-process host logic of the sharded path, world size 2,
gloo on CPU: the canonical contiguous split (rd_shard_range from the C
library), per-rank partials exchanged over the process group, the rank-order
fold, dtype/op mismatch detection, and the NCCL unique-id broadcast that
Comm.from_process_group performs. The device side of reduce_multi (NCCL
all-gather + rd_combine_kernel) is covered by the GPU tests."""
from __future__ import annotations

import ctypes
import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = [("int32", "sum", "uniform_bits"), ("uint32", "and", "sparse_clear"), ("int64", "prod", "odd"),
         ("float32", "sum", "u01"), ("float64", "sum", "normalish"), ("float32", "max", "planted"),
         ("float64", "prod", "near_one"), ("int32", "xor", "uniform_bits"),
         # exact sums (reading R17): the rank-order merge of exact partials is bit-exact
         ("float32", "sum_exact", "wide"), ("float64", "sum_exact", "wide_full")]


def _worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import inputs
    import oracle
    import paper_1710_07358_b200 as rd
    dist.init_process_group("gloo", rank=rank, world_size=world)
    results = {}
    for n in (0, 1, 7, 1000, 5533214):
        for dtype, op, wl in CASES:
            b, c = rd.shard_range(n, world, rank)
            shard = inputs.generate(c, dtype, wl, seed=3, offset=b, n_total=n)
            f = oracle.Fold(dtype, op).fold(shard)
            blob = bytes(ctypes.string_at(ctypes.addressof(f.st), ctypes.sizeof(f.st)))
            gathered = [None] * world
            dist.all_gather_object(gathered, (rank, b, c, blob))
            # rank-order fold of the exchanged partials (the exchange step of reduce_multi)
            gathered.sort()
            acc = oracle.Fold(dtype, op)
            pos = 0
            for r, bb, cc, bl in gathered:
                assert bb == pos
                pos += cc
                g = oracle.Fold(dtype, op)
                ctypes.memmove(ctypes.addressof(g.st), bl, len(bl))
                acc.merge(g)
            assert pos == n
            res = acc.result()
            results[(n, dtype, op)] = (res.value.tobytes(), res.exact, res.sum_abs)
    # a rank that disagrees on the op must be detected when the partials are folded
    f = oracle.Fold("float32", "sum" if rank == 0 else "max").fold(np.ones(4, np.float32))
    blob = bytes(ctypes.string_at(ctypes.addressof(f.st), ctypes.sizeof(f.st)))
    gathered = [None] * world
    dist.all_gather_object(gathered, blob)
    acc = oracle.Fold("float32", "sum")
    mismatch = False
    for bl in gathered:
        g = oracle.Fold("float32", "sum")
        ctypes.memmove(ctypes.addressof(g.st), bl, len(bl))
        try:
            acc.merge(g)
        except oracle.OracleError:
            mismatch = True
    # FusedComm.from_process_group is collective-safe: with no GPU here mailbox
    # creation fails, and every rank raises (none is left waiting in an exchange)
    fused_raised = False
    try:
        rd.FusedComm.from_process_group(device=0)
    except rd.ReduceError:
        fused_raised = True
    # NCCL unique id broadcast (what Comm.from_process_group does before rd_comm_init)
    uid = rd.broadcast_unique_id()
    uid_bytes = ctypes.string_at(ctypes.addressof(uid), 128)
    ids = [None] * world
    dist.all_gather_object(ids, uid_bytes)
    import pickle
    with open(os.path.join(outdir, f"rank{rank}.pkl"), "wb") as fh:
        pickle.dump({"results": results, "mismatch": mismatch, "ids": ids, "fused_raised": fused_raised}, fh)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_exchange_and_rank_order_fold():
    sys.path.insert(0, ROOT)
    import pickle
    import inputs
    import oracle
    from paper_1710_07358_b200.build import build_library
    build_library()
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, _free_port(), d), nprocs=world, join=True,
                           start_method="spawn")
        outs = [pickle.load(open(os.path.join(d, f"rank{r}.pkl"), "rb")) for r in range(world)]
    # every rank got the identical folded result
    assert outs[0]["results"] == outs[1]["results"]
    for (n, dtype, op), (vbytes, exact, sabs) in outs[0]["results"].items():
        wl = [c[2] for c in [x for x in CASES if x[0] == dtype and x[1] == op]][0]
        x = inputs.generate(n, dtype, wl, seed=3)
        full = oracle.reduce(x, op)
        if dtype.startswith("float") and op in ("sum", "prod"):
            scale = full.sum_abs if op == "sum" else abs(full.exact)
            eps = 2.0 ** -23 if dtype == "float32" else 2.0 ** -52
            assert abs(exact - full.exact) <= 4 * eps * scale, (n, dtype, op)
        else:
            assert vbytes == full.value.tobytes(), (n, dtype, op)
    assert outs[0]["mismatch"] and outs[1]["mismatch"]
    assert outs[0]["fused_raised"] and outs[1]["fused_raised"]
    assert outs[0]["ids"][0] == outs[0]["ids"][1] == outs[1]["ids"][0]
    assert outs[0]["ids"][0] != bytes(128)
