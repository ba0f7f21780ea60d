#!/usr/bin/env python
"""Sharded reduction, one process per GPU:

    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \\
        examples/multi_gpu_reduce.py [--log2n 30] [--op sum]

Each rank generates its contiguous block of one logical float32 array
(rd.shard_range), then reduces it with both exchange paths:
  * rd.Comm      -- reduce kernel + NCCL all-gather of 32-byte records + rank-order fold
  * rd.FusedComm -- the exchange inside the reduce kernel (peer stores over NVLink)
Both give the bitwise-identical result on every rank.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import inputs  # noqa: E402
import paper_1710_07358_b200 as rd  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--log2n", type=int, default=28)
    p.add_argument("--op", default="sum")
    args = p.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    n = 1 << args.log2n
    begin, count = rd.shard_range(n, world, rank)
    x = torch.empty(count, dtype=torch.float32, device="cuda")
    inputs.fill_device(x, "u01", seed=1, offset=begin, n_total=n)

    nccl = rd.Comm.from_process_group()
    fused = rd.FusedComm.from_process_group()
    a = nccl.reduce(x, args.op)
    b = fused.reduce(x, args.op)
    nccl.check()
    fused.check()
    same = a.item() == b.item()
    if rank == 0:
        print(f"{world} rank(s), n = 2^{args.log2n}: {args.op} = {a.item()!r} (NCCL) "
              f"{b.item()!r} (fused)  identical={same}")
    dist.barrier()
    fused.destroy()
    nccl.destroy()
    dist.destroy_process_group()
    sys.exit(0 if same else 1)


if __name__ == "__main__":
    main()
