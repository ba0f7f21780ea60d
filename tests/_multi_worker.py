"""One rank of the multi-GPU parity run (tests/test_gpu_multi.py launches it with
torch.distributed.run, one process per GPU). Rank r holds the r-th contiguous
block (rd.shard_range) of each logical array; reduce_multi (NCCL all-gather of
records + rank-order fold) and reduce_fused (the exchange inside the reduce
kernel, peer stores over NVLink) must give the bitwise-identical result on every
rank, equal to the oracle on the whole array. Exit code 0 = all
checks passed."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import inputs  # noqa: E402
import paper_1710_07358_b200 as rd  # noqa: E402
from tests import _parity  # noqa: E402

CASES = [("float32", "sum", (1 << 24) + 7), ("float32", "max", (1 << 22) + 3), ("int32", "xor", 5533214),
         ("float64", "sum", (1 << 21) + 1), ("float32", "sum_exact", (1 << 22) + 9),
         ("float64", "sum_exact", 100003), ("float32", "argmin", (1 << 20) + 5), ("int64", "prod", 4099),
         ("uint32", "min", 7), ("float32", "sum", 0)]


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    nccl = rd.Comm.from_process_group()
    fused = rd.FusedComm.from_process_group()
    failures = []
    for dtype, op, n in CASES:
        wl = inputs.default_workload(dtype, op) if op != "sum_exact" else "wide"
        b, c = rd.shard_range(n, world, rank)
        x = torch.empty(c, dtype=getattr(torch, dtype), device=dev)
        inputs.fill_device(x, wl, seed=7, offset=b, n_total=n)
        outs = []
        for cm in (nccl, fused):
            r = cm.reduce(x, op)
            cm.check()
            r = r if isinstance(r, tuple) else (r,)
            outs.append(b"".join(bytes(t.reshape(1).view(torch.uint8).cpu().numpy()) for t in r))
        gathered = [None] * world
        dist.all_gather_object(gathered, outs)
        if any(g != gathered[0] for g in gathered) or gathered[0][0] != gathered[0][1]:
            failures.append(f"{dtype} {op} n={n}: ranks/paths differ {gathered}")
            continue
        if rank == 0:
            xh = inputs.generate(n, dtype, wl, seed=7)
            raw = gathered[0][0]
            s = np.dtype(dtype).itemsize
            try:
                if op in ("argmin", "argmax"):
                    v = np.frombuffer(raw[:s], dtype)[0]
                    i = int(np.frombuffer(raw[s:s + 8], np.int64)[0])
                    _parity.check((v, i), xh, op)
                else:
                    _parity.check(np.frombuffer(raw, dtype)[0], xh, op)
            except AssertionError as e:
                failures.append(f"{dtype} {op} n={n}: {e}")
    # ranks that disagree on the op: every rank reports RD_ERR_MISMATCH (both paths)
    if world >= 2:
        x = torch.ones(1000, dtype=torch.float32, device=dev)
        for cm in (nccl, fused):
            op = "sum" if rank == 0 else ("sum_exact" if cm is fused else "max")
            cm.reduce(x, op)
            try:
                cm.check()
                failures.append(f"rank {rank}: mismatch not reported ({type(cm).__name__})")
            except rd.ReduceError as e:
                if e.status != 6:
                    failures.append(f"rank {rank}: status {e.status} instead of RD_ERR_MISMATCH")
    flags = [None] * world
    dist.all_gather_object(flags, failures)
    dist.barrier()
    torch.cuda.synchronize()
    fused.destroy()
    nccl.destroy()
    dist.destroy_process_group()
    bad = [f for fl in flags for f in fl]
    if rank == 0:
        print(f"{world} rank(s): {len(CASES)} cases, {len(bad)} failure(s)")
        for f in bad:
            print("FAIL", f)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
