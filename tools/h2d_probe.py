#!/usr/bin/env python
"""PCIe host->device ceiling for the e2e leg: pinned 1 GiB copies with torch
(one stream; two streams; chunked), next to reduce_host itself."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1710_07358_b200 as rd  # noqa: E402

n = 1 << 28
h = torch.empty(n, dtype=torch.float32, pin_memory=True).uniform_()
d = torch.empty(n, dtype=torch.float32, device="cuda")
res = {}


def timeit(name, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    res[name] = round(n * 4 * reps / (time.perf_counter() - t) / 1e9, 2)


timeit("torch_copy_1stream_1GiB", lambda: d.copy_(h, non_blocking=True))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def two():
    half = n // 2
    with torch.cuda.stream(s1):
        d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        d[half:].copy_(h[half:], non_blocking=True)


timeit("torch_copy_2streams_1GiB", two)
timeit("reduce_host_1GiB", lambda: rd.reduce_host(h, "sum"))
print(json.dumps(res))
