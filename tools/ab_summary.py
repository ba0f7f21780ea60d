#!/usr/bin/env python
"""Mean GB/s per (workload, pair, library) of an ab_lib.py JSON-lines log.
    python tools/ab_summary.py gpurun_out/ab_fair.jsonl"""
import collections
import json
import sys

d = collections.defaultdict(list)
for line in open(sys.argv[1]):
    r = json.loads(line)
    for k, v in r.items():
        if k not in ("wl", "lib", "round"):
            d[(r.get("wl", ""), k, r["lib"])].append(v)
for k in sorted(d):
    print(*k, [round(x) for x in d[k]], "mean", round(sum(d[k]) / len(d[k]), 1))
