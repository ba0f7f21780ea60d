"""Small inputs: AUTO's plan vs the one-cluster kernel forced to 8 / 16 CTAs,
graph-captured us per launch (the evidence for kClusterMaxBytes)."""
import sys, os, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch
import paper_1710_07358_b200 as rd
from sweep import graph_us, make
for log2n in (16, 17, 18, 19, 20, 21):
    for dt in ("float32", "float64"):
        n = 1 << log2n
        x = make(n, dt, "u01")
        o = torch.empty((), dtype=x.dtype, device="cuda")
        r = {"log2n": log2n, "dtype": dt, "auto": graph_us(lambda: rd.reduce(x, "sum", out=o)),
             "auto_plan": rd.reduce_ex(x, "sum", out=o)[1]["variant"] + ":" + str(rd.reduce_ex(x, "sum", out=o)[1]["grid"])}
        for g in (8, 16):
            r[f"cluster{g}"] = graph_us(lambda: rd.reduce_ex(x, "sum", variant="cluster", grid=g, out=o))
        print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
