#!/usr/bin/env python
"""Time RD_SUM_EXACT at n = 2^28 for each (dtype, workload) in THIS process's
kernel configuration (RD_TUNE_EXACT="U,E,M" selects it); one JSON line each.

    for c in 2,2,1 4,2,3; do RD_TUNE_EXACT=$c python tools/tune_exact.py; done
    for c in 16,2 24,1; do RD_TUNE_EXACT_BULK=$c python tools/tune_exact.py --variant bulk; done
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import paper_1710_07358_b200 as rd  # noqa: E402
from sweep import make, time_launch  # noqa: E402

if __name__ == "__main__":
    variant = sys.argv[sys.argv.index("--variant") + 1] if "--variant" in sys.argv else "vector"
    cfg = os.environ.get("RD_TUNE_EXACT_BULK" if variant == "bulk" else "RD_TUNE_EXACT", "default")
    n = 1 << 28
    for dtype in ("float32", "float64"):
        for wl in ("u01", "normalish", "wide"):
            x = make(n, dtype, wl)
            o = torch.empty((), dtype=x.dtype, device="cuda")
            _, info = rd.reduce_ex(x, "sum_exact", variant=variant, out=o)
            r = time_launch(lambda: rd.reduce_ex(x, "sum_exact", variant=variant, out=o), n * x.element_size(),
                            reps=10)
            r.update({"cfg": f"{variant}:{cfg}", "dtype": dtype, "workload": wl,
                      "regs": info["regs_per_thread"], "ctas_per_sm": info["ctas_per_sm"]})
            print(json.dumps(r), flush=True)
            del x
