import ctypes, json, os, sys
import torch
L = ctypes.CDLL(sys.argv[1])
L.reduce.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
out = torch.empty(2, dtype=torch.int64, device="cuda")
res = {}
DT = int(os.environ.get("AB_DT", "3"))
for log2n in [int(v) for v in os.environ.get("AB_LOG2N", "14,16,18").split(",")]:
    x = torch.rand(1 << log2n, device="cuda", dtype=torch.float64 if DT == 4 else torch.float32)
    gs = torch.cuda.Stream()
    with torch.cuda.stream(gs):
        L.reduce(x.data_ptr(), x.numel(), DT, 10, out.data_ptr(), gs.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gs):
        for _ in range(100):
            L.reduce(x.data_ptr(), x.numel(), DT, 10, out.data_ptr(), gs.cuda_stream)
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) * 10.0)
    res[f"2^{log2n}"] = round(sorted(ts)[3], 3)
print(json.dumps({"lib": os.path.relpath(sys.argv[1]), "dt": DT, **res}))
