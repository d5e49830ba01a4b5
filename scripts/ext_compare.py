"""Extension kernels (union default, grouped, staged, gather): bit-identity and timing
of A x at one sphere size (development aid).  Usage: ext_compare.py [h]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08734_b200 import api

h = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0125
P = api.Problem("sphere", h=h, p=3, c=1.0)
ops = {}
for name, env in (("gather", {"CPDDG_EXT_GATHER": "1"}), ("staged", {"CPDDG_EXT": "staged"}),
                  ("grouped", {"CPDDG_EXT": "grouped"}), ("union", {})):
    for k, v in env.items():
        os.environ[k] = v
    ops[name] = api.DeviceHelmholtz.from_problem(P)
    for k in env:
        del os.environ[k]
x = torch.rand(P.n_active, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
ys = {k: A.apply(x) for k, A in ops.items()}
for k in ("staged", "grouped", "union"):
    print(f"{k} vs gather bit-identical:", bool(torch.equal(ys["gather"], ys[k])),
          "max diff", float((ys["gather"] - ys[k]).abs().max()))
for name, A in ops.items():
    # 100 applies captured in one CUDA graph: device time without Python
    # launch overhead
    y = torch.empty_like(x)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            A.apply(x, out=y)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(100):
            A.apply(x, out=y)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 500
    alg, stream = A.bytes()
    print(f"{name}: {ms * 1e3:.1f} us/apply  alg {alg / 1e6:.1f} MB ({alg / ms / 1e6:.0f} GB/s) "
          f"streamed {stream / 1e6:.1f} MB ({stream / ms / 1e6:.0f} GB/s)")
