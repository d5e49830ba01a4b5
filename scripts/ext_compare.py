"""Staged vs gather extension kernel: bit-identity and timing (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08734_b200 import api

h = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0125
P = api.Problem("sphere", h=h, p=3, c=1.0)
os.environ["CPDDG_EXT_GATHER"] = "1"
Ag = api.DeviceHelmholtz.from_problem(P)
del os.environ["CPDDG_EXT_GATHER"]
As = api.DeviceHelmholtz.from_problem(P)
x = torch.rand(P.n_active, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
yg, ys = Ag.apply(x), As.apply(x)
print("bit-identical:", bool(torch.equal(yg, ys)), "max diff", float((yg - ys).abs().max()))
for name, A in (("gather", Ag), ("staged", As)):
    for _ in range(5):
        A.apply(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        A.apply(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    alg, stream = A.bytes()
    print(f"{name}: {ms * 1e3:.1f} us/apply  alg {alg / 1e6:.1f} MB ({alg / ms / 1e9:.0f} GB/s) streamed {stream / 1e6:.1f} MB")
