"""Row-layout vs column-layout backward: agreement and timing (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08734_b200 import api, inputs
h = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0125
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 256
P = api.Problem("sphere", h=h, p=3, c=1.0)
P.decompose(inputs.rcb_partition(P.active_cp, ns), 3, "oras", 4.0, 40.0)
Ms = {}
for lay in ("rows", "cols"):
    os.environ["CPDDG_BWD_LAYOUT"] = lay
    Ms[lay] = api.SchwarzPreconditioner.from_problem(P)
x = torch.from_numpy(inputs.uniform_vector(P.n_active, 1)).cuda()
zr, zc = Ms["rows"].apply(x), Ms["cols"].apply(x)
print("rel diff cols vs rows:", float((zr - zc).norm() / zr.norm()))
for lay, M in Ms.items():
    for _ in range(3): M.apply(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): M.apply(x)
    e1.record(); torch.cuda.synchronize()
    print(f"{lay}: {e0.elapsed_time(e1) / 10:.3f} ms  stats {M.stats()['factor_bytes'] / 1e9:.2f} GB")
