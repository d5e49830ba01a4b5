"""Wall/device time of small solves with and without kernel profiling (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1909_08734_b200 import api, inputs
P = api.Problem("circle", h=0.0125, p=3, c=1.0)
cp = P.active_cp
P.decompose(inputs.sector_partition(cp, 8), 2, "oras", 1.0, -1.0)
A = api.DeviceHelmholtz.from_problem(P); M = api.SchwarzPreconditioner.from_problem(P)
b = torch.from_numpy(inputs.rhs_circle(cp)).cuda()
for prof in (False, True, False, True):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rs = [api.gmres_solve(A, b, M, 1e-10, 2000, 50, profile=prof) for _ in range(5)]
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"profile={prof}: wall {1e3 * (t1 - t0) / 5:.2f} ms/solve, device {[round(r.log.device_seconds * 1e3, 2) for r in rs]}, its {rs[0].log.iterations}")
