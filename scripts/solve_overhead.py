"""Host overhead of one solve call: wall time of api.gmres_solve (device idle
before and after) against the device time the library reports (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1909_08734_b200 import api, inputs
P = api.Problem("sphere", h=0.0125, p=3, c=1.0, device_setup=True)
P.decompose(inputs.rcb_partition(P.active_cp, 256), 3, "oras", 4.0, 40.0)
A = api.DeviceHelmholtz.from_problem(P); M = api.SchwarzPreconditioner.from_problem(P)
b = torch.from_numpy(inputs.rhs_sphere(P.active_cp)).cuda()
for _ in range(3): api.gmres_solve(A, b, M, 1e-10, 2000, 50)
torch.cuda.synchronize()
rows = []
for _ in range(10):
    t0 = time.perf_counter(); r = api.gmres_solve(A, b, M, 1e-10, 2000, 50); torch.cuda.synchronize(); t1 = time.perf_counter()
    rows.append((1e3 * (t1 - t0), 1e3 * r.log.device_seconds))
print("wall ms / device ms / difference:")
for w, d in rows: print(f"  {w:8.3f} {d:8.3f} {w - d:7.3f}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
rs = [api.gmres_solve(A, b, M, 1e-10, 2000, 50) for _ in range(10)]
e1.record(); torch.cuda.synchronize()
print("10 solves back to back: events", e0.elapsed_time(e1) / 10, "ms per solve; device", np.mean([1e3 * r.log.device_seconds for r in rs]))
for keep in (True, False, True, False):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    rs, dev = [], []
    for _ in range(10):
        r = api.gmres_solve(A, b, M, 1e-10, 2000, 50)
        dev.append(1e3 * r.log.device_seconds)
        if keep: rs.append(r)
    e1.record(); torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"keep results={keep}: events {e0.elapsed_time(e1) / 10:.3f} ms, wall {1e2 * (t1 - t0):.3f} ms, device {np.mean(dev):.3f} ms per solve")
