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
# outliers over many calls: where does a stalled call spend its time?
torch.cuda.synchronize()
ts = []
for _ in range(150):
    t0 = time.perf_counter(); r = api.gmres_solve(A, b, M, 1e-10, 2000, 50); t1 = time.perf_counter()
    ts.append((t0, t1, 1e3 * r.log.device_seconds))
gaps = [1e3 * (ts[k + 1][0] - ts[k][1]) for k in range(len(ts) - 1)]
over = [1e3 * (t1 - t0) - d for (t0, t1, d) in ts]
print(f"150 calls: device ms min/median/max {min(d for *_, d in ts):.2f}/{np.median([d for *_, d in ts]):.2f}/{max(d for *_, d in ts):.2f}; "
      f"in-call overhead ms median/max {np.median(over):.3f}/{max(over):.3f}; between-call gap ms median/max {np.median(gaps):.3f}/{max(gaps):.3f}")
print("calls with > 2 ms outside the device time:", [(k, round(o, 2)) for k, o in enumerate(over) if o > 2.0])
print("device-time outliers (> median + 3 ms):", [(k, round(d, 2)) for k, (*_, d) in enumerate(ts) if d > np.median([x for *_, x in ts]) + 3.0])
