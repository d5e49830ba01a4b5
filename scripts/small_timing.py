"""Timed-region behaviour of millisecond solves: profiled vs not, with and
without an nvidia-smi sampler running (development aid)."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08734_b200 import api, inputs
P = api.Problem("circle", h=0.0125, p=3, c=1.0)
cp = P.active_cp
P.decompose(inputs.sector_partition(cp, 8), 2, "oras", 1.0, -1.0)
A = api.DeviceHelmholtz.from_problem(P); M = api.SchwarzPreconditioner.from_problem(P)
b = torch.from_numpy(inputs.rhs_circle(cp)).cuda()
def run(prof, k=100):
    for _ in range(3): api.gmres_solve(A, b, M, 1e-10, 2000, 50, profile=prof)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): api.gmres_solve(A, b, M, 1e-10, 2000, 50, profile=prof)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k
import bench
for smi in (False, True):
    cs = bench.ClockSampler(0) if smi else None
    if cs: cs.start()
    time.sleep(0.5)
    print(f"bench ClockSampler={smi}: profiled {run(True):.3f} ms/solve, plain {run(False):.3f} ms/solve", flush=True)
    if cs: print(cs.stop())
