"""Pipelined (speculative) Arnoldi steps vs the synchronous loop (profile=True
disables the pipelining): identical histories, and wall time per solve."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1909_08734_b200 import api, inputs
for surf, h, ns in (("circle", 0.0125, 8), ("sphere", 0.05, 16), ("sphere", 0.0125, 256)):
    P = api.Problem(surf, h=h, p=3, c=1.0)
    cp = P.active_cp
    part = inputs.sector_partition(cp, ns) if surf == "circle" else inputs.rcb_partition(cp, ns)
    P.decompose(part, 3 if surf == "sphere" else 2, "oras", 4.0, 40.0)
    A = api.DeviceHelmholtz.from_problem(P); M = api.SchwarzPreconditioner.from_problem(P)
    b = torch.from_numpy(inputs.rhs_sphere(cp) if surf == "sphere" else inputs.rhs_circle(cp)).cuda()
    os.environ["CPDDG_GMRES_SYNC"] = "1"; ref = api.gmres_solve(A, b, M, 1e-10, 2000, 50); del os.environ["CPDDG_GMRES_SYNC"]
    ts = []
    for _ in range(5):
        r = api.gmres_solve(A, b, M, 1e-10, 2000, 50)
        ts.append(r.log.device_seconds)
    same = r.log.iterations == ref.log.iterations and np.array_equal(np.asarray(r.log.residuals), np.asarray(ref.log.residuals))
    print(f"{surf} h={h} N={P.n_active}: its {r.log.iterations} identical={same} pipelined {min(ts)*1e3:.2f} ms (median {np.median(ts)*1e3:.2f})  sync/profiled {ref.log.device_seconds*1e3:.2f} ms", flush=True)
