"""A/B of an environment knob read at preconditioner build (development aid):
python ab_env.py VAR valueA valueB  -- headline GMRES solves, interleaved."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1909_08734_b200 import api, inputs
var, va, vb = sys.argv[1:4]
P = api.Problem("sphere", h=0.0125, p=3, c=1.0)
P.decompose(inputs.rcb_partition(P.active_cp, 256), 3, "oras", 4.0, 40.0)
A = api.DeviceHelmholtz.from_problem(P)
Ms = {}
for v in (va, vb):
    os.environ[var] = v
    Ms[v] = api.SchwarzPreconditioner.from_problem(P)
b = torch.from_numpy(inputs.rhs_sphere(P.active_cp)).cuda()
ts = {va: [], vb: []}
for rep in range(4):
    for v in (va, vb):
        r = api.gmres_solve(A, b, Ms[v], 1e-10, 2000, 50)
        ts[v].append(r.log.device_seconds)
for v in (va, vb):
    print(f"{var}={v}: its {r.log.iterations} times ms {[round(t * 1e3, 2) for t in ts[v]]} min {min(ts[v]) * 1e3:.2f}")
