"""Headline preconditioner + operator applies, for ncu captures (few launches)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08734_b200 import api, inputs
h = float(os.environ.get("CPDDG_H", "0.0125")); ns = int(os.environ.get("CPDDG_NS", "256")); no = int(os.environ.get("CPDDG_NO", "3"))
P = api.Problem("sphere", h=h, p=3, c=1.0)
P.decompose(inputs.rcb_partition(P.active_cp, ns), no, "oras", 4.0, 40.0)
A = api.DeviceHelmholtz.from_problem(P)
M = api.SchwarzPreconditioner.from_problem(P)
x = torch.from_numpy(inputs.uniform_vector(P.n_active, 1)).cuda()
for _ in range(3):
    z = M.apply(x)
    y = A.apply(x)
torch.cuda.synchronize()
print("profile_kernels ok", P.n_active, M.stats()["algorithmic_bytes"], A.bytes())
