"""Headline operator applies only (no preconditioner), for ncu launch lists and
captures of the operator kernels: 3 warm-up applies then 5 (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08734_b200 import api, inputs
P = api.Problem("sphere", h=0.0125, p=3, c=1.0)
A = api.DeviceHelmholtz.from_problem(P)
x = torch.from_numpy(inputs.uniform_vector(P.n_active, 1)).cuda()
y = torch.empty_like(x)
for _ in range(8):
    A.apply(x, out=y)
torch.cuda.synchronize()
print("op_prof ok", P.n_active, A.bytes())
