"""Small streamed-path workload for compute-sanitizer (development aid):
sphere h = 0.1 in 200 RCB parts (TMA-streamed record solve), the register
fallback, an operator apply and a short GMRES solve."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08734_b200 import api, inputs
P = api.Problem("sphere", h=0.1, p=3, c=1.0)
P.decompose(inputs.rcb_partition(P.active_cp, 200), 2, "oras", 4.0, 40.0)
A = api.DeviceHelmholtz.from_problem(P)
M = api.SchwarzPreconditioner.from_problem(P)
x = torch.from_numpy(inputs.uniform_vector(P.n_active, 3)).cuda()
z = M.apply(x); y = A.apply(x)
b = torch.from_numpy(inputs.rhs_sphere(P.active_cp)).cuda()
r = api.gmres_solve(A, b, M, 1e-10, 200, 50)
os.environ["CPDDG_TMA_RING_LIMIT"] = "1024"
Mf = api.SchwarzPreconditioner.from_problem(P)
zf = Mf.apply(x)
torch.cuda.synchronize()
print("ok", M.stats()["apply_mode"], Mf.stats()["apply_mode"], r.log.iterations, float((z - zf).abs().max()))
