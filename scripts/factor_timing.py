"""Device factorisation time, k_factor (CPDDG_FACTOR=v1) vs k_factor2 (default),
each built three times in one process (the first includes module loading and
clock ramp-up), plus bitwise equality of M x (development aid).
Usage: factor_timing.py [h] [n_subdomains]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08734_b200 import api, inputs

h = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0125
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 256
P = api.Problem("sphere", h=h, p=3, c=1.0, device_setup=True)
P.decompose(inputs.rcb_partition(P.active_cp, ns), 3, "oras", 4.0, 40.0)
x = torch.from_numpy(inputs.uniform_vector(P.n_active, 3)).cuda()
z = {}
for v in ("v2", "v1", "v2", "v1"):
    os.environ["CPDDG_FACTOR"] = v
    for rep in range(2):
        M = api.SchwarzPreconditioner.from_problem(P)
        st = M.stats()
        z[v] = M.apply(x)
        print(v, rep, f"factor {st['factor_seconds']:.4f} s  probe {st['max_probe_residual']:.3g}", flush=True)
        del M
print("bitwise equal M x:", bool(torch.equal(z["v1"], z["v2"])))
