"""Dense-inverse vs envelope preconditioner on BASELINE config 2 (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08734_b200 import api, inputs
P = api.Problem("sphere", h=0.05, p=3, c=1.0)
P.decompose(inputs.rcb_partition(P.active_cp, 64), 2, "oras", 4.0, 40.0)
A = api.DeviceHelmholtz.from_problem(P)
b = torch.from_numpy(inputs.rhs_sphere(P.active_cp)).cuda()
for v in ("0", "1"):
    os.environ["CPDDG_DENSE"] = v
    t0 = time.time(); M = api.SchwarzPreconditioner.from_problem(P); torch.cuda.synchronize(); t1 = time.time()
    x = torch.rand(P.n_active, dtype=torch.float64, device="cuda")
    for _ in range(3): M.apply(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): M.apply(x)
    e1.record(); torch.cuda.synchronize()
    rs = [api.gmres_solve(A, b, M, 1e-10, 2000, 50) for _ in range(3)]
    print(f"dense={v}: build {t1 - t0:.2f} s, apply {e0.elapsed_time(e1) / 20:.3f} ms, solve {min(r.log.device_seconds for r in rs) * 1e3:.2f} ms, its {rs[0].log.iterations}, bytes {M.stats()['factor_bytes'] / 1e9:.2f} GB", flush=True)
