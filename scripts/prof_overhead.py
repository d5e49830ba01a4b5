"""Cost of per-kernel CUDA-event profiling (gmres_solve(profile=True)) on a
BASELINE config: device time per solve with and without it, interleaved.

    python scripts/prof_overhead.py [headline|circle|...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_1909_08734_b200 import api

cfg = sys.argv[1] if len(sys.argv) > 1 else "headline"
w = bench.CONFIGS[cfg]
P, part, b_host, obj = bench.build_problem(w)
P.decompose(part, w["n_overlap"], w["method"], w["alpha"], w["alpha_cross"])
A = api.DeviceHelmholtz.from_problem(P)
M = api.SchwarzPreconditioner.from_problem(P)
b = torch.from_numpy(b_host).cuda()
for _ in range(3):
    api.gmres_solve(A, b, M, w["rel_tol"], w["max_iter"], w["gmres_restart"])
res = {False: [], True: []}
for _ in range(5):
    for prof in (False, True):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = api.gmres_solve(A, b, M, w["rel_tol"], w["max_iter"], w["gmres_restart"], profile=prof)
        e1.record()
        torch.cuda.synchronize()
        res[prof].append(e0.elapsed_time(e1))
for prof, v in res.items():
    print(f"[{cfg}] profile={prof}: ms per solve median {np.median(v):.2f} min {min(v):.2f}  its {r.log.iterations}")
