"""Development check of the preconditioner solve paths at a BASELINE config:
per-apply time (CUDA events, 20 applies after warm-up) and agreement with the
round-1 path (k_solve_tma), then one GMRES solve per path.

    CPDDG_VERBOSE=1 python scripts/win_check.py [headline|torus|...] [ENV=VAL,...]..."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_1909_08734_b200 import api

cfg = sys.argv[1] if len(sys.argv) > 1 else "headline"
variants = sys.argv[2:] or ["CPDDG_SOLVE=tma", ""]
w = bench.CONFIGS[cfg]
P, part, b_host, obj = bench.build_problem(w)
P.decompose(part, w["n_overlap"], w["method"], w["alpha"], w["alpha_cross"])
A = api.DeviceHelmholtz.from_problem(P)
x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, P.n_active)).cuda()
b = torch.from_numpy(b_host).cuda()
zs = {}
for v in variants:
    env = dict(kv.split("=", 1) for kv in v.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    t0 = time.perf_counter()
    M = api.SchwarzPreconditioner.from_problem(P)
    torch.cuda.synchronize()
    tb = time.perf_counter() - t0
    for k, val in old.items():
        if val is None:
            os.environ.pop(k)
        else:
            os.environ[k] = val
    st = M.stats()
    z = M.apply(x)
    for _ in range(3):
        M.apply(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        M.apply(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    zs[v] = z.cpu().numpy()
    r = api.gmres_solve(A, b, M, w["rel_tol"], w["max_iter"], w["gmres_restart"])
    r = api.gmres_solve(A, b, M, w["rel_tol"], w["max_iter"], w["gmres_restart"])
    d = np.linalg.norm(zs[v] - zs[variants[0]]) / np.linalg.norm(zs[variants[0]])
    print(f"[{cfg}] {v or 'default'}: mode {st['apply_mode']} build {tb:.2f}s apply {ms:.3f} ms "
          f"{st['algorithmic_bytes'] / ms / 1e6:.0f} GB/s  rel diff vs {variants[0]} {d:.2e}  "
          f"gmres its {r.log.iterations} solve {r.log.device_seconds * 1e3:.1f} ms", flush=True)
