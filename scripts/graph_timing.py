"""GMRES wall time per solve: device-driven cycle graphs (default) vs the
host-driven Arnoldi loop (CPDDG_GMRES_GRAPH=0), BASELINE configs 1 and 2 and
the headline (development aid).  Usage: graph_timing.py [circle|sphere05|headline]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1909_08734_b200 import api

names = sys.argv[1:] or ["circle", "sphere05"]
for name in names:
    w = bench.CONFIGS[name]
    P, part, b_host, _ = bench.build_problem(w)
    P.decompose(part, w["n_overlap"], w["method"], w["alpha"], w["alpha_cross"])
    A = api.DeviceHelmholtz.from_problem(P)
    M = api.SchwarzPreconditioner.from_problem(P)
    b = torch.from_numpy(b_host).cuda()
    k = 100 if P.n_active < 100000 else 5

    def run(prof=False):
        for _ in range(3):
            r = api.gmres_solve(A, b, M, w["rel_tol"], w["max_iter"], w["gmres_restart"], profile=prof)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            r = api.gmres_solve(A, b, M, w["rel_tol"], w["max_iter"], w["gmres_restart"], profile=prof)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k, r

    tg, rg = run()
    os.environ["CPDDG_GMRES_GRAPH"] = "1"
    tgp, rgp = run(True)
    os.environ["CPDDG_GMRES_GRAPH"] = "0"
    th, rh = run()
    del os.environ["CPDDG_GMRES_GRAPH"]
    kt = rgp.log.kernel_times
    print(f"{name}: N_A {P.n_active} iterations {rg.log.iterations}/{rh.log.iterations}  graph {tg:.3f} ms/solve "
          f"(profiled {tgp:.3f}; pc {1e6 * kt['pc_seconds'] / max(kt['pc_launches'], 1):.1f} us/apply, "
          f"op {1e6 * kt['op_seconds'] / max(kt['op_launches'], 1):.1f} us/apply)  host loop {th:.3f} ms/solve  "
          f"same u: {bool(torch.equal(rg.u, rh.u))}", flush=True)
