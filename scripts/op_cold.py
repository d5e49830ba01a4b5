"""Operator apply timing in the three cache states that matter (development aid):
warm back to back (CUDA graph of 100 applies), cold (L2 flushed by a 512 MB
write before each apply), and in-solve (right after a preconditioner apply,
which streams ~10 GB through L2), plus the per-launch figure of a profiled
GMRES solve.  Variants are operator handles created under different
environment switches; their outputs must be bit-identical.
Usage: op_cold.py [config] [VAR=val[,VAR=val]] ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1909_08734_b200 import api

cfg = sys.argv[1] if len(sys.argv) > 1 else "headline"
variants = sys.argv[2:] or ["CPDDG_OP_PREFETCH=0", "CPDDG_OP_PREFETCH=1"]
w = bench.CONFIGS[cfg]
P, part, b_host, _ = bench.build_problem(w)
P.decompose(part, w["n_overlap"], w["method"], w["alpha"], w["alpha_cross"])
M = api.SchwarzPreconditioner.from_problem(P)
ops = {}
for var in variants:
    env = dict(kv.split("=", 1) for kv in var.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    ops[var] = api.DeviceHelmholtz.from_problem(P)
    for k, v in old.items():
        if v is None:
            del os.environ[k]
        else:
            os.environ[k] = v
n = P.n_active
x = torch.rand(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
b = torch.from_numpy(b_host).cuda()
ys = {k: A.apply(x) for k, A in ops.items()}
first = next(iter(ys))
for k in ys:
    print(f"{k}: bit-identical to {first}: {bool(torch.equal(ys[k], ys[first]))}", flush=True)
flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
z = torch.empty_like(x)
for name, A in ops.items():
    alg, streamed = A.bytes()
    y = torch.empty_like(x)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            A.apply(x, out=y)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(100):
            A.apply(x, out=y)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    warm = e0.elapsed_time(e1) / 500
    cold, insolve = 0.0, 0.0
    R = 30
    for r in range(R):
        flush.fill_(float(r))
        e0.record()
        A.apply(x, out=y)
        e1.record()
        torch.cuda.synchronize()
        cold += e0.elapsed_time(e1) / R
        M.apply(x, out=z)
        e0.record()
        A.apply(z, out=y)
        e1.record()
        torch.cuda.synchronize()
        insolve += e0.elapsed_time(e1) / R
    res = api.gmres_solve(A, b, M, w["rel_tol"], w["max_iter"], w["gmres_restart"], profile=True)
    kt = res.log.kernel_times
    prof = kt["op_seconds"] / max(kt["op_launches"], 1) * 1e3
    # device-driven cycles with device timestamps around the operator (the
    # interval also holds one 1-thread stamp launch)
    os.environ["CPDDG_GMRES_GRAPH"] = "1"
    res = api.gmres_solve(A, b, M, w["rel_tol"], w["max_iter"], w["gmres_restart"], profile=True)
    del os.environ["CPDDG_GMRES_GRAPH"]
    kt = res.log.kernel_times
    ingraph = kt["op_seconds"] / max(kt["op_launches"], 1) * 1e3
    print(f"{name}: alg {alg / 1e6:.1f} MB streamed {streamed / 1e6:.1f} MB | warm {warm * 1e3:.1f} us "
          f"({alg / warm / 1e6:.0f} GB/s) | cold {cold * 1e3:.1f} us ({alg / cold / 1e6:.0f} GB/s) | "
          f"after pc {insolve * 1e3:.1f} us ({alg / insolve / 1e6:.0f} GB/s) | in gmres {prof * 1e3:.1f} us "
          f"({alg / prof / 1e6:.0f} GB/s) | in gmres graph {ingraph * 1e3:.1f} us ({alg / ingraph / 1e6:.0f} GB/s), "
          f"{res.log.iterations} it, {res.log.device_seconds * 1e3:.1f} ms",
          flush=True)
