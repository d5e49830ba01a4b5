"""Windowed bulk-copy solve vs register-staged solve: agreement and timing (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import torch
from paper_1909_08734_b200 import api, inputs, _lib
h = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0125
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 256
P = api.Problem("sphere", h=h, p=3, c=1.0)
P.decompose(inputs.rcb_partition(P.active_cp, ns), 3, "oras", 4.0, 40.0)
Ms = {}
for v in ("0", "1"):
    os.environ["CPDDG_SOLVE_WINDOW"] = v
    Ms[v] = api.SchwarzPreconditioner.from_problem(P)
x = torch.from_numpy(inputs.uniform_vector(P.n_active, 1)).cuda()
z0, z1 = Ms["0"].apply(x), Ms["1"].apply(x)
torch.cuda.synchronize()
print("max |dz| / |z|:", float((z0 - z1).abs().max() / z0.abs().max()), "bitwise:", bool(torch.equal(z0, z1)), flush=True)
L = _lib.lib(); L.cpddg_pc_apply_mode.argtypes = [C.c_void_p] * 3 + [C.c_int, C.c_void_p]
z = torch.empty_like(x)
for v, M in Ms.items():
    for mode in (0, 1, 2):
        f = lambda: L.cpddg_pc_apply_mode(M.handle, C.c_void_p(x.data_ptr()), C.c_void_p(z.data_ptr()), mode, None)
        for _ in range(3): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): f()
        e1.record(); torch.cuda.synchronize()
        print(f"win={v} mode {mode}: {e0.elapsed_time(e1) / 20:.3f} ms", flush=True)
