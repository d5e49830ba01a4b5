"""Per-block timing trace of the column backward of CTA 0 (development aid;
run with CPDDG_BWD_LAYOUT=cols CPDDG_BWD_PREFETCH=16+pf)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1909_08734_b200 import api, inputs, _lib
P = api.Problem("sphere", h=0.0125, p=3, c=1.0)
P.decompose(inputs.rcb_partition(P.active_cp, 256), 3, "oras", 4.0, 40.0)
M = api.SchwarzPreconditioner.from_problem(P)
L = _lib.lib(); L.cpddg_pc_apply_mode.argtypes = [C.c_void_p] * 3 + [C.c_int, C.c_void_p]
x = torch.from_numpy(inputs.uniform_vector(P.n_active, 1)).cuda(); z = torch.empty_like(x)
for _ in range(3):
    L.cpddg_pc_apply_mode(M.handle, C.c_void_p(x.data_ptr()), C.c_void_p(z.data_ptr()), 2, None)
torch.cuda.synchronize()
t = np.zeros((1024, 20), np.int64)
L.cpddg_dev_trace(t.ctypes.data_as(C.c_void_p))
nb = int(np.argmax(t[:, 0] == 0)) or 1024
t = t[:nb]
step = np.diff(t[:, 0])
w0 = t[:-1, 1] - t[:-1, 0]
items = t[1:-1, 2:17] - t[1:-1, 0:1]
fin = t[1:-1, 18] - t[1:-1, 17]
bar = t[1:-1, 17] - t[1:-1, 0]
print(f"blocks {nb}: step cycles mean {step.mean():.0f} p50 {np.median(step):.0f}")
print(f"warp0 {w0.mean():.0f}; items done per warp mean {items.mean():.0f} max {items.max(1).mean():.0f}; panel barrier passed {bar.mean():.0f}; finalize+stash+tables {fin.mean():.0f}")
os.environ["CPDDG_BWD_LAYOUT"] = "rows"
Mr = api.SchwarzPreconditioner.from_problem(P)
zr = Mr.apply(x)
L.cpddg_pc_apply_mode(M.handle, C.c_void_p(x.data_ptr()), C.c_void_p(z.data_ptr()), 0, None)
print("check vs rows layout (full apply):", float((zr - z).norm() / zr.norm()))
print("plo0/pend samples:", [(int(v) >> 32, int(v) & 0xffffffff) for v in t[1:8, 19]], "cols 2..18 of row 5:", t[5, 2:19] - t[5, 0])
