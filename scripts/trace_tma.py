"""Per-block trace of the TMA forward solve of CTA 0 (development aid; CPDDG_SOLVE_DEBUG=16)."""
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
    L.cpddg_pc_apply_mode(M.handle, C.c_void_p(x.data_ptr()), C.c_void_p(z.data_ptr()), 1, None)
torch.cuda.synchronize()
t = np.zeros((1024, 20), np.int64)
L.cpddg_dev_trace(t.ctypes.data_as(C.c_void_p))
nb = int(np.argmax(t[:, 0] == 0)) or 1024
t = t[:nb]
step = np.diff(t[:, 0])
w0 = t[:-1, 1] - t[:-1, 0]
ready = t[1:-1, 3:16] - t[1:-1, 0:1]
done = t[1:-1, 17] - t[1:-1, 0]
print(f"blocks {nb}: step cycles mean {step.mean():.0f} p50 {np.median(step):.0f} p90 {np.percentile(step, 90):.0f}")
print(f"warp0 {np.median(w0):.0f}; panel data ready (median over warps) {np.median(ready):.0f}, max-warp {np.median(ready.max(1)):.0f}; last panel warp done {np.median(done):.0f}")
print("warp0 pre-update", np.median(t[:-1, 18] - t[:-1, 0]), "substitution", np.median(t[:-1, 1] - t[:-1, 18]))
