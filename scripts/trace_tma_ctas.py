"""Per-CTA start/end of one k_solve_tma apply (development aid; CPDDG_SOLVE_DEBUG=32)."""
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
    L.cpddg_pc_apply_mode(M.handle, C.c_void_p(x.data_ptr()), C.c_void_p(z.data_ptr()), 0, None)
torch.cuda.synchronize()
t = np.zeros((1024, 20), np.int64)
L.cpddg_dev_trace(t.ctypes.data_as(C.c_void_p))
t = t[:148]
st = (t[:, 0] - t[:, 0].min()) / 1e3; en = (t[:, 1] - t[:, 0].min()) / 1e3; dur = en - st
print(f"span {en.max():.0f} us; CTA durations min {dur.min():.0f} p10 {np.percentile(dur, 10):.0f} p50 {np.median(dur):.0f} p90 {np.percentile(dur, 90):.0f} max {dur.max():.0f}")
for k in (1, 2, 3):
    sel = t[:, 2] == k
    if sel.any(): print(f"  CTAs with {k} subdomains: {sel.sum()}, duration mean {dur[sel].mean():.0f} max {dur[sel].max():.0f}")
