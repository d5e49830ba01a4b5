"""Per-block trace of the record forward solve of one CTA (development aid):
CPDDG_SOLVE_DEBUG = 16 | (cta << 16)."""
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
t = t[:nb - 1]
st = t[:, 0]
step = np.diff(st)
rel = lambda c: (t[:-1, c] - st[:-1])
print(f"{os.environ.get('CPDDG_SOLVE_DEBUG')}: blocks {nb}: step cycles mean {step.mean():.0f} p50 {np.median(step):.0f} p90 {np.percentile(step, 90):.0f}")
print(f"  warp0 done {rel(1).mean():.0f}; w1 row0(pre) {rel(2).mean():.0f}; w1 rows {rel(3).mean():.0f}; w1 issue_pre {rel(4).mean():.0f}; w1 reduce+wait {rel(5).mean():.0f}")
pw = np.stack([rel(6 + w) for w in range(1, 14)], 1)
print(f"  panel warps done mean {pw.mean():.0f} max-over-warps mean {pw.max(1).mean():.0f}")
