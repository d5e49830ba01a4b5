"""Per-CTA start/end of one preconditioner apply (development aid; run with
CPDDG_SOLVE_DEBUG=32): timeline of resident CTAs, per-SM load."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1909_08734_b200 import api, inputs, _lib
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
P = api.Problem("sphere", h=0.0125, p=3, c=1.0)
P.decompose(inputs.rcb_partition(P.active_cp, 256), 3, "oras", 4.0, 40.0)
M = api.SchwarzPreconditioner.from_problem(P)
L = _lib.lib(); L.cpddg_pc_apply_mode.argtypes = [C.c_void_p] * 3 + [C.c_int, C.c_void_p]
x = torch.from_numpy(inputs.uniform_vector(P.n_active, 1)).cuda(); z = torch.empty_like(x)
for _ in range(3):
    L.cpddg_pc_apply_mode(M.handle, C.c_void_p(x.data_ptr()), C.c_void_p(z.data_ptr()), mode, None)
torch.cuda.synchronize()
t = np.zeros((1024, 20), np.int64)
L.cpddg_dev_trace(t.ctypes.data_as(C.c_void_p))
n = P.n_sub
t = t[:n]
t0 = t[:, 0].min()
st = (t[:, 0] - t0) / 1e3; en = (t[:, 1] - t0) / 1e3; dur = en - st
sizes = np.array([P.local(int(j))["n"] if isinstance(P.local(int(j)), dict) else 0 for j in t[:, 3]]) if False else None
print(f"kernel span {en.max():.1f} us; CTA duration min {dur.min():.1f} p50 {np.median(dur):.1f} max {dur.max():.1f}; start max {st.max():.1f}")
for q in (10, 25, 50, 75, 90, 100):
    print(f"  {q}% of CTAs done by {np.percentile(en, q):.1f} us")
sm = t[:, 2]
per_sm = np.bincount(sm, minlength=148)
print("CTAs per SM histogram:", np.bincount(per_sm))
grid = np.linspace(0, en.max(), 12)
print("active CTAs over time:", [int(((st <= g) & (en > g)).sum()) for g in grid])
order = np.argsort(-dur)[:8]
print("longest CTAs (block, sub, sm, dur us):", [(int(i), int(t[i, 3]), int(sm[i]), round(float(dur[i]), 1)) for i in order])
