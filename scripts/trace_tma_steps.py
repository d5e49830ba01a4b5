"""Per-step trace of one CTA of k_solve_tma (development aid):
CPDDG_SOLVE_DEBUG = 16 | (cta << 16) [| 1: stream only].  Cycles from step 0."""
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
    rc = L.cpddg_pc_apply_mode(M.handle, C.c_void_p(x.data_ptr()), C.c_void_p(z.data_ptr()), mode, None)
torch.cuda.synchronize()
t = np.zeros((1024, 20), np.int64)
rc2 = L.cpddg_dev_trace(t.ctypes.data_as(C.c_void_p))
print("rc apply", rc, "rc trace", rc2, M.stats())
print("nonzero per column:", (t != 0).sum(0)[:12])
n = 1024
while n > 0 and t[n - 1, 0] == 0: n -= 1
if n < 3: sys.exit(0)
t = t[:n]
st = t[:, 0]
step = np.diff(st)
print(f"{os.environ.get('CPDDG_SOLVE_DEBUG')} mode {mode}: steps {n}: step cycles mean {step.mean():.0f} p50 {np.median(step):.0f} p90 {np.percentile(step, 90):.0f}")
rel = lambda c: t[:, c] - st
print(f"  mean from step start: wait done {rel(1).mean():.0f}, warp0 done {rel(2).mean():.0f}, consumer w2 done {rel(3).mean():.0f}, barrier out {rel(4).mean():.0f}")
lead = t[:, 1] - t[:, 5]
print(f"  item landed-or-waited minus issued: mean {lead.mean():.0f} p10 {np.percentile(lead, 10):.0f} p90 {np.percentile(lead, 90):.0f}; issued before step start: mean {(st - t[:, 5]).mean():.0f}")
print(f"  producer: slot wait {(t[:, 7] - t[:, 6]).mean():.0f}, ring wait {(t[:, 8] - t[:, 7]).mean():.0f}, issue {(t[:, 5] - t[:, 8]).mean():.0f}; bytes mean {t[:, 9].mean():.0f}")
print(f"  warp 0: matvec start {rel(10).mean():.0f}, after T^-1 part {rel(11).mean():.0f}, done {rel(2).mean():.0f}")
seg = lambda a, b: (st[b] - st[a]) / max(1, b - a)
half = n // 2
print(f"  step cycles: first half {seg(0, half - 1):.0f}, second half {seg(half, n - 1):.0f}")
for q in range(0, n - 64, 64):
    print(f"    steps {q}-{q + 63}: {seg(q, q + 63):.0f} cycles/step, wait {np.mean(t[q:q + 64, 1] - st[q:q + 64]):.0f}, bytes {t[q:q + 64, 9].mean():.0f}")
for a in list(range(0, 4)) + list(range(300, 304)):
    if a < n: print("  ", a, [int(v - st[0]) for v in t[a, :9]], int(t[a, 9]))
