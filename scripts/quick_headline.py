"""Quick device timing of one configuration (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1909_08734_b200 import api, inputs
h = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0125
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 256
no = int(sys.argv[3]) if len(sys.argv) > 3 else 3
meth = sys.argv[4] if len(sys.argv) > 4 else "oras"
t0 = time.time(); P = api.Problem("sphere", h=h, p=3, c=1.0); t1 = time.time()
part = inputs.rcb_partition(P.active_cp, ns)
P.decompose(part, no, meth, 4.0, 40.0); t2 = time.time()
A = api.DeviceHelmholtz.from_problem(P); M = api.SchwarzPreconditioner.from_problem(P); torch.cuda.synchronize(); t3 = time.time()
st = M.stats()
print(f"N_A={P.n_active} setup {t1-t0:.1f}s decomp {t2-t1:.1f}s op+pc {t3-t2:.1f}s  pc: {st}", flush=True)
b = torch.from_numpy(inputs.rhs_sphere(P.active_cp)).cuda()
x = torch.rand(P.n_active, dtype=torch.float64, device="cuda")
import ctypes as C
from paper_1909_08734_b200 import _lib
L = _lib.lib(); L.cpddg_pc_apply_mode.argtypes = [C.c_void_p]*3 + [C.c_int, C.c_void_p]
z = torch.empty_like(x)
def mode(m):
    return lambda: L.cpddg_pc_apply_mode(M.handle, C.c_void_p(x.data_ptr()), C.c_void_p(z.data_ptr()), m, C.c_void_p(torch.cuda.current_stream().cuda_stream))
for name, f in [("op", lambda: A.apply(x)), ("pc", lambda: M.apply(x)), ("pc_fwd", mode(1)), ("pc_bwd", mode(2))]:
    for _ in range(3): f()
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): f()
    e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / 20
    print(f"{name}: {ms:.3f} ms", flush=True)
a_alg, a_str = A.bytes()
print(f"op alg bytes {a_alg/1e6:.1f} MB streamed {a_str/1e6:.1f} MB; pc bytes {st['factor_bytes']/1e9:.2f} GB")
for prof in (False, True, False, True):
    r2 = api.gmres_solve(A, b, M, 1e-10, 2000, 50, profile=prof)
    print(f"  gmres profile={prof}: t {r2.log.device_seconds:.3f}s kt={r2.log.kernel_times}")
res = api.gmres_solve(A, b, M, 1e-10, 2000, 50)
print(f"gmres: iters {res.log.iterations} conv {res.log.converged} t {res.log.device_seconds:.3f}s launches {res.log.kernel_launches} final rel {res.log.final_true_residual/float(b.norm()):.3e}")
print(f"DOF.iters/s = {P.n_active*res.log.iterations/res.log.device_seconds:.3e}")
