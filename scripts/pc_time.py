"""Time one preconditioner mode at the headline (development aid; reads
CPDDG_SOLVE_* experiment knobs from the environment)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08734_b200 import api, inputs, _lib
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
h = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0125
ns = int(sys.argv[3]) if len(sys.argv) > 3 else 256
P = api.Problem("sphere", h=h, p=3, c=1.0)
P.decompose(inputs.rcb_partition(P.active_cp, ns), 3, "oras", 4.0, 40.0)
M = api.SchwarzPreconditioner.from_problem(P)
L = _lib.lib(); L.cpddg_pc_apply_mode.argtypes = [C.c_void_p] * 3 + [C.c_int, C.c_void_p]
x = torch.from_numpy(inputs.uniform_vector(P.n_active, 1)).cuda(); z = torch.empty_like(x)
f = lambda: L.cpddg_pc_apply_mode(M.handle, C.c_void_p(x.data_ptr()), C.c_void_p(z.data_ptr()), mode,
                                  C.c_void_p(torch.cuda.current_stream().cuda_stream))
for _ in range(3): f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(30): f()
e1.record(); torch.cuda.synchronize()
env = {k: v for k, v in os.environ.items() if k.startswith("CPDDG_")}
print(f"mode {mode} {env}: {e0.elapsed_time(e1) / 30:.3f} ms", flush=True)
