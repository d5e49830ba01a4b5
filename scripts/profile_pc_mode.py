"""Run the preconditioner in one mode (0 both, 1 forward, 2 backward) a few times (ncu target)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_08734_b200 import api, inputs, _lib
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
P = api.Problem("sphere", h=0.0125, p=3, c=1.0)
P.decompose(inputs.rcb_partition(P.active_cp, 256), 3, "oras", 4.0, 40.0)
M = api.SchwarzPreconditioner.from_problem(P)
L = _lib.lib(); L.cpddg_pc_apply_mode.argtypes = [C.c_void_p] * 3 + [C.c_int, C.c_void_p]
x = torch.from_numpy(inputs.uniform_vector(P.n_active, 1)).cuda(); z = torch.empty_like(x)
for _ in range(3):
    L.cpddg_pc_apply_mode(M.handle, C.c_void_p(x.data_ptr()), C.c_void_p(z.data_ptr()), mode, C.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize(); print("ok mode", mode)
