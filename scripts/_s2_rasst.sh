mkdir -p gpurun_out/s2
timeout 900 python -c "
import sys, time; sys.path.insert(0,'.')
import numpy as np, torch
from paper_1909_08734_b200 import api, inputs
P = api.Problem('torus', h=0.01, p=3, c=1.0, major_radius=1.0, minor_radius=0.4)
cp = P.active_cp
P.decompose(inputs.rcb_partition(cp, 512), 2, 'ras')
A = api.DeviceHelmholtz.from_problem(P); M = api.SchwarzPreconditioner.from_problem(P)
b = torch.from_numpy(inputs.rhs_trig(cp, seed=2024)).cuda()
for _ in range(2):
    r = api.stationary_solve(A, b, M, 1e-10, 5000)
    print('RAS stationary torus: iters', r.log.iterations, 'converged', r.log.converged, 'device s', round(r.log.device_seconds, 3), 'final rel', r.log.final_true_residual / float(b.norm()), 'apply_mode', M.stats()['apply_mode'])
" > gpurun_out/s2/rasst.log 2>&1
