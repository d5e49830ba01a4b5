mkdir -p gpurun_out/s2
o=gpurun_out/s2/mgsb.log; : > $o
for b in 4 2 1 3; do CPDDG_MGS_BPS=$b timeout 300 python -c "
import sys, os; sys.path.insert(0,'.')
import torch
from paper_1909_08734_b200 import api, inputs
P = api.Problem('sphere', h=0.0125, p=3, c=1.0)
P.decompose(inputs.rcb_partition(P.active_cp, 256), 3, 'oras', 4.0, 40.0)
A = api.DeviceHelmholtz.from_problem(P); M = api.SchwarzPreconditioner.from_problem(P)
b = torch.from_numpy(inputs.rhs_sphere(P.active_cp)).cuda()
ts = []
for _ in range(4):
    r = api.gmres_solve(A, b, M, 1e-10, 2000, 50); ts.append(r.log.device_seconds)
rp = api.gmres_solve(A, b, M, 1e-10, 2000, 50, profile=True)
kt = rp.log.kernel_times
print(f'bps={os.environ[\"CPDDG_MGS_BPS\"]}: its {r.log.iterations} solve min {min(ts)*1e3:.1f} ms; pc {kt[\"pc_seconds\"]*1e3:.1f} op {kt[\"op_seconds\"]*1e3:.1f}; rest {min(ts)*1e3 - kt[\"pc_seconds\"]*1e3 - kt[\"op_seconds\"]*1e3:.1f} ms; res {r.log.residuals[-1]:.6e}')
" >> $o 2>&1; done
