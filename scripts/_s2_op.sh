mkdir -p gpurun_out/s2
o=gpurun_out/s2/op.log; : > $o
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "operator or staged" > gpurun_out/s2/parity_op.log 2>&1
for e in 1 0 1 0; do CPDDG_EXT_PIPE=$e timeout 300 python -c "
import sys, os; sys.path.insert(0,'.')
import torch
from paper_1909_08734_b200 import api, inputs
P = api.Problem('sphere', h=0.0125, p=3, c=1.0)
A = api.DeviceHelmholtz.from_problem(P)
x = torch.rand(P.n_active, dtype=torch.float64, device='cuda')
for _ in range(5): A.apply(x)
torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200): A.apply(x)
e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / 200
alg, strm = A.bytes()
print(f'pipe={os.environ[\"CPDDG_EXT_PIPE\"]}: op {ms*1e3:.1f} us, B_op {alg/1e6:.1f} MB -> {alg/ms/1e6:.0f} GB/s')
" >> $o 2>&1; done
