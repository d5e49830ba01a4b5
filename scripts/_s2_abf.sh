mkdir -p gpurun_out/s2
o=gpurun_out/s2/abf.log; : > $o
for v in head new; do cp scripts/ablib/libcpddg_$v.so paper_1909_08734_b200/lib/libcpddg.so; echo "== $v" >> $o; timeout 120 python -c "
import sys; sys.path.insert(0,'.')
from paper_1909_08734_b200 import api, inputs
P = api.Problem('sphere', h=0.0125, p=3, c=1.0)
P.decompose(inputs.rcb_partition(P.active_cp, 256), 3, 'oras', 4.0, 40.0)
for _ in range(2):
    M = api.SchwarzPreconditioner.from_problem(P); st = M.stats(); print('factor_seconds', st['factor_seconds'], 'probe', st['max_probe_residual'])
" >> $o 2>&1; done
cp scripts/ablib/libcpddg_new.so paper_1909_08734_b200/lib/libcpddg.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s2/parity_abf.log 2>&1
