"""Register-resident vs streamed MGS: identical GMRES history and timing (development aid)."""
import os, subprocess, sys, json
code = r'''
import os, sys, json
sys.path.insert(0, "/root/repo")
import torch
from paper_1909_08734_b200 import api, inputs
P = api.Problem("sphere", h=float(sys.argv[1]), p=3, c=1.0)
P.decompose(inputs.rcb_partition(P.active_cp, int(sys.argv[2])), 3, "oras", 4.0, 40.0)
A = api.DeviceHelmholtz.from_problem(P); M = api.SchwarzPreconditioner.from_problem(P)
b = torch.from_numpy(inputs.rhs_sphere(P.active_cp)).cuda()
r = api.gmres_solve(A, b, M, 1e-10, 2000, 50)
r = api.gmres_solve(A, b, M, 1e-10, 2000, 50, profile=True)
print(json.dumps(dict(it=r.log.iterations, res=[float(v) for v in r.log.residuals[-3:]], t=r.log.device_seconds, kt=r.log.kernel_times)))
'''
for h, ns in ((0.05, 16), (0.0125, 256)):
    outs = {}
    for mode in ("reg", "stream"):
        env = dict(os.environ, CPDDG_MGS=mode)
        outs[mode] = json.loads(subprocess.run([sys.executable, "-c", code, str(h), str(ns)], env=env, capture_output=True, text=True, check=True).stdout.strip().splitlines()[-1])
    print(h, "identical history:", outs["reg"]["res"] == outs["stream"]["res"] and outs["reg"]["it"] == outs["stream"]["it"])
    for k, v in outs.items(): print("  ", k, v)
