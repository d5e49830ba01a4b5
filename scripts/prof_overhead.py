"""Host wall time vs device time per small solve (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1909_08734_b200 import api, inputs
P = api.Problem("circle", h=0.0125, p=3, c=1.0)
cp = P.active_cp
P.decompose(inputs.sector_partition(cp, 8), 2, "oras", 1.0, -1.0)
A = api.DeviceHelmholtz.from_problem(P); M = api.SchwarzPreconditioner.from_problem(P)
b = torch.from_numpy(inputs.rhs_circle(cp)).cuda()
for _ in range(3): api.gmres_solve(A, b, M, 1e-10, 2000, 50)
for prof in (False, True):
    walls, devs = [], []
    for _ in range(30):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = api.gmres_solve(A, b, M, 1e-10, 2000, 50, profile=prof)
        t1 = time.perf_counter()
        walls.append(t1 - t0); devs.append(r.log.device_seconds)
    walls, devs = np.array(walls) * 1e3, np.array(devs) * 1e3
    print(f"profile={prof} wall ms: median {np.median(walls):.2f} min {walls.min():.2f} max {walls.max():.2f}; device ms: median {np.median(devs):.2f} min {devs.min():.2f} max {devs.max():.2f}")
import subprocess
print(subprocess.run("nproc; cat /proc/loadavg; cat /sys/devices/system/cpu/cpu0/cpufreq/scaling_governor 2>/dev/null", shell=True, capture_output=True, text=True).stdout)
