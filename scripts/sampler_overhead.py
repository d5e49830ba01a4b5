"""Cost of sampling clocks during the timed region: headline solves with no
sampler, with `nvidia-smi -lms` (bench.py's ClockSampler) and with an
in-process NVML thread (development aid)."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_1909_08734_b200 import api

w = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "headline"]
P, part, b_host, obj = bench.build_problem(w)
P.decompose(part, w["n_overlap"], w["method"], w["alpha"], w["alpha_cross"])
A = api.DeviceHelmholtz.from_problem(P)
M = api.SchwarzPreconditioner.from_problem(P)
b = torch.from_numpy(b_host).cuda()
for _ in range(3):
    api.gmres_solve(A, b, M, w["rel_tol"], w["max_iter"], w["gmres_restart"])


def run(k=5):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        api.gmres_solve(A, b, M, w["rel_tol"], w["max_iter"], w["gmres_restart"])
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


class Nvml:
    def __init__(self, ms):
        import pynvml as N
        self.N, self.ms, self.stop_ = N, ms, False
        N.nvmlInit()
        self.hdl = N.nvmlDeviceGetHandleByIndex(0)
        self.samples = []

    def loop(self):
        N = self.N
        while not self.stop_:
            self.samples.append((N.nvmlDeviceGetClockInfo(self.hdl, N.NVML_CLOCK_SM),
                                 N.nvmlDeviceGetCurrentClocksEventReasons(self.hdl)))
            time.sleep(self.ms / 1000)

    def __enter__(self):
        self.th = threading.Thread(target=self.loop, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop_ = True
        self.th.join()


for rep in range(2):
    print("none", round(run(), 2))
    cs = bench.ClockSampler(0, 200)
    cs.start()
    t = run()
    print("nvidia-smi 200ms", round(t, 2), cs.stop())
    for ms in (100, 20):
        with Nvml(ms) as nv:
            t = run()
        print(f"nvml {ms}ms", round(t, 2), len(nv.samples), nv.samples[:2])
