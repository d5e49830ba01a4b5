"""Exact zeros in the streamed factor arrays (development aid): how much of the
envelope storage the no-pivot LU never fills."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1909_08734_b200 import api, inputs, _lib
P = api.Problem("sphere", h=0.0125, p=3, c=1.0, device_setup=True)
P.decompose(inputs.rcb_partition(P.active_cp, 256), 3, "oras", 4.0, 40.0)
M = api.SchwarzPreconditioner.from_problem(P)
o = np.zeros(6, np.int64)
_lib.check(_lib.lib().cpddg_pc_debug_zero_stats(M.handle, o))
print(f"L: {o[0]} entries, {o[1] / o[0]:.3f} zero, {16 * o[2] / o[0]:.3f} in all-zero 16-segments")
print(f"U: {o[3]} entries, {o[4] / o[3]:.3f} zero, {16 * o[5] / o[3]:.3f} in all-zero 16-segments")
print("stats", M.stats())
