"""Sum over subdomains of nnz(L + U) of the oracle's local LU (SuperLU with
COLAMD ordering -- scipy.sparse.linalg.splu -- the algorithmic ancestor of the
reference's Eigen SparseLU<COLAMDOrdering>, direct.hpp:41-61) for a bench
configuration, against the device path's stored factor entries: the
denominator SURVEY.md 8(d) asks for (Sigma stored / Sigma nnz(L+U)).
Host-only (no GPU).  Usage: oracle_lu_fill.py [config] > profiles/r02_factor_format.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import splu

import bench
from paper_1909_08734_b200 import api, inputs

name = sys.argv[1] if len(sys.argv) > 1 else "headline"
w = bench.CONFIGS[name]
P = api.Problem(w["surface"], h=w["h"], p=w["p"], c=w["c"], tube_radius=w.get("tube_radius_h", 0.0) * w["h"])
cp = P.active_cp
part = inputs.rcb_partition(cp, w["n_subdomains"]) if w["partition"] == "rcb" else \
    inputs.sector_partition(cp, w["n_subdomains"])
P.decompose(part, w["n_overlap"], w["method"], w["alpha"], w["alpha_cross"])
t0 = time.perf_counter()
tot_lu = tot_a = tot_n = 0
per = []
for j in range(P.n_sub):
    L = P.local(j)
    n = L["n_overlap"] + L["n_bc"]
    A = sp.csr_matrix((L["val"], L["col"], L["ptr"]), shape=(n, n)).tocsc()
    f = splu(A, permc_spec="COLAMD", options=dict(SymmetricMode=False))
    nnz = int(f.L.nnz + f.U.nnz - n)  # unit diagonal of L counted once
    per.append(nnz)
    tot_lu += nnz
    tot_a += A.nnz
    tot_n += n
print(json.dumps({
    "config": bench.workload_name(w), "n_subdomains": P.n_sub, "local_rows_total": tot_n, "local_nnz_A": tot_a,
    "oracle_lu": "scipy SuperLU, COLAMD column ordering (SymmetricMode off)",
    "sum_nnz_LU": tot_lu, "mean_nnz_LU_per_subdomain": tot_lu / P.n_sub, "max_nnz_LU": max(per),
    "seconds": time.perf_counter() - t0}, indent=1))
