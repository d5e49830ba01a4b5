"""Oracle results for the north-star scale point at the BASELINE tube radius
(SURVEY.md Appendix A.1/A.3): sphere h = 0.0125 with tube radius sqrt(17) h
(663,454 DOF), 256 RCB, N_O = 3, ORAS alpha = 4, alpha_cross = 40, GMRES(50)
to 1e-10 -- bench.py --config headline_r17.  The reference has no tube-radius
override (proj/include/cpdd/band.hpp:157), so oracle/_ref cannot build this
band; the oracle restatement (oracle/cpdd_oracle.py: SuperLU-COLAMD local
solves, the reference's MGS/Givens GMRES, CSR SpMV) runs on the band, A and
local systems of this repository's HOST setup, which is bit-exact with the
reference's algorithms (tests/test_setup_parity.py) for any radius.  Stores
the iteration count, residuals and a strided sample of u in
scale_points.json / scale_headline_r17.npz.  CPU only (~10 minutes, ~20 GB).

    python tests/golden/make_scale_points.py headline_r17
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import scipy.sparse as sp

import cpdd_oracle as O
from paper_1909_08734_b200 import api, inputs

STRIDE = 997
CONFIGS = {"headline_r17": dict(h=0.0125, tube=17 ** 0.5, n_subdomains=256, n_overlap=3)}


def main(name):
    w = CONFIGS[name]
    t0 = time.time()
    P = api.Problem("sphere", h=w["h"], p=3, c=1.0, tube_radius=w["tube"] * w["h"])
    cp = P.active_cp
    part = inputs.rcb_partition(cp, w["n_subdomains"])
    _, moves = P.decompose(part, w["n_overlap"], "oras", 4.0, 40.0)
    ptr, col, val = P.csr("A")
    A = sp.csr_matrix((val, col, ptr), shape=(P.n_active, P.n_active))
    M = O.Schwarz([P.local(j) for j in range(P.n_sub)])
    t1 = time.time()
    b = inputs.rhs_sphere(cp)
    out = O.gmres_solve(lambda v: A @ v, M, b, 1e-10, 2000, 50)
    t2 = time.time()
    u = out["u"]
    rec = dict(n_active=P.n_active, n_ghost=P.n_ghost, align_moves=moves, iterations=out["iterations"],
               converged=out["converged"], final_rel_residual=out["final_true_residual"] / float(np.linalg.norm(b)),
               u_norm2=float(np.linalg.norm(u)), u_norm_inf=float(np.abs(u).max()), sample_stride=STRIDE,
               _how=f"tests/golden/make_scale_points.py {name}: oracle restatement (SuperLU-COLAMD local solves) "
                    f"on the host setup; setup + factorisations {t1 - t0:.0f} s, solve {t2 - t1:.0f} s")
    path = os.path.join(HERE, "scale_points.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    d[name] = rec
    json.dump(d, open(path, "w"), indent=2)
    np.savez_compressed(os.path.join(HERE, f"scale_{name}.npz"), u_sample=u[::STRIDE],
                        residuals=np.asarray(out["residuals"]))
    print(name, rec)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "headline_r17")
