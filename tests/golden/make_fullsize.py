"""Full-size reference results for BASELINE configs 4 (torus) and 5 (displaced
icosphere TriMesh) with oracle/_ref (the unmodified reference headers + shim):
the reference's own gmres_solve and DirectSolver on the local systems, which
are taken from this repository's setup (bit-identical to the reference's
assemble_local, tests/test_setup_parity.py; the reference's serial
build_subdomains would add hours at 512 subdomains).  Writes iteration counts,
residuals and a strided sample of the solution into fullsize_reference.json /
fullsize_<name>.npz.  CPU only; minutes per configuration.

    python tests/golden/make_fullsize.py torus|trimesh|torus_ras_stationary
"""
import json
import os
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np

import ref
from paper_1909_08734_b200 import api, inputs

STRIDE = 997
CONFIGS = {
    "torus": dict(surface="torus", major_radius=1.0, minor_radius=0.4, h=0.01, n_subdomains=512, n_overlap=2),
    "trimesh": dict(surface="obj", h=0.01, n_subdomains=512, n_overlap=2, subdivisions=6, mesh_seed=5),
    # BASELINE config 4's other run: RAS as a stationary solver
    "torus_ras_stationary": dict(surface="torus", major_radius=1.0, minor_radius=0.4, h=0.01, n_subdomains=512,
                                 n_overlap=2, method="ras", mode="stationary"),
}


def main(name):
    w = CONFIGS[name]
    obj = None
    if w["surface"] == "obj":
        v, f = inputs.displaced_icosphere(w["subdivisions"], seed=w["mesh_seed"])
        obj = os.path.join(tempfile.mkdtemp(prefix="cpddg_mesh_"), "icosphere.obj")
        inputs.write_obj(obj, v, f)
    P = api.Problem(w["surface"], h=w["h"], p=3, c=1.0, obj_path=obj, major_radius=w.get("major_radius", 2 / 3),
                    minor_radius=w.get("minor_radius", 1 / 3))
    cp = P.active_cp
    part = inputs.rcb_partition(cp, w["n_subdomains"])
    method, mode = w.get("method", "oras"), w.get("mode", "gmres")
    _, moves = (P.decompose(part, w["n_overlap"], "ras") if method == "ras"
                else P.decompose(part, w["n_overlap"], "oras", 4.0, 40.0))
    b = inputs.rhs_trig(cp, seed=2024)
    cfg = dict(surface=w["surface"], h=w["h"], p=3, c=1.0, method=method, mode=mode, gmres_restart=50,
               n_overlap=w["n_overlap"], n_subdomains=w["n_subdomains"], rel_tol=1e-10,
               max_iter=2000 if mode == "gmres" else 5000)
    if method == "oras":
        cfg.update(alpha=4.0, alpha_cross=40.0)
    if w["surface"] == "torus":
        cfg.update(major_radius=w["major_radius"], minor_radius=w["minor_radius"])
    if obj:
        cfg.update(obj=obj)
    t0 = time.time()
    R = ref.RefProblem(cfg, workers=os.cpu_count())
    assert R.n_active == P.n_active
    ref.set_locals(R, [P.local(j) for j in range(P.n_sub)])
    t1 = time.time()
    out = R.solve(b)
    t2 = time.time()
    u = out["u"]
    key = f"{name.split('_')[0]}_h{w['h']}_rcb{w['n_subdomains']}_no{w['n_overlap']}_" + (
        "oras_a4_ax40" if method == "oras" else f"{method}_{mode}")
    rec = dict(n_active=P.n_active, n_ghost=P.n_ghost, align_moves=moves, iterations=out["iterations"],
               converged=out["converged"],
               final_rel_residual=out["final_true_residual"] / float(np.linalg.norm(b)),
               u_norm2=float(np.linalg.norm(u)), u_norm_inf=float(np.abs(u).max()), sample_stride=STRIDE,
               _how=f"tests/golden/make_fullsize.py {name}: oracle/_ref {mode} solve, {os.cpu_count()} threads, "
                    f"local factorisations {t1 - t0:.0f} s, solve {t2 - t1:.0f} s")
    path = os.path.join(HERE, "fullsize_reference.json")
    d = json.load(open(path))
    d[key] = rec
    json.dump(d, open(path, "w"), indent=2)
    np.savez_compressed(os.path.join(HERE, f"fullsize_{name}.npz"), u_sample=u[::STRIDE],
                        residuals=np.asarray(out["residuals"]))
    print(key, rec)


if __name__ == "__main__":
    main(sys.argv[1])
