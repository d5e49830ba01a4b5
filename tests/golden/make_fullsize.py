"""Full-size reference results for BASELINE configs 4 (torus) and 5 (displaced
icosphere TriMesh) with oracle/_ref (the unmodified reference headers + shim):
the reference's own gmres_solve and DirectSolver on the local systems, which
are taken from this repository's setup (bit-identical to the reference's
assemble_local, tests/test_setup_parity.py; the reference's serial
build_subdomains would add hours at 512 subdomains).  Writes iteration counts,
residuals and a strided sample of the solution into fullsize_reference.json /
fullsize_<name>.npz.  CPU only; minutes per configuration.

    python tests/golden/make_fullsize.py torus|trimesh|torus_ras_stationary
    python tests/golden/make_fullsize.py headline [oras|ras|oras_std]

The `headline` mode (BASELINE config 3: sphere h=0.0125, 256 RCB, N_O=3) runs
the reference's OWN pipeline end to end -- build_problem, load_partition +
align_interfaces, build_subdomains, assemble_local and DirectSolver
(ref.RefProblem.decompose, proj/include/cpdd/pipeline.hpp:186-216), then
gmres_solve (solve.hpp:128-214) -- with no input from this repository's setup
code: the partition is inputs.rcb_partition on the reference band's own
closest points and the right-hand side inputs.rhs_sphere on them.  It stores
the aligned-label hash, A x and M x on uniform_vector(N_A, 11) (strided
samples plus the componentwise-scale row sums sum_j |A_ij x_j|), and the
solution (strided sample, norms), in fullsize_headline_<method>.npz and
fullsize_reference.json.
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


HEADLINE = {
    # BASELINE config 3 runs: ORAS with the modified cross-point condition, RAS,
    # and ORAS with the standard Robin condition (alpha_cross = alpha)
    "oras": dict(method="oras", alpha=4.0, alpha_cross=40.0, max_iter=2000),
    "ras": dict(method="ras", max_iter=2000),
    "oras_std": dict(method="oras", alpha=4.0, alpha_cross=4.0, max_iter=2000),
    # 32 subdomains of up to 28.6k rows: beyond the round-1 shared-memory cap (25.6k)
    "oras_ns32": dict(method="oras", alpha=4.0, alpha_cross=40.0, max_iter=2000, n_subdomains=32),
}
HEADLINE_STRIDE = 97


def label_hash(labels) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(labels, np.int32).tobytes()).hexdigest()


def headline(which):
    w = HEADLINE[which]
    ns = w.get("n_subdomains", 256)
    cfg = dict(surface="sphere", h=0.0125, p=3, c=1.0, method=w["method"], mode="gmres", gmres_restart=50,
               n_overlap=3, n_subdomains=ns, rel_tol=1e-10, max_iter=w["max_iter"])
    if w["method"] == "oras":
        cfg.update(alpha=w["alpha"], alpha_cross=w["alpha_cross"])
    t0 = time.time()
    R = ref.RefProblem(cfg, workers=os.cpu_count())
    cp = R.band()["cp"][: R.n_active]
    part = inputs.rcb_partition(cp, ns)
    aligned, moves = R.decompose(part)
    t1 = time.time()
    n = R.n_active
    x = inputs.uniform_vector(n, 11)
    Ax = R.apply_A(x)
    ptr, col, val = R.csr("A")
    scale = np.add.reduceat(np.abs(val) * np.abs(x[col]), ptr[:-1].astype(np.int64))
    del ptr, col, val
    Mx = R.pc_apply(x)
    b = inputs.rhs_sphere(cp)
    t2 = time.time()
    out = R.solve(b)
    t3 = time.time()
    u = out["u"]
    S = HEADLINE_STRIDE
    rec = dict(n_active=n, n_ghost=R.n_ghost, align_moves=moves, label_sha256=label_hash(aligned),
               n_subdomains=R.n_sub, iterations=out["iterations"], converged=out["converged"],
               final_rel_residual=out["final_true_residual"] / float(np.linalg.norm(b)),
               u_norm2=float(np.linalg.norm(u)), u_norm_inf=float(np.abs(u).max()),
               Ax_norm2=float(np.linalg.norm(Ax)), Mx_norm2=float(np.linalg.norm(Mx)),
               sample_stride=S, probe_seed=11, cfg=cfg,
               _how=(f"tests/golden/make_fullsize.py headline {which}: oracle/_ref own pipeline "
                     f"(build_problem, align_interfaces, build_subdomains, assemble_local, DirectSolver; "
                     f"{os.cpu_count()} threads) {t1 - t0:.0f} s, A x / M x {t2 - t1:.0f} s, "
                     f"gmres_solve {t3 - t2:.0f} s"))
    path = os.path.join(HERE, "fullsize_reference.json")
    d = json.load(open(path))
    d.setdefault("headline_refpipeline", {})[which] = rec
    json.dump(d, open(path, "w"), indent=2)
    np.savez_compressed(os.path.join(HERE, f"fullsize_headline_{which}.npz"), u_sample=u[::S], Ax_sample=Ax[::S],
                        Ax_scale_sample=scale[::S], Mx_sample=Mx[::S], residuals=np.asarray(out["residuals"]))
    print(which, {k: v for k, v in rec.items() if k != "cfg"})


if __name__ == "__main__":
    if sys.argv[1] == "headline":
        for which in (sys.argv[2:] or list(HEADLINE)):
            headline(which)
    else:
        main(sys.argv[1])
