"""Generate tests/golden/*.npz from the REFERENCE (oracle/_ref/libcpdd_ref.so,
the unmodified /root/reference headers compiled against oracle/shim).

Run here (needs /root/reference and `make -C oracle`):
    python tests/golden/make_golden.py
Each case stores the reference's outputs on seeded inputs: A x and M x for
x ~ U(-1,1) (splitmix64), the aligned partition, and the solve (u, iteration
count, residual history).  Inputs follow SURVEY.md section 8(d): sector / RCB
partitions, the BASELINE right-hand sides, p = 3, c = 1, reference tube radius.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import ref  # noqa: E402
from paper_1909_08734_b200 import inputs  # noqa: E402

CASES = {
    # BASELINE config 1 (circle, 8 angular sectors, N_O = 2, GMRES(50) and stationary RAS)
    "circle_ras_gmres": dict(cfg=dict(surface="circle", h=0.0125, method="ras", mode="gmres", gmres_restart=50,
                                      n_overlap=2, n_subdomains=8), part="sector", rhs="circle"),
    "circle_oras_gmres": dict(cfg=dict(surface="circle", h=0.0125, method="oras", mode="gmres", gmres_restart=50,
                                       n_overlap=2, n_subdomains=8, alpha=1.0), part="sector", rhs="circle"),
    "circle_ras_stationary": dict(cfg=dict(surface="circle", h=0.0125, method="ras", mode="stationary",
                                           n_overlap=2, n_subdomains=8, max_iter=20000), part="sector", rhs="circle"),
    # coarse sphere: ORAS with the modified cross-point condition, and RAS
    "sphere10_oras_gmres": dict(cfg=dict(surface="sphere", h=0.1, method="oras", mode="gmres", gmres_restart=50,
                                         n_overlap=2, n_subdomains=16, alpha=4.0, alpha_cross=40.0),
                                part="rcb", rhs="sphere"),
    "sphere10_oras_stationary": dict(cfg=dict(surface="sphere", h=0.1, method="oras", mode="stationary",
                                              n_overlap=2, n_subdomains=16, alpha=4.0, alpha_cross=40.0,
                                              max_iter=20000), part="rcb", rhs="sphere"),
    # BASELINE config 2 (sphere h = 0.05, 64 RCB, N_O = 2)
    "sphere05_oras_gmres": dict(cfg=dict(surface="sphere", h=0.05, method="oras", mode="gmres", gmres_restart=50,
                                         n_overlap=2, n_subdomains=64, alpha=4.0, alpha_cross=40.0),
                                part="rcb", rhs="sphere"),
    "sphere05_ras_gmres": dict(cfg=dict(surface="sphere", h=0.05, method="ras", mode="gmres", gmres_restart=50,
                                        n_overlap=2, n_subdomains=64), part="rcb", rhs="sphere"),
    # standard Robin condition (alpha_cross = alpha) at BASELINE config 2
    "sphere05_oras_std_gmres": dict(cfg=dict(surface="sphere", h=0.05, method="oras", mode="gmres",
                                             gmres_restart=50, n_overlap=2, n_subdomains=64, alpha=4.0),
                                    part="rcb", rhs="sphere"),
    # displaced icosphere (BASELINE config 5 geometry, subdivision 3), TriMesh closest points
    "trimesh3_oras_gmres": dict(cfg=dict(surface="obj", obj=os.path.join(HERE, "icosphere3.obj"), h=0.05,
                                         method="oras", mode="gmres", gmres_restart=50, n_overlap=2,
                                         n_subdomains=16, alpha=4.0, alpha_cross=40.0), part="rcb", rhs="trig"),
    # coarse torus (BASELINE config 4 geometry), seeded trigonometric right-hand side
    "torus04_oras_gmres": dict(cfg=dict(surface="torus", major_radius=1.0, minor_radius=0.4, h=0.04,
                                        method="oras", mode="gmres", gmres_restart=50, n_overlap=2,
                                        n_subdomains=32, alpha=2.0, alpha_cross=20.0), part="rcb", rhs="trig"),
}


def make_case(name, spec):
    cfg = dict(p=3, c=1.0, rel_tol=1e-10, max_iter=2000)
    cfg.update(spec["cfg"])
    R = ref.RefProblem(cfg, workers=os.cpu_count() or 1)
    B = R.band()
    na = R.n_active
    cp = B["cp"][:na]
    part = inputs.sector_partition(cp, cfg["n_subdomains"]) if spec["part"] == "sector" \
        else inputs.rcb_partition(cp, cfg["n_subdomains"])
    b = {"circle": inputs.rhs_circle, "sphere": inputs.rhs_sphere,
         "trig": lambda q: inputs.rhs_trig(q, seed=2024)}[spec["rhs"]](cp)
    x = inputs.uniform_vector(na, 11)
    Ax = R.apply_A(x)
    aligned, moves = R.decompose(part)
    Mx = R.pc_apply(x)
    sol = R.solve(b)
    cfg_store = dict(cfg)
    if "obj" in cfg_store:
        cfg_store["obj"] = os.path.basename(cfg_store["obj"])  # resolved against tests/golden/
    np.savez_compressed(os.path.join(HERE, name + ".npz"),
                        cfg=np.array(repr(cfg_store)), n_active=na, n_ghost=R.n_ghost,
                        part_in=part, part_aligned=aligned, moves=moves, x=x, Ax=Ax, Mx=Mx, b=b,
                        u=sol["u"], iterations=sol["iterations"], converged=sol["converged"],
                        residuals=sol["residuals"], final_true_residual=sol["final_true_residual"])
    print(f"{name}: N_A={na} moves={moves} iters={sol['iterations']} conv={sol['converged']}", flush=True)


if __name__ == "__main__":
    only = sys.argv[1:]
    for name, spec in CASES.items():
        if not only or name in only:
            make_case(name, spec)
