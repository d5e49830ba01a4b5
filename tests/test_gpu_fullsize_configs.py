"""BASELINE configs 4 (torus h = 0.01, 512 RCB) and 5 (displaced icosphere,
subdivision 6, h = 0.01, 512 RCB) at full size, ORAS-GMRES(50) with the
modified cross-point condition, against the reference's own full-size solves
(tests/golden/make_fullsize.py: oracle/_ref gmres_solve + DirectSolver):
iteration counts, final residuals and a strided sample of the solution
(1e-8 relative, BASELINE.json north_star)."""
import json
import os
import tempfile

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

CASES = {
    "torus": ("torus_h0.01_rcb512_no2_oras_a4_ax40",
              dict(surface="torus", major_radius=1.0, minor_radius=0.4, h=0.01)),
    "trimesh": ("trimesh_h0.01_rcb512_no2_oras_a4_ax40", dict(surface="obj", h=0.01)),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_full_size_config_matches_reference(name):
    import torch

    from paper_1909_08734_b200 import api, inputs
    key, w = CASES[name]
    golden = json.load(open(os.path.join(GOLDEN, "fullsize_reference.json")))
    npz = os.path.join(GOLDEN, f"fullsize_{name}.npz")
    if key not in golden or not os.path.exists(npz):
        pytest.skip(f"no full-size reference for {name} (tests/golden/make_fullsize.py)")
    ref = golden[key]
    sample = np.load(npz)["u_sample"]
    obj = None
    if w["surface"] == "obj":
        v, f = inputs.displaced_icosphere(6, seed=5)
        obj = os.path.join(tempfile.mkdtemp(prefix="cpddg_mesh_"), "icosphere.obj")
        inputs.write_obj(obj, v, f)
    P = api.Problem(w["surface"], h=w["h"], p=3, c=1.0, obj_path=obj, major_radius=w.get("major_radius", 2 / 3),
                    minor_radius=w.get("minor_radius", 1 / 3))
    assert (P.n_active, P.n_ghost) == (ref["n_active"], ref["n_ghost"])
    cp = P.active_cp
    _, moves = P.decompose(inputs.rcb_partition(cp, 512), 2, "oras", 4.0, 40.0)
    assert moves == ref["align_moves"]
    b_host = inputs.rhs_trig(cp, seed=2024)
    A = api.DeviceHelmholtz.from_problem(P)
    M = api.SchwarzPreconditioner.from_problem(P)
    b = torch.from_numpy(b_host).cuda()
    r = api.gmres_solve(A, b, M, 1e-10, 2000, 50)
    assert r.log.converged and abs(r.log.iterations - ref["iterations"]) <= 2
    assert r.log.final_true_residual <= 1e-10 * np.linalg.norm(b_host) * 1.5
    u = r.u.cpu().numpy()
    us = u[::ref["sample_stride"]]
    assert np.max(np.abs(us - sample)) <= 1e-8 * ref["u_norm_inf"]
    assert abs(np.linalg.norm(u) - ref["u_norm2"]) <= 1e-8 * ref["u_norm2"]


def test_torus_ras_stationary_matches_reference():
    """BASELINE config 4's other run: RAS as a stationary solver on the full
    torus (h = 0.01, 512 RCB parts, overlap 2), against the reference's own
    stationary_solve at full size (tests/golden/make_fullsize.py
    torus_ras_stationary): iteration count within +-2, solution sample 1e-8."""
    import torch

    from paper_1909_08734_b200 import api, inputs
    key = "torus_h0.01_rcb512_no2_ras_stationary"
    golden = json.load(open(os.path.join(GOLDEN, "fullsize_reference.json")))
    npz = os.path.join(GOLDEN, "fullsize_torus_ras_stationary.npz")
    if key not in golden or not os.path.exists(npz):
        pytest.skip("no full-size reference for torus RAS stationary (tests/golden/make_fullsize.py)")
    ref = golden[key]
    sample = np.load(npz)["u_sample"]
    P = api.Problem("torus", h=0.01, p=3, c=1.0, major_radius=1.0, minor_radius=0.4)
    assert (P.n_active, P.n_ghost) == (ref["n_active"], ref["n_ghost"])
    cp = P.active_cp
    _, moves = P.decompose(inputs.rcb_partition(cp, 512), 2, "ras")
    assert moves == ref["align_moves"]
    b_host = inputs.rhs_trig(cp, seed=2024)
    A = api.DeviceHelmholtz.from_problem(P)
    M = api.SchwarzPreconditioner.from_problem(P)
    r = api.stationary_solve(A, torch.from_numpy(b_host).cuda(), M, 1e-10, 5000)
    assert r.log.converged == ref["converged"] and abs(r.log.iterations - ref["iterations"]) <= 2
    u = r.u.cpu().numpy()
    assert np.max(np.abs(u[::ref["sample_stride"]] - sample)) <= 1e-8 * ref["u_norm_inf"]
    assert abs(np.linalg.norm(u) - ref["u_norm2"]) <= 1e-8 * ref["u_norm2"]
