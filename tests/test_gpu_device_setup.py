"""Device setup against the host setup, which is
itself bit-exact with the reference (tests/test_setup_parity.py against
oracle/_ref): the band built on the GPU -- flood fill, closest points
(circle, sphere, torus with glibc's hypot, TriMesh ring search), stencil
closure, lexicographic actives and ghosts -- must be byte-identical (lattice
indices, closest points, normals, distances) on every BASELINE.json
configuration, with both tube radii."""
import os
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SQ13, SQ17 = np.sqrt(13.0), np.sqrt(17.0)

CASES = {
    "circle_h0.0125": dict(surface="circle", h=0.0125),
    "circle_h0.0125_sqrt13h": dict(surface="circle", h=0.0125, tube=SQ13),
    "sphere_h0.05": dict(surface="sphere", h=0.05),
    "sphere_h0.05_sqrt17h": dict(surface="sphere", h=0.05, tube=SQ17),
    "sphere_h0.0125": dict(surface="sphere", h=0.0125),
    "sphere_h0.0125_sqrt17h": dict(surface="sphere", h=0.0125, tube=SQ17),
    "torus_h0.01": dict(surface="torus", h=0.01, major_radius=1.0, minor_radius=0.4),
    "torus_h0.05_sqrt17h": dict(surface="torus", h=0.05, major_radius=1.0, minor_radius=0.4, tube=SQ17),
    "trimesh_h0.01": dict(surface="obj", h=0.01, subdiv=6),
    "trimesh3_h0.05": dict(surface="obj", h=0.05, subdiv=3),
}


def _problem(w, device):
    from paper_1909_08734_b200 import api, inputs
    obj = None
    if w["surface"] == "obj":
        v, f = inputs.displaced_icosphere(w["subdiv"], seed=5)
        obj = os.path.join(tempfile.mkdtemp(prefix="cpddg_mesh_"), "mesh.obj")
        inputs.write_obj(obj, v, f)
    return api.Problem(w["surface"], h=w["h"], p=3, c=1.0, obj_path=obj,
                       major_radius=w.get("major_radius", 2 / 3), minor_radius=w.get("minor_radius", 1 / 3),
                       tube_radius=w.get("tube", 0.0) * w["h"], device_setup=device)


@pytest.mark.parametrize("name", sorted(CASES))
def test_device_band_is_byte_identical_to_host(name):
    w = CASES[name]
    H = _problem(w, False)
    G = _problem(w, True)
    assert (G.n_active, G.n_ghost) == (H.n_active, H.n_ghost)
    bh, bg = H.band(), G.band()
    for k in ("ix", "cp", "normal", "dist"):
        assert bh[k].tobytes() == bg[k].tobytes(), k
    # E and A are assembled from the band: same bits
    if H.n_active < 100000:
        for which in ("E", "A"):
            for a, b in zip(H.csr(which), G.csr(which)):
                assert a.tobytes() == b.tobytes()


DECOMP = {
    "circle_sectors8_ras": dict(surface="circle", h=0.0125, parts=("sectors", 8), no=2, method="ras"),
    "circle_sectors8_oras": dict(surface="circle", h=0.0125, parts=("sectors", 8), no=2, method="oras"),
    "sphere05_rcb64_oras": dict(surface="sphere", h=0.05, parts=("rcb", 64), no=2, method="oras"),
    "sphere05_rcb64_ras_no3": dict(surface="sphere", h=0.05, parts=("rcb", 64), no=3, method="ras"),
    "sphere0125_rcb256_oras_no3": dict(surface="sphere", h=0.0125, parts=("rcb", 256), no=3, method="oras"),
    "sphere0125_rcb32_oras_no3": dict(surface="sphere", h=0.0125, parts=("rcb", 32), no=3, method="oras"),
    "torus_h0.01_rcb512_oras": dict(surface="torus", h=0.01, major_radius=1.0, minor_radius=0.4,
                                    parts=("rcb", 512), no=2, method="oras"),
    "trimesh_h0.01_rcb512_oras": dict(surface="obj", h=0.01, subdiv=6, parts=("rcb", 512), no=2, method="oras"),
}


@pytest.mark.parametrize("name", sorted(DECOMP))
def test_device_subdomain_sets_are_identical_to_host(name):
    """align_interfaces + build_subdomains on the device: aligned labels, move
    count, every index set, every boundary node (integer fields and the bits
    of x, cp, cp_local, conormal, dq) and every local system equal the host's."""
    from paper_1909_08734_b200 import inputs
    w = DECOMP[name]
    H = _problem(w, False)
    G = _problem(w, True)
    cp = H.active_cp
    kind, n = w["parts"]
    part = inputs.rcb_partition(cp, n) if kind == "rcb" else inputs.sector_partition(cp, n)
    ah, mh = H.decompose(part, w["no"], w["method"], 4.0, 40.0)
    ag, mg = G.decompose(part, w["no"], w["method"], 4.0, 40.0)
    assert mg == mh and np.array_equal(ag, ah)
    assert G.n_sub == H.n_sub
    for j in range(H.n_sub):
        sh, sg = H.subdomain(j), G.subdomain(j)
        for k in ("disjoint", "overlap", "final_layer", "ghosts", "bc_int"):
            assert np.array_equal(sh[k], sg[k]), (j, k)
        assert sh["bc_real"].tobytes() == sg["bc_real"].tobytes(), j
        for k in ("fallback_count", "n_lambda", "n_cross_flagged"):
            assert sh[k] == sg[k], (j, k)
    for j in range(0, H.n_sub, max(1, H.n_sub // 16)):
        lh, lg = H.local(j), G.local(j)
        for k in ("ptr", "col", "val", "scatter_local", "scatter_global"):
            assert lh[k].tobytes() == lg[k].tobytes(), (j, k)


def test_device_sets_beyond_limits_fall_back_to_host():
    """More than 1023 subdomains exceed the device sets' index packing: the
    host restatement runs instead and the result is the host's."""
    from paper_1909_08734_b200 import inputs
    w = dict(surface="sphere", h=0.0125)
    H = _problem(w, False)
    G = _problem(w, True)
    part = inputs.rcb_partition(H.active_cp, 1024)
    ah, mh = H.decompose(part, 1, "oras", 4.0, 40.0)
    ag, mg = G.decompose(part, 1, "oras", 4.0, 40.0)
    assert mg == mh and np.array_equal(ag, ah) and G.n_sub == H.n_sub == 1024
    for j in (0, 511, 1023):
        assert np.array_equal(H.subdomain(j)["overlap"], G.subdomain(j)["overlap"])
