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
