"""Host setup (band, E, A, alignment, subdomains, local systems) vs the
reference built in oracle/_ref: bit for bit.  Plus the reference's own
golden value N_A = 41094 (proj/tests/test_band.cpp:115-126) and the
reference's error behaviour for bad partitions / parameters."""
import numpy as np
import pytest

from conftest import needs_ref

from paper_1909_08734_b200 import api, errors, inputs


def test_band_golden_count_sphere_h25_p2():
    """proj/tests/test_band.cpp:115-126: unit sphere, h = 1/25, p = 2 -> 41094 actives."""
    P = api.Problem("sphere", h=1.0 / 25.0, p=2)
    assert P.n_active == 41094


def test_extension_and_helmholtz_identities():
    """E 1 = 1 (test_operators.cpp:125-139) and A 1 = c 1 (:284-297) on the host matrices."""
    import scipy.sparse as sp
    for surf, h, p in [("circle", 0.05, 3), ("sphere", 0.1, 3), ("torus", 0.08, 2)]:
        P = api.Problem(surf, h=h, p=p, c=3.7, major_radius=1.0, minor_radius=0.4)
        ptr, col, val = P.csr("E")
        E = sp.csr_matrix((val, col, ptr), shape=(P.n_active + P.n_ghost, P.n_active))
        assert np.abs(E @ np.ones(P.n_active) - 1).max() <= 1e-12
        assert np.all(np.diff(ptr) == (p + 1) ** P.dim)
        ptr, col, val = P.csr("A")
        A = sp.csr_matrix((val, col, ptr), shape=(P.n_active, P.n_active))
        assert np.abs(A @ np.ones(P.n_active) - 3.7).max() <= 1e-10 * (2 * P.dim / h ** 2)


CASES = [
    ("circle", dict(h=0.0125, p=3), "sector", 8, 2, "oras", 1.0, -1.0),
    ("circle", dict(h=0.05, p=3), "sector", 4, 3, "ras", 1.0, -1.0),
    ("sphere", dict(h=0.1, p=3), "rcb", 16, 2, "oras", 4.0, 40.0),
    ("sphere", dict(h=0.1, p=2), "rcb", 8, 3, "ras", 1.0, -1.0),
    ("torus", dict(h=0.06, p=3, major_radius=1.0, minor_radius=0.4), "rcb", 16, 2, "oras", 2.0, 20.0),
    ("obj", dict(h=0.1, p=3), "rcb", 8, 2, "oras", 4.0, 40.0),
]


@needs_ref
@pytest.mark.parametrize("surf,geo,pk,ns,no,meth,alpha,ax", CASES)
def test_setup_bit_exact_vs_reference(surf, geo, pk, ns, no, meth, alpha, ax):
    import os

    import ref
    from conftest import GOLDEN
    cfg = dict(surface=surf, c=1.0, method=meth, n_overlap=no, n_subdomains=ns, alpha=alpha, alpha_cross=ax, **geo)
    obj = os.path.join(GOLDEN, "icosphere3.obj") if surf == "obj" else None
    if obj:
        cfg["obj"] = obj
    R = ref.RefProblem(cfg, workers=4)
    P = api.Problem(surf, h=geo["h"], p=geo["p"], c=1.0, major_radius=geo.get("major_radius", 2 / 3),
                    minor_radius=geo.get("minor_radius", 1 / 3), obj_path=obj, workers=4)
    assert (P.n_active, P.n_ghost) == (R.n_active, R.n_ghost)
    B, RB = P.band(), R.band()
    for k in ("ix", "cp", "normal", "dist"):
        assert np.array_equal(B[k].view(np.uint8), RB[k].view(np.uint8)), k
    for which in ("E", "A"):
        a, b = P.csr(which), R.csr(which)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        assert np.array_equal(a[2].view(np.int64), b[2].view(np.int64)), which
    cp = B["cp"][: P.n_active]
    part = inputs.sector_partition(cp, ns) if pk == "sector" else inputs.rcb_partition(cp, ns)
    aligned, moves = P.decompose(part, no, meth, alpha, ax)
    raligned, rmoves = R.decompose(part, factor=False)
    assert np.array_equal(aligned, raligned) and moves == rmoves
    for j in range(P.n_sub):
        S, RS = P.subdomain(j), R.subdomain(j)
        for k in ("disjoint", "overlap", "final_layer", "ghosts"):
            assert np.array_equal(S[k], getattr(RS, k)), (j, k)
        assert np.array_equal(S["bc_int"], RS.bc_int), j
        assert np.array_equal(S["bc_real"].view(np.int64), RS.bc_real.view(np.int64)), j
        assert S["fallback_count"] == RS.fallback_count and S["n_lambda"] == RS.n_lambda
        L, RL = P.local(j), R.local(j)
        assert (L["n_overlap"], L["n_bc"]) == (RL["n_overlap"], RL["n_bc"])
        for k in ("ptr", "col", "scatter_local", "scatter_global"):
            assert np.array_equal(L[k], RL[k]), (j, k)
        assert np.array_equal(L["val"].view(np.int64), RL["val"].view(np.int64)), j


def test_cross_points_flag_on_sphere():
    """subdomain.hpp:305-309: with several parts meeting, some BC nodes are cross-flagged."""
    P = api.Problem("sphere", h=0.1, p=3)
    P.decompose(inputs.rcb_partition(P.active_cp, 8), 2, "oras", 2.0, 80.0)
    assert sum(P.subdomain(j)["n_cross_flagged"] for j in range(P.n_sub)) > 0


def test_partition_validation_matches_load_partition():
    """partition.hpp:519-552 error behaviour, and align_interfaces' empty-part refusal."""
    P = api.Problem("circle", h=0.05, p=3)
    n = P.n_active
    with pytest.raises(errors.ConfigError, match="entries but the mesh has"):
        P.decompose(np.zeros(n - 1, np.int32), 2, "ras")
    bad = np.zeros(n, np.int32)
    bad[0] = -1
    with pytest.raises(errors.ConfigError, match="negative label"):
        P.decompose(bad, 2, "ras")
    gap = np.zeros(n, np.int32)
    gap[: n // 2] = 2
    with pytest.raises(errors.ConfigError, match="skip part 1"):
        P.decompose(gap, 2, "ras")
    with pytest.raises(errors.ConfigError):
        P.decompose(np.zeros(n, np.int32), 0, "ras")
    with pytest.raises(errors.ConfigError, match="alpha_cross must be at least alpha"):
        P.decompose(np.zeros(n, np.int32), 2, "oras", 4.0, 2.0)
    # a singleton part that alignment pulls into its neighbour (test_partition.cpp:197-214)
    part = inputs.sector_partition(P.active_cp, 2)
    moved = None
    for i in range(n):
        cand = part.copy()
        cand[i] = 2
        try:
            P.decompose(cand, 2, "ras")
        except errors.ConfigError as e:
            moved = str(e)
            break
    assert moved is not None and "emptied part" in moved


def test_decompose_is_deterministic_across_worker_counts():
    P1 = api.Problem("sphere", h=0.1, p=3, workers=1)
    P8 = api.Problem("sphere", h=0.1, p=3, workers=8)
    part = inputs.rcb_partition(P1.active_cp, 16)
    P1.decompose(part, 2, "oras", 4.0, 40.0)
    P8.decompose(part, 2, "oras", 4.0, 40.0)
    for j in range(16):
        a, b = P1.local(j), P8.local(j)
        assert np.array_equal(a["ptr"], b["ptr"]) and np.array_equal(a["col"], b["col"])
        assert np.array_equal(a["val"].view(np.int64), b["val"].view(np.int64))
