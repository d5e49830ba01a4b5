"""Pins of the oracle (CPU, test infrastructure):
  * the reference built in oracle/_ref passes the reference's OWN GTest
    suites (proj/tests/*.cpp, incl. the N_A = 41094 band golden value);
  * the numpy/scipy restatement (oracle/cpdd_oracle.py) reproduces the
    reference's outputs stored in tests/golden/ (generated from oracle/_ref by
    tests/golden/make_golden.py) and the reference run live."""
import ast
import os
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, needs_ref

import cpdd_oracle as O
from paper_1909_08734_b200 import api, inputs

REF_SUITES = ["test_band", "test_operators", "test_partition", "test_solve", "test_transmission",
              "test_subdomain", "test_geometry"]


@needs_ref
@pytest.mark.parametrize("suite", REF_SUITES)
def test_reference_suite_passes_against_shim(suite):
    exe = os.path.join(ROOT, "oracle", "_ref", suite)
    if not os.path.exists(exe):
        pytest.skip(f"{suite} not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, TEST_TMPDIR="/tmp"))
    tail = r.stderr.strip().splitlines()[-1]
    assert r.returncode == 0 and " 0 failed" in tail, r.stderr[-3000:]


def _golden(name):
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    return g, ast.literal_eval(str(g["cfg"]))


SMALL = ["circle_ras_gmres", "circle_oras_gmres", "sphere10_oras_gmres", "circle_ras_stationary",
         "sphere10_oras_stationary"]


@pytest.mark.parametrize("name", SMALL)
def test_restatement_matches_golden(name):
    """Operator (assembled by the restatement from the band), preconditioner
    (SuperLU-COLAMD local solves) and the solver loops vs the reference."""
    g, cfg = _golden(name)
    P = api.Problem(cfg["surface"], h=cfg["h"], p=cfg["p"], c=cfg["c"])
    B = P.band()
    na = P.n_active
    E = O.build_extension(B["ix"], B["cp"], na, cfg["h"], cfg["p"])
    A = O.assemble_helmholtz(B["ix"], E, na, cfg["h"], cfg["c"])
    ptr, col, val = P.csr("A")
    assert O.op_rel_error(ptr, col, val, g["x"], A @ g["x"], g["Ax"]) <= 1e-12
    P.decompose(g["part_in"], cfg["n_overlap"], cfg["method"], cfg.get("alpha", 1.0), cfg.get("alpha_cross", -1.0))
    M = O.Schwarz([P.local(j) for j in range(P.n_sub)])
    assert np.linalg.norm(M(g["x"]) - g["Mx"]) <= 1e-9 * np.linalg.norm(g["Mx"])
    if cfg["mode"] == "gmres":
        r = O.gmres_solve(lambda v: A @ v, M, g["b"], cfg["rel_tol"], cfg["max_iter"], cfg.get("gmres_restart", 0))
    else:
        r = O.stationary_solve(lambda v: A @ v, M, g["b"], cfg["rel_tol"], cfg["max_iter"])
    assert r["converged"] and abs(r["iterations"] - int(g["iterations"])) <= 2
    assert np.linalg.norm(r["u"] - g["u"]) <= 1e-8 * np.linalg.norm(g["u"])


def test_weights_exact_hit_and_partition_of_unity():
    """interp.hpp:35-54: unit vector on exact hits, weights sum to one,
    polynomial exactness up to degree p (test_operators.cpp:141-160)."""
    for p in (1, 2, 3, 4):
        t = np.array([0.0, 0.3, 1.0, p / 2 + 0.1, float(p)])
        w = O.weights_1d(p, t)
        assert np.allclose(w.sum(1), 1.0, atol=1e-14)
        assert np.array_equal(w[0], np.eye(p + 1)[0]) and np.array_equal(w[-1], np.eye(p + 1)[p])
        for k in range(p + 1):
            assert np.allclose(w @ (np.arange(p + 1) ** k), t ** k, atol=1e-12)
    with pytest.raises(ValueError):
        O.weights_1d(3, np.array([3.5]))


@needs_ref
def test_restatement_matches_reference_live_torus():
    import ref
    cfg = dict(surface="torus", major_radius=1.0, minor_radius=0.4, h=0.08, p=3, c=1.0, method="oras",
               mode="gmres", gmres_restart=20, n_overlap=2, n_subdomains=8, alpha=2.0, alpha_cross=20.0,
               rel_tol=1e-10, max_iter=500)
    R = ref.RefProblem(cfg, workers=4)
    B = R.band()
    na = R.n_active
    E = O.build_extension(B["ix"], B["cp"], na, R.h, R.p)
    A = O.assemble_helmholtz(B["ix"], E, na, R.h, 1.0)
    x = inputs.uniform_vector(na, 5)
    ptr, col, val = R.csr("A")
    assert O.op_rel_error(ptr, col, val, x, A @ x, R.apply_A(x)) <= 1e-12
    part = inputs.rcb_partition(B["cp"][:na], 8)
    R.decompose(part)
    locs = []
    for j in range(R.n_sub):
        L = R.local(j)
        L["overlap"] = R.subdomain(j).overlap
        locs.append(L)
    M = O.Schwarz(locs)
    assert np.linalg.norm(M(x) - R.pc_apply(x)) <= 1e-9 * np.linalg.norm(R.pc_apply(x))
    b = inputs.rhs_trig(B["cp"][:na], seed=7)
    o = O.gmres_solve(lambda v: A @ v, M, b, 1e-10, 500, 20)
    r = R.solve(b)
    assert abs(o["iterations"] - r["iterations"]) <= 2
    assert np.linalg.norm(o["u"] - r["u"]) <= 1e-8 * np.linalg.norm(r["u"])


def test_inputs_are_deterministic():
    a = inputs.rhs_trig(np.random.default_rng(0).normal(size=(50, 3)), seed=11)
    b = inputs.rhs_trig(np.random.default_rng(0).normal(size=(50, 3)), seed=11)
    assert np.array_equal(a, b)
    ks, ph = inputs.trig_modes(11)
    assert ks.min() >= -4 and ks.max() <= 4 and ph.min() >= 0 and ph.max() < 2 * np.pi
    assert inputs.SplitMix64(1).next_u64() == 0x910A2DEC89025CC1  # splitmix64 reference output
    part = inputs.rcb_partition(np.random.default_rng(1).normal(size=(1000, 3)), 16)
    assert sorted(np.bincount(part)) == [62] * 8 + [63] * 8
