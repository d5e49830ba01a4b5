"""The headline configuration at full size (BASELINE configs[2]: N_A = 558,806),
checked through size-independent properties and the reference's own full-size
results (tests/golden/fullsize_reference.json, measured with oracle/_ref):
operator identities, factor probe residuals, iteration counts, final residuals
and the discretisation error against the exact solution."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def headline():
    from paper_1909_08734_b200 import api, inputs
    ref = json.load(open(os.path.join(GOLDEN, "fullsize_reference.json")))["sphere_h0.0125_rcb256_no3"]
    P = api.Problem("sphere", h=0.0125, p=3, c=1.0)
    part = inputs.rcb_partition(P.active_cp, 256)
    return P, part, ref


def test_band_and_alignment_match_reference(headline):
    P, part, ref = headline
    assert (P.n_active, P.n_ghost) == (ref["n_active"], ref["n_ghost"])
    _, moves = P.decompose(part, 3, "ras")
    assert moves == ref["align_moves"]


def test_operator_identities_full_size(headline):
    """A 1 = c 1 (test_operators.cpp:284-297) and linearity, on the device."""
    import torch

    from paper_1909_08734_b200 import api, inputs
    P, _, _ = headline
    A = api.DeviceHelmholtz.from_problem(P)
    one = torch.ones(P.n_active, dtype=torch.float64, device="cuda")
    y = A.apply(one)
    gamma = 6.0 / 0.0125 ** 2
    assert float((y - 1.0).abs().max()) <= 1e-10 * gamma
    x1 = torch.from_numpy(inputs.uniform_vector(P.n_active, 1)).cuda()
    x2 = torch.from_numpy(inputs.uniform_vector(P.n_active, 2)).cuda()
    lhs = A.apply(2.5 * x1 - x2)
    rhs = 2.5 * A.apply(x1) - A.apply(x2)
    assert float((lhs - rhs).abs().max()) <= 1e-12 * gamma * 4


@pytest.mark.parametrize("method,alpha,ax,key", [("oras", 4.0, 40.0, "oras_a4_ax40"), ("ras", 1.0, -1.0, "ras")])
def test_solve_matches_reference_full_size(headline, method, alpha, ax, key):
    import torch

    from paper_1909_08734_b200 import api, inputs
    P, part, ref = headline
    P.decompose(part, 3, method, alpha, ax)
    A = api.DeviceHelmholtz.from_problem(P)
    M = api.SchwarzPreconditioner.from_problem(P)
    assert M.stats()["max_probe_residual"] <= 1e-12
    b = inputs.rhs_sphere(P.active_cp)
    res = api.gmres_solve(A, torch.from_numpy(b).cuda(), M, 1e-10, 2000, 50)
    r = ref[key]
    assert res.log.converged == r["converged"]
    assert abs(res.log.iterations - r["iterations"]) <= 2
    rel = res.log.final_true_residual / np.linalg.norm(b)
    assert rel <= 1e-10 and abs(rel - r["final_rel_residual"]) <= 0.05 * r["final_rel_residual"]
    u = res.u.cpu().numpy()
    err = np.abs(u - inputs.exact_sphere(P.active_cp)).max()
    assert abs(err - r["err_inf_vs_exact"]) <= 1e-3 * r["err_inf_vs_exact"]


def test_standard_oras_stagnates_like_the_reference(headline):
    """BASELINE config 3 with the standard Robin condition (alpha_cross =
    alpha = 4): the reference's GMRES(50) stagnates -- 2000 iterations, not
    converged, relative residual 0.99975 (fullsize_reference.json) -- the
    cross-point pathology that the modified condition removes.  The device
    solve reproduces the stagnation and its level."""
    import torch

    from paper_1909_08734_b200 import api, inputs
    P, part, ref = headline
    r = ref["oras_a4_ax4"]
    P.decompose(part, 3, "oras", 4.0, 4.0)
    A = api.DeviceHelmholtz.from_problem(P)
    M = api.SchwarzPreconditioner.from_problem(P)
    b = inputs.rhs_sphere(P.active_cp)
    res = api.gmres_solve(A, torch.from_numpy(b).cuda(), M, 1e-10, 2000, 50)
    assert not res.log.converged and not r["converged"]
    assert res.log.iterations == r["iterations"] == 2000
    rel = res.log.final_true_residual / np.linalg.norm(b)
    assert abs(rel - r["final_rel_residual"]) <= 1e-3
