"""Device path vs the reference (golden vectors from oracle/_ref) and the
oracle restatement (oracle/cpdd_oracle.py), through the C ABI.

Tolerances (BASELINE.json north_star): operator applies 1e-12 in the
componentwise-scaled metric max_i |dy_i| / sum_j |A_ij x_j|; final solutions
1e-8 relative; GMRES / stationary iteration counts within +-2.  The
preconditioner apply is checked at 1e-9 relative (different LU backends,
each with a ~1e-12 residual contract)."""
import ast
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

CASES = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and not f.startswith(("fullsize_", "scale_")))


def _setup(name):
    import torch

    from paper_1909_08734_b200 import api
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    cfg = ast.literal_eval(str(g["cfg"]))
    obj = os.path.join(GOLDEN, cfg["obj"]) if "obj" in cfg else None
    P = api.Problem(cfg["surface"], h=cfg["h"], p=cfg["p"], c=cfg["c"], obj_path=obj,
                    major_radius=cfg.get("major_radius", 2.0 / 3.0), minor_radius=cfg.get("minor_radius", 1.0 / 3.0))
    assert P.n_active == int(g["n_active"]) and P.n_ghost == int(g["n_ghost"])
    aligned, moves = P.decompose(g["part_in"], cfg["n_overlap"], cfg["method"], cfg.get("alpha", 1.0),
                                 cfg.get("alpha_cross", -1.0))
    assert np.array_equal(aligned, g["part_aligned"]) and moves == int(g["moves"])
    A = api.DeviceHelmholtz.from_problem(P)
    M = api.SchwarzPreconditioner.from_problem(P)
    return g, cfg, P, A, M, torch


@pytest.mark.parametrize("name", CASES)
def test_operator_matches_reference(name):
    import cpdd_oracle as O
    g, cfg, P, A, M, torch = _setup(name)
    x = g["x"]
    y = A.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    ptr, col, val = P.csr("A")
    assert O.op_rel_error(ptr, col, val, x, y, g["Ax"]) <= 1e-12
    # normwise as well
    assert np.linalg.norm(y - g["Ax"]) <= 1e-13 * np.linalg.norm(np.abs(val)) * np.linalg.norm(x) + 1e-12 * np.linalg.norm(g["Ax"])


@pytest.mark.parametrize("name", CASES)
def test_preconditioner_matches_reference(name):
    g, cfg, P, A, M, torch = _setup(name)
    z = M.apply(torch.from_numpy(g["x"]).cuda()).cpu().numpy()
    assert np.linalg.norm(z - g["Mx"]) <= 1e-9 * np.linalg.norm(g["Mx"])
    # deterministic: a second apply is bitwise identical
    z2 = M.apply(torch.from_numpy(g["x"]).cuda()).cpu().numpy()
    assert np.array_equal(z, z2)


@pytest.mark.parametrize("name", CASES)
def test_solve_matches_reference(name):
    from paper_1909_08734_b200 import api
    g, cfg, P, A, M, torch = _setup(name)
    b = torch.from_numpy(g["b"]).cuda()
    if cfg["mode"] == "gmres":
        res = api.gmres_solve(A, b, M, cfg["rel_tol"], cfg["max_iter"], cfg.get("gmres_restart", 0))
    else:
        res = api.stationary_solve(A, b, M, cfg["rel_tol"], cfg["max_iter"])
    u = res.u.cpu().numpy()
    it_ref = int(g["iterations"])
    assert res.log.converged
    assert abs(res.log.iterations - it_ref) <= 2, (res.log.iterations, it_ref)
    assert len(res.log.residuals) == res.log.iterations + 1
    assert abs(res.log.residuals[0] - np.linalg.norm(g["b"])) <= 1e-12 * np.linalg.norm(g["b"])
    assert res.log.residuals[-1] <= cfg["rel_tol"] * res.log.residuals[0]
    assert np.linalg.norm(u - g["u"]) <= 1e-8 * np.linalg.norm(g["u"])
    assert abs(res.log.final_true_residual - np.linalg.norm(g["b"] - A.apply(res.u).cpu().numpy())) <= \
        1e-6 * res.log.final_true_residual + 1e-300


def test_against_oracle_restatement_small_sphere():
    """GMRES(50) ORAS on a sphere, device vs the numpy/scipy restatement."""
    import torch

    import cpdd_oracle as O
    from paper_1909_08734_b200 import api, inputs
    P = api.Problem("sphere", h=0.1, p=3, c=1.0)
    part = inputs.rcb_partition(P.active_cp, 8)
    P.decompose(part, 2, "oras", 2.0, 20.0)
    A = api.DeviceHelmholtz.from_problem(P)
    M = api.SchwarzPreconditioner.from_problem(P)
    ptr, col, val = P.csr("A")
    Mo = O.Schwarz([P.local(j) for j in range(P.n_sub)])
    b = inputs.rhs_sphere(P.active_cp)
    ref = O.gmres_solve(lambda v: O.csr_apply(ptr, col, val, v), Mo, b, 1e-10, 500, 50)
    res = api.gmres_solve(A, torch.from_numpy(b).cuda(), M, 1e-10, 500, 50)
    assert abs(res.log.iterations - ref["iterations"]) <= 2
    assert np.linalg.norm(res.u.cpu().numpy() - ref["u"]) <= 1e-8 * np.linalg.norm(ref["u"])
    x = inputs.uniform_vector(P.n_active, 5)
    z = M.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    zo = Mo(x)
    assert np.linalg.norm(z - zo) <= 1e-9 * np.linalg.norm(zo)


def test_plain_gmres_without_preconditioner():
    import torch

    import cpdd_oracle as O
    from paper_1909_08734_b200 import api, inputs
    P = api.Problem("circle", h=0.05, p=3, c=1.0)
    A = api.DeviceHelmholtz.from_problem(P)
    ptr, col, val = P.csr("A")
    b = inputs.rhs_circle(P.active_cp)
    ref = O.gmres_solve(lambda v: O.csr_apply(ptr, col, val, v), None, b, 1e-10, 400)
    res = api.gmres_solve(A, torch.from_numpy(b).cuda(), None, 1e-10, 400)
    assert res.log.converged and abs(res.log.iterations - ref["iterations"]) <= 2
    assert np.linalg.norm(res.u.cpu().numpy() - ref["u"]) <= 1e-8 * np.linalg.norm(ref["u"])


def test_zero_rhs_short_circuits():
    import torch

    from paper_1909_08734_b200 import api, inputs
    P = api.Problem("circle", h=0.1, p=2, c=1.0)
    P.decompose(inputs.sector_partition(P.active_cp, 2), 2, "ras")
    A = api.DeviceHelmholtz.from_problem(P)
    M = api.SchwarzPreconditioner.from_problem(P)
    zero = torch.zeros(P.n_active, dtype=torch.float64, device="cuda")
    for res in (api.stationary_solve(A, zero, M, 1e-8, 50), api.gmres_solve(A, zero, M, 1e-8, 50)):
        assert res.log.converged and res.log.iterations == 0
        assert res.log.residuals == [0.0] and res.log.final_true_residual == 0.0
        assert float(res.u.abs().max()) == 0.0


def test_single_subdomain_is_exact_inverse():
    import torch

    from paper_1909_08734_b200 import api, inputs
    P = api.Problem("circle", h=0.1, p=2, c=1.0)
    P.decompose(np.zeros(P.n_active, np.int32), 4, "ras")
    A = api.DeviceHelmholtz.from_problem(P)
    M = api.SchwarzPreconditioner.from_problem(P)
    b = torch.from_numpy(inputs.uniform_vector(P.n_active, 3)).cuda()
    res = api.stationary_solve(A, b, M, 1e-10, 50)
    assert res.log.converged and res.log.iterations == 1 and len(res.log.residuals) == 2
    assert res.log.final_true_residual <= 1e-10 * float(b.norm())


def _identity_locals(n, s):
    return [dict(n_overlap=n, n_bc=0, overlap=np.arange(n), scatter_local=np.arange(n),
                 scatter_global=np.arange(n), ptr=np.arange(n + 1), col=np.arange(n), val=np.full(n, s))]


def test_divergence_is_detected():
    """solve.hpp:115 -- a preconditioner scaled -3x makes the iteration grow."""
    import torch

    from paper_1909_08734_b200 import api, errors, inputs
    P = api.Problem("circle", h=0.1, p=2, c=1.0)
    A = api.DeviceHelmholtz.from_problem(P)
    M = api.SchwarzPreconditioner.from_locals(P.n_active, _identity_locals(P.n_active, -1.0 / 3.0))
    b = torch.from_numpy(inputs.uniform_vector(P.n_active, 41)).cuda()
    with pytest.raises(errors.DivergenceError):
        api.stationary_solve(A, b, M, 1e-8, 1000)


def test_singular_local_factor_raises():
    """direct.hpp:47-50: a singular local system is a DivergenceError."""
    from paper_1909_08734_b200 import api, errors
    with pytest.raises(errors.DivergenceError, match="singular factorization of subdomain 0"):
        api.SchwarzPreconditioner.from_locals(10, _identity_locals(10, 0.0))


def test_overlapping_scatter_rejected():
    from paper_1909_08734_b200 import api, errors
    L = _identity_locals(10, 1.0) * 2
    with pytest.raises(errors.InternalError):
        api.SchwarzPreconditioner.from_locals(10, L)


def test_drop_in_band_descriptor_matches_setup():
    """cpddg_op_create from plain band arrays (the reference BandGrid fields)
    gives the same operator as the setup-built one, bit for bit."""
    import torch

    from paper_1909_08734_b200 import api, inputs
    P = api.Problem("sphere", h=0.1, p=3, c=1.0)
    B = P.band()
    A1 = api.DeviceHelmholtz.from_problem(P)
    A2 = api.DeviceHelmholtz.from_band(3, 3, 0.1, 1.0, P.n_active, B["ix"], B["cp"])
    x = torch.from_numpy(inputs.uniform_vector(P.n_active, 9)).cuda()
    assert torch.equal(A1.apply(x), A2.apply(x))


@pytest.mark.parametrize("h", [0.1, 0.025])
def test_staged_extension_matches_gather_kernel(h, monkeypatch):
    """The union-staged extension kernel (d = 3, p = 3 default), the
    per-base grouped kernel (CPDDG_EXT=grouped), the tiled staged kernel
    (CPDDG_EXT=staged) and the plain gather kernel (CPDDG_EXT_GATHER=1, read at
    create time) give bitwise equal A x: same weights, same summation order."""
    import torch

    from paper_1909_08734_b200 import api, inputs
    P = api.Problem("sphere", h=h, p=3, c=1.0)
    staged = api.DeviceHelmholtz.from_problem(P)
    monkeypatch.setenv("CPDDG_EXT_GATHER", "1")
    gather = api.DeviceHelmholtz.from_problem(P)
    monkeypatch.delenv("CPDDG_EXT_GATHER")
    monkeypatch.setenv("CPDDG_EXT", "staged")
    tiled = api.DeviceHelmholtz.from_problem(P)
    monkeypatch.setenv("CPDDG_EXT", "grouped")
    grouped = api.DeviceHelmholtz.from_problem(P)
    x = torch.from_numpy(inputs.uniform_vector(P.n_active, 5)).cuda()
    for other in (staged, tiled, grouped):
        assert torch.equal(other.apply(x), gather.apply(x))
    # the union (default), grouped and tiled tables were really built
    assert len({staged.bytes()[1], gather.bytes()[1], tiled.bytes()[1], grouped.bytes()[1]}) == 4


@pytest.mark.parametrize("name", ["sphere05_oras_gmres", "torus04_oras_gmres"])
def test_factor_kernels_agree(name, monkeypatch):
    """The pipelined factorisation (k_factor2, default) and the round-1 kernel
    (CPDDG_FACTOR=v1) use the same tensor-core fragments in the same k order:
    bitwise equal factors, hence bitwise equal M x."""
    g, cfg, P, A, M, torch = _setup(name)
    from paper_1909_08734_b200 import api
    monkeypatch.setenv("CPDDG_FACTOR", "v1")
    M1 = api.SchwarzPreconditioner.from_problem(P)
    x = torch.from_numpy(g["x"]).cuda()
    assert torch.equal(M.apply(x), M1.apply(x))
    assert M.stats()["max_probe_residual"] == M1.stats()["max_probe_residual"]


@pytest.mark.parametrize("name", ["sphere05_oras_gmres", "circle_ras_gmres"])
def test_factor_layouts_agree(name, monkeypatch):
    """The factor layouts give the same preconditioner: nonsymmetric
    envelopes (default) vs the symmetric profile (CPDDG_ENVELOPE=sym), and
    the reversed-U-row backward (default) vs the column backward
    (CPDDG_BWD_LAYOUT=cols).  All four within 1e-13 of each other and of the
    reference at the usual 1e-9."""
    import torch

    from paper_1909_08734_b200 import api
    g, cfg, P, A, M, torch = _setup(name)
    x = torch.from_numpy(g["x"]).cuda()
    z0 = M.apply(x).cpu().numpy()
    for env, val in (("CPDDG_ENVELOPE", "sym"), ("CPDDG_BWD_LAYOUT", "cols")):
        monkeypatch.setenv(env, val)
        Mv = api.SchwarzPreconditioner.from_problem(P)
        z = Mv.apply(x).cpu().numpy()
        assert np.linalg.norm(z - z0) <= 1e-13 * np.linalg.norm(z0), (env, val)
        assert np.linalg.norm(z - g["Mx"]) <= 1e-9 * np.linalg.norm(g["Mx"])
    st = M.stats()
    assert st["profile_entries"] <= st["factor_entries"]


def test_dense_small_system_mode_matches_envelope_solve(monkeypatch):
    """Small configurations use dense local inverses (k_solve_dense); they
    agree with the envelope triangular solves to 1e-12 and with the
    reference at the usual 1e-9, and the solve takes the same iterations."""
    import torch

    from paper_1909_08734_b200 import api
    g, cfg, P, A, M, torch = _setup("circle_oras_gmres")
    monkeypatch.setenv("CPDDG_DENSE", "0")
    Me = api.SchwarzPreconditioner.from_problem(P)
    assert M.stats()["apply_mode"] == 1 and Me.stats()["apply_mode"] in (0, 2, 3)  # envelope: register or streamed
    x = torch.from_numpy(g["x"]).cuda()
    zd, ze = M.apply(x).cpu().numpy(), Me.apply(x).cpu().numpy()
    assert np.linalg.norm(zd - ze) <= 1e-12 * np.linalg.norm(ze)
    assert np.linalg.norm(zd - g["Mx"]) <= 1e-9 * np.linalg.norm(g["Mx"])
    b = torch.from_numpy(g["b"]).cuda()
    rd = api.gmres_solve(A, b, M, 1e-10, 500, 50)
    re = api.gmres_solve(A, b, Me, 1e-10, 500, 50)
    assert rd.log.iterations == re.log.iterations == int(g["iterations"]) and rd.log.converged


def test_pipelined_gmres_matches_synchronous_loop(monkeypatch):
    """The pipelined Arnoldi loop (a step is enqueued before the host reads
    the previous Hessenberg column) reproduces the synchronous loop
    (CPDDG_GMRES_SYNC=1) bit for bit, restarts and kernel profiling included."""
    import torch

    from paper_1909_08734_b200 import api, inputs
    P = api.Problem("sphere", h=0.1, p=3, c=1.0)
    P.decompose(inputs.rcb_partition(P.active_cp, 8), 2, "oras", 4.0, 40.0)
    A = api.DeviceHelmholtz.from_problem(P)
    M = api.SchwarzPreconditioner.from_problem(P)
    b = torch.from_numpy(inputs.rhs_sphere(P.active_cp)).cuda()
    for restart in (50, 5):
        a = api.gmres_solve(A, b, M, 1e-10, 500, restart)
        ap = api.gmres_solve(A, b, M, 1e-10, 500, restart, profile=True)
        monkeypatch.setenv("CPDDG_GMRES_SYNC", "1")
        s = api.gmres_solve(A, b, M, 1e-10, 500, restart)
        monkeypatch.delenv("CPDDG_GMRES_SYNC")
        assert torch.equal(a.u, ap.u) and ap.log.kernel_times["pc_launches"] >= ap.log.iterations
        assert a.log.iterations == s.log.iterations and a.log.converged
        assert np.array_equal(np.asarray(a.log.residuals), np.asarray(s.log.residuals))
        assert torch.equal(a.u, s.u)


@pytest.mark.parametrize("name", ["circle_oras_gmres", "sphere05_oras_gmres", "sphere05_ras_gmres"])
def test_graph_gmres_matches_host_loop(name, monkeypatch):
    """Device-driven cycles (one CUDA graph launch per restart cycle: the
    Arnoldi step's Givens update, convergence and breakdown tests on the
    device, a while-conditional node) reproduce the host-driven loop
    (CPDDG_GMRES_GRAPH=0) bit for bit: residual histories, iteration counts,
    solutions; with restarts and with the profiling stamps."""
    g, cfg, P, A, M, torch = _setup(name)
    from paper_1909_08734_b200 import api
    b = torch.from_numpy(g["b"]).cuda()
    for restart in (50, 7):
        d = api.gmres_solve(A, b, M, 1e-10, 500, restart)
        monkeypatch.setenv("CPDDG_GMRES_GRAPH", "1")  # profiled graph: device timestamps
        dp = api.gmres_solve(A, b, M, 1e-10, 500, restart, profile=True)
        monkeypatch.setenv("CPDDG_GMRES_GRAPH", "0")
        h = api.gmres_solve(A, b, M, 1e-10, 500, restart)
        monkeypatch.delenv("CPDDG_GMRES_GRAPH")
        assert d.log.iterations == h.log.iterations and d.log.converged == h.log.converged
        assert np.array_equal(np.asarray(d.log.residuals), np.asarray(h.log.residuals))
        assert torch.equal(d.u, h.u) and torch.equal(d.u, dp.u)
        assert d.log.final_true_residual == h.log.final_true_residual
        kt = dp.log.kernel_times
        assert kt["pc_launches"] >= dp.log.iterations and kt["pc_seconds"] > 0 and kt["op_seconds"] > 0


@pytest.mark.parametrize("name", ["circle_oras_gmres", "circle_ras_gmres"])
def test_register_mgs_matches_block_mgs(name, monkeypatch):
    """The latency-trimmed single-CTA orthogonalisation (k_mgs_block_reg,
    n <= 4096) reproduces k_mgs_block (CPDDG_MGS=block) bit for bit: residual
    histories and solutions, graph- and host-driven.  (Circle ORAS amplifies
    any roundoff difference to ~1e-7 of the initial residual by the last
    iterations, so bitwise equality is the meaningful check.)"""
    g, cfg, P, A, M, torch = _setup(name)
    from paper_1909_08734_b200 import api
    assert P.n_active <= 4096
    b = torch.from_numpy(g["b"]).cuda()
    monkeypatch.setenv("CPDDG_MGS", "block")
    A_blk = api.DeviceHelmholtz.from_problem(P)  # own Krylov workspace and graph
    for graph in ("1", "0"):
        monkeypatch.setenv("CPDDG_GMRES_GRAPH", graph)
        monkeypatch.delenv("CPDDG_MGS")
        d = api.gmres_solve(A, b, M, 1e-10, 500, 50)
        monkeypatch.setenv("CPDDG_MGS", "block")
        h = api.gmres_solve(A_blk, b, M, 1e-10, 500, 50)
        assert d.log.iterations == h.log.iterations
        assert np.array_equal(np.asarray(d.log.residuals), np.asarray(h.log.residuals))
        assert torch.equal(d.u, h.u)


@pytest.mark.parametrize("name", ["circle_ras_stationary", "sphere10_oras_stationary"])
def test_graph_stationary_matches_host_loop(name, monkeypatch):
    """The stationary iteration as one graph launch (device checks, while
    node) reproduces the host-driven loop bit for bit."""
    g, cfg, P, A, M, torch = _setup(name)
    from paper_1909_08734_b200 import api
    b = torch.from_numpy(g["b"]).cuda()
    for mi in (int(cfg.get("max_iter", 500)), 7, 0):
        d = api.stationary_solve(A, b, M, 1e-10, mi)
        monkeypatch.setenv("CPDDG_GMRES_GRAPH", "0")
        h = api.stationary_solve(A, b, M, 1e-10, mi)
        monkeypatch.delenv("CPDDG_GMRES_GRAPH")
        assert d.log.iterations == h.log.iterations and d.log.converged == h.log.converged
        assert np.array_equal(np.asarray(d.log.residuals), np.asarray(h.log.residuals))
        assert torch.equal(d.u, h.u) and d.log.final_true_residual == h.log.final_true_residual


def test_graph_gmres_short_cycles_and_max_iter(monkeypatch):
    """Cycle and max_iter limits inside the graph loop: max_iter reached in the
    middle of a cycle (not converged), restart 1, and max_iter = 1."""
    g, cfg, P, A, M, torch = _setup("sphere05_oras_gmres")
    from paper_1909_08734_b200 import api
    b = torch.from_numpy(g["b"]).cuda()
    for restart, mi in ((50, 13), (1, 9), (5, 1), (3, 8)):
        d = api.gmres_solve(A, b, M, 1e-10, mi, restart)
        monkeypatch.setenv("CPDDG_GMRES_GRAPH", "0")
        h = api.gmres_solve(A, b, M, 1e-10, mi, restart)
        monkeypatch.delenv("CPDDG_GMRES_GRAPH")
        assert d.log.iterations == h.log.iterations == mi and not d.log.converged
        assert np.array_equal(np.asarray(d.log.residuals), np.asarray(h.log.residuals))
        assert torch.equal(d.u, h.u)


def test_paired_mgs_matches_single_projection_mgs(monkeypatch):
    """The cooperative orthogonalisation takes two projections per grid barrier
    (k_mgs_pair: h_b = V_b.w - h_a (V_b.V_a), the modified Gram-Schmidt
    coefficient with the subtraction moved across the dot product); one
    projection per barrier (CPDDG_MGS=single, k_mgs_reg) gives the same
    iteration count, residual history and solution to rounding, in the
    device-driven cycles and in the host loop, over several restart cycles."""
    import torch

    from paper_1909_08734_b200 import api, inputs
    P = api.Problem("sphere", h=0.05, p=3, c=1.0)
    P.decompose(inputs.rcb_partition(P.active_cp, 64), 2, "oras", 4.0, 40.0)
    A = api.DeviceHelmholtz.from_problem(P)
    M = api.SchwarzPreconditioner.from_problem(P)
    b = torch.from_numpy(inputs.rhs_sphere(P.active_cp)).cuda()
    for graph in ("1", "0"):
        monkeypatch.setenv("CPDDG_GMRES_GRAPH", graph)
        for restart in (50, 7):
            pair = api.gmres_solve(A, b, M, 1e-10, 1000, restart)
            monkeypatch.setenv("CPDDG_MGS", "single")
            single = api.gmres_solve(A, b, M, 1e-10, 1000, restart)
            monkeypatch.delenv("CPDDG_MGS")
            assert pair.log.converged and pair.log.iterations == single.log.iterations
            rp, rs_ = np.asarray(pair.log.residuals), np.asarray(single.log.residuals)
            assert np.max(np.abs(rp - rs_) / rs_[0]) <= 1e-12
            up, us = pair.u.cpu().numpy(), single.u.cpu().numpy()
            assert np.linalg.norm(up - us) <= 1e-11 * np.linalg.norm(us)
            again = api.gmres_solve(A, b, M, 1e-10, 1000, restart)
            assert torch.equal(again.u, pair.u)  # bitwise reproducible
    monkeypatch.delenv("CPDDG_GMRES_GRAPH")


def test_run_solve_pipeline_with_files(tmp_path):
    """run_solve (pipeline.hpp:183-241) fed through a partition file and an rhs
    file, writing the reference's output files."""
    import json

    from paper_1909_08734_b200 import api, inputs, io
    g = np.load(os.path.join(GOLDEN, "circle_oras_gmres.npz"))
    io.write_partition(str(tmp_path / "part.txt"), g["part_in"])
    io.write_rhs(str(tmp_path / "rhs.txt"), g["b"])
    cfg = dict(surface="circle", h=0.0125, p=3, c=1.0, method="oras", mode="gmres", gmres_restart=50,
               rel_tol=1e-10, max_iter=2000, n_overlap=2, n_subdomains=8, alpha=1.0,
               partition_in=str(tmp_path / "part.txt"), rhs="file:" + str(tmp_path / "rhs.txt"),
               partition_out=str(tmp_path / "aligned.txt"), output_dir=str(tmp_path))
    out = api.run_solve(cfg, exact=lambda cp: np.sin(np.arctan2(cp[:, 1], cp[:, 0])) +
                        np.sin(12 * np.arctan2(cp[:, 1], cp[:, 0])))
    assert out["problem"].device_setup and 0 <= out["err_rms"] <= out["err_inf"]
    host = api.run_solve(dict(cfg, device_setup=False, partition_out="", output_dir=""))
    assert not host["problem"].device_setup and host["err_inf"] == -1.0
    assert np.array_equal(out["u"], host["u"]) and np.array_equal(out["part"], host["part"])
    assert out["fallback_anchors"] == host["fallback_anchors"] >= 0
    assert out["log"].converged and abs(out["log"].iterations - int(g["iterations"])) <= 2
    assert np.linalg.norm(out["u"] - g["u"]) <= 1e-8 * np.linalg.norm(g["u"])
    assert np.array_equal(io.read_partition(str(tmp_path / "aligned.txt"), len(g["b"])), g["part_aligned"])
    lines = (tmp_path / "iterations.csv").read_text().splitlines()
    assert lines[0] == "iter,residual_2norm" and len(lines) == out["log"].iterations + 2
    assert (tmp_path / "solution.csv").read_text().startswith("x,y,z,u\n")
    assert (tmp_path / "timings.csv").read_text().splitlines()[-1].startswith("preconditioned_solve,")


def test_streamed_record_and_chain_solves_agree(monkeypatch):
    """Every preconditioner solve path gives the same A_j^-1 (to 1e-12) and the
    same GMRES iteration count, and matches the oracle restatement (SuperLU per
    subdomain) at the usual 1e-9:

    * k_solve_win, the default: windowed, TMA-streamed record solve, RB = 16
      (apply_mode 3) on the balanced schedule (subdomains cut across two SMs,
      state handed over through global memory: bitwise equal to whole
      subdomains per SM, CPDDG_WIN_SPLIT=0); also with RB = 8, with y kept in global memory
      (CPDDG_WIN_GY=1, apply_mode 4: the path for windows larger than shared
      memory), and with a ring so small that every item's data is read from
      HBM (CPDDG_WIN_RING);
    * k_solve_tma (CPDDG_SOLVE=tma, whole y in shared memory, RB = 8) and its
      register-staged fallback when an item would not fit its ring;
    * the register-staged record solve (CPDDG_SOLVE=reg) and the
      substitution-chain solve on reversed U rows (CPDDG_BLOCKINV=0).

    Sphere h = 0.05 cut into 256 RCB parts, so the streamed paths are taken."""
    import torch

    import cpdd_oracle as O
    from paper_1909_08734_b200 import api, inputs
    P = api.Problem("sphere", h=0.05, p=3, c=1.0)
    P.decompose(inputs.rcb_partition(P.active_cp, 256), 2, "oras", 4.0, 40.0)
    A = api.DeviceHelmholtz.from_problem(P)

    def build(**env):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        m = api.SchwarzPreconditioner.from_problem(P)
        for k in env:
            monkeypatch.delenv(k)
        return m

    M = build()
    assert M.stats()["apply_mode"] == 3
    # 256 subdomains on fewer SMs: the balanced schedule cuts subdomains across two SMs
    assert M.stats()["win_cuts"] > 0 and M.stats()["win_bal_efficiency"] >= M.stats()["win_lpt_efficiency"]
    variants = {
        "win_unsplit": (build(CPDDG_WIN_SPLIT="0"), 3),
        "win_rb8": (build(CPDDG_WIN_RB="8"), 3),
        "win_rb8_unsplit": (build(CPDDG_WIN_RB="8", CPDDG_WIN_SPLIT="0"), 3),
        "win_global_y": (build(CPDDG_WIN_GY="1"), 4),
        "win_items_from_hbm": (build(CPDDG_WIN_RING="9216"), 3),
        "tma": (build(CPDDG_SOLVE="tma"), 2),
        "tma_fallback": (build(CPDDG_SOLVE="tma", CPDDG_TMA_RING_LIMIT="1024"), 0),
        "reg": (build(CPDDG_SOLVE="reg"), 0),
        "chain": (build(CPDDG_SOLVE="reg", CPDDG_BLOCKINV="0"), 0),
    }
    for name, (m, mode) in variants.items():
        assert m.stats()["apply_mode"] == mode, name
    x = inputs.uniform_vector(P.n_active, 11)
    xd = torch.from_numpy(x).cuda()
    z = M.apply(xd).cpu().numpy()
    zc = variants["chain"][0].apply(xd).cpu().numpy()
    nz = np.linalg.norm(zc)
    for name, (m, _) in variants.items():
        assert np.linalg.norm(m.apply(xd).cpu().numpy() - zc) <= 1e-12 * nz, name
    assert np.linalg.norm(z - zc) <= 1e-12 * nz
    assert np.array_equal(z, M.apply(xd).cpu().numpy())  # bitwise reproducible
    # the hand-over of a cut subdomain carries exactly the state the unsplit kernel holds
    assert variants["win_unsplit"][0].stats()["win_cuts"] == 0
    assert np.array_equal(z, variants["win_unsplit"][0].apply(xd).cpu().numpy())
    assert np.array_equal(variants["win_rb8"][0].apply(xd).cpu().numpy(),
                          variants["win_rb8_unsplit"][0].apply(xd).cpu().numpy())
    locs = [P.local(j) for j in range(P.n_sub)]
    z_ref = O.schwarz_apply(locs, x)
    assert np.linalg.norm(z - z_ref) <= 1e-9 * np.linalg.norm(z_ref)
    b = torch.from_numpy(inputs.rhs_sphere(P.active_cp)).cuda()
    its = [api.gmres_solve(A, b, m, 1e-10, 1000, 50).log.iterations
           for m in [M] + [v[0] for v in variants.values()]]
    assert len(set(its)) == 1, its
    # kernel shared-memory limits are per kernel: a preconditioner with smaller
    # subdomains built afterwards must not break the earlier, larger one
    Ps = api.Problem("sphere", h=0.1, p=3, c=1.0)
    Ps.decompose(inputs.rcb_partition(Ps.active_cp, 200), 2, "oras", 4.0, 40.0)
    Msmall = api.SchwarzPreconditioner.from_problem(Ps)
    assert Msmall.stats()["max_rows"] < M.stats()["max_rows"]
    assert np.array_equal(M.apply(xd).cpu().numpy(), z)
