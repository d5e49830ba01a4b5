"""The local solver's robustness, as the reference's DirectSolver has it
(proj/include/cpdd/direct.hpp:36-68: Eigen SparseLU with partial pivoting;
singular systems raise DivergenceError):

* a local system whose no-pivot device LU breaks down (zero pivots) is
  refactored on the host with partial pivoting and solved exactly;
* pivoting every subdomain (CPDDG_PIVOT=all) gives the same preconditioner
  as the no-pivot device factors;
* a singular local system raises DivergenceError("singular factorization");
* the local-vector window of k_solve_win falls back to HBM when it does not
  fit shared memory, and any subdomain size runs (round 1 capped it at
  25,600 rows)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _one_subdomain(A):
    """A single subdomain covering every unknown: M = A^-1."""
    import scipy.sparse as sp
    A = sp.csr_matrix(A)
    n = A.shape[0]
    idx = np.arange(n, dtype=np.int32)
    return dict(n_overlap=n, n_bc=0, overlap=idx, scatter_local=idx, scatter_global=idx,
                ptr=A.indptr.astype(np.int64), col=A.indices.astype(np.int32), val=A.data.astype(np.float64))


def _needs_pivoting(n=400, seed=3):
    """Diagonally dominant banded matrix with row pairs (2i, 2i+1) swapped:
    nonsingular, well conditioned, and with zero diagonal entries."""
    rng = np.random.default_rng(seed)
    A = np.zeros((n, n))
    for i in range(n):
        for j in range(max(0, i - 3), min(n, i + 4)):
            A[i, j] = rng.uniform(-1, 1)
        A[i, i] = 8.0
    P = np.arange(n)
    P[0::2], P[1::2] = np.arange(1, n, 2), np.arange(0, n, 2)
    A = A[P]
    A[np.abs(A) < 1e-300] = 0.0
    for i in range(n):  # zero the diagonal where the swap left a band entry there
        A[i, i] = 0.0
    return A


def test_zero_pivot_system_is_pivoted_and_solved_exactly():
    import torch

    from paper_1909_08734_b200 import api
    A = _needs_pivoting()
    assert np.all(np.diag(A) == 0.0) and np.linalg.cond(A) < 1e3
    M = api.SchwarzPreconditioner.from_locals(A.shape[0], [_one_subdomain(A)])
    st = M.stats()
    assert st["n_pivoted"] == 1 and st["max_probe_residual"] <= 1e-12
    x = np.random.default_rng(5).uniform(-1, 1, A.shape[0])
    z = M.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    z_ref = np.linalg.solve(A, x)
    assert np.linalg.norm(z - z_ref) <= 1e-12 * np.linalg.norm(z_ref)


def test_singular_local_system_raises_divergence():
    from paper_1909_08734_b200 import api, errors
    A = _needs_pivoting()
    A[7, :] = 0.0  # a zero row: singular for any pivoting
    with pytest.raises(errors.DivergenceError, match="singular factorization"):
        api.SchwarzPreconditioner.from_locals(A.shape[0], [_one_subdomain(A)])


def test_pivoting_every_subdomain_matches_the_device_factors(monkeypatch):
    import torch

    from paper_1909_08734_b200 import api, inputs
    P = api.Problem("sphere", h=0.05, p=3, c=1.0)
    P.decompose(inputs.rcb_partition(P.active_cp, 64), 2, "oras", 4.0, 40.0)
    A = api.DeviceHelmholtz.from_problem(P)
    M = api.SchwarzPreconditioner.from_problem(P)
    monkeypatch.setenv("CPDDG_PIVOT", "all")
    Mp = api.SchwarzPreconditioner.from_problem(P)
    assert M.stats()["n_pivoted"] == 0 and Mp.stats()["n_pivoted"] == 64
    assert Mp.stats()["max_probe_residual"] <= 1e-12
    x = torch.from_numpy(inputs.uniform_vector(P.n_active, 11)).cuda()
    z, zp = M.apply(x).cpu().numpy(), Mp.apply(x).cpu().numpy()
    assert np.linalg.norm(z - zp) <= 1e-11 * np.linalg.norm(z)
    b = torch.from_numpy(inputs.rhs_sphere(P.active_cp)).cuda()
    r, rp = (api.gmres_solve(A, b, m, 1e-10, 1000, 50) for m in (M, Mp))
    assert r.log.iterations == rp.log.iterations
    assert np.linalg.norm(r.u.cpu().numpy() - rp.u.cpu().numpy()) <= 1e-9 * np.linalg.norm(r.u.cpu().numpy())


def test_large_subdomains_run_with_the_window_in_hbm(monkeypatch):
    """Sphere h = 0.025 in 4 subdomains (local systems of ~15k rows): the
    default shared-memory window, the same solve with the window forced into
    HBM (the path for subdomains whose envelope rows outgrow shared memory),
    and the oracle restatement agree."""
    import torch

    import cpdd_oracle as O
    from paper_1909_08734_b200 import api, inputs
    P = api.Problem("sphere", h=0.025, p=3, c=1.0)
    P.decompose(inputs.rcb_partition(P.active_cp, 4), 2, "oras", 4.0, 40.0)
    M = api.SchwarzPreconditioner.from_problem(P)
    monkeypatch.setenv("CPDDG_WIN_GY", "1")
    Mg = api.SchwarzPreconditioner.from_problem(P)
    assert M.stats()["apply_mode"] == 3 and Mg.stats()["apply_mode"] == 4
    assert M.stats()["max_rows"] > 12000
    x = inputs.uniform_vector(P.n_active, 11)
    xd = torch.from_numpy(x).cuda()
    z, zg = M.apply(xd).cpu().numpy(), Mg.apply(xd).cpu().numpy()
    assert np.linalg.norm(z - zg) <= 1e-12 * np.linalg.norm(z)
    locs = [P.local(j) for j in range(P.n_sub)]
    z_ref = O.schwarz_apply(locs, x)
    assert np.linalg.norm(z - z_ref) <= 1e-9 * np.linalg.norm(z_ref)


def test_unreferenced_closure_unknowns_are_dropped(monkeypatch):
    """ORAS closures hold ring / ghost-type unknowns that only their own
    transmission row refers to (transmission.hpp:84-92) and that are never
    scattered back (:66-69): the device path removes them before the analysis.
    The reduced preconditioner equals the whole one (CPDDG_DROP=0) and the
    oracle restatement; RAS closures (unit rows) reduce as before; a hand-made
    chain of such unknowns is removed to the fixed point."""
    import torch

    import cpdd_oracle as O
    from paper_1909_08734_b200 import api, inputs
    P = api.Problem("sphere", h=0.05, p=3, c=1.0)
    P.decompose(inputs.rcb_partition(P.active_cp, 64), 2, "oras", 4.0, 40.0)
    A = api.DeviceHelmholtz.from_problem(P)
    M = api.SchwarzPreconditioner.from_problem(P)
    monkeypatch.setenv("CPDDG_DROP", "0")
    Mw = api.SchwarzPreconditioner.from_problem(P)
    monkeypatch.delenv("CPDDG_DROP")
    st, sw = M.stats(), Mw.stats()
    assert sw["n_dropped"] == 0 and st["n_dropped"] > 0
    assert st["n_rows_total"] == sw["n_rows_total"] - st["n_dropped"]
    assert st["n_dropped"] >= 0.2 * sw["n_rows_total"]       # ~26 % of the unknowns at this size
    assert st["factor_entries"] <= 0.8 * sw["factor_entries"]  # and ~30 % of the streamed entries
    x = inputs.uniform_vector(P.n_active, 11)
    xd = torch.from_numpy(x).cuda()
    z, zw = M.apply(xd).cpu().numpy(), Mw.apply(xd).cpu().numpy()
    assert np.linalg.norm(z - zw) <= 1e-12 * np.linalg.norm(zw)
    locs = [P.local(j) for j in range(P.n_sub)]
    z_ref = O.schwarz_apply(locs, x)
    assert np.linalg.norm(z - z_ref) <= 1e-9 * np.linalg.norm(z_ref)
    b = torch.from_numpy(inputs.rhs_sphere(P.active_cp)).cuda()
    r, rw = (api.gmres_solve(A, b, m, 1e-10, 1000, 50) for m in (M, Mw))
    assert r.log.iterations == rw.log.iterations
    assert np.linalg.norm(r.u.cpu().numpy() - rw.u.cpu().numpy()) <= 1e-9 * np.linalg.norm(rw.u.cpu().numpy())

    # RAS: the closure rows are unit rows; ghost-type ones drop, the rest is the Dirichlet reduction
    P.decompose(inputs.rcb_partition(P.active_cp, 64), 2, "ras")
    Mr = api.SchwarzPreconditioner.from_problem(P)
    assert Mr.stats()["n_reduced"] == 64
    zr = Mr.apply(xd).cpu().numpy()
    zr_ref = O.schwarz_apply([P.local(j) for j in range(P.n_sub)], x)
    assert np.linalg.norm(zr - zr_ref) <= 1e-9 * np.linalg.norm(zr_ref)

    # a chain: unknown 5 is referenced only by row 6, unknown 6 only by its own row
    import scipy.sparse as sp
    rng = np.random.default_rng(5)
    n = 7
    B = np.zeros((n, n))
    B[:5, :5] = rng.uniform(-1, 1, (5, 5)) + 6 * np.eye(5)
    B[5, 5], B[5, :3] = 2.0, (0.5, -0.25, 0.125)
    B[6, 6], B[6, 5], B[6, 1] = 4.0, 1.0, -1.0
    Bs = sp.csr_matrix(B)
    idx = np.arange(5, dtype=np.int32)
    loc = dict(n_overlap=5, n_bc=2, overlap=idx, scatter_local=idx, scatter_global=idx,
               ptr=Bs.indptr.astype(np.int64), col=Bs.indices.astype(np.int32), val=Bs.data.astype(np.float64))
    Mc = api.SchwarzPreconditioner.from_locals(5, [loc])
    assert Mc.stats()["n_dropped"] == 2 and Mc.stats()["n_rows_total"] == 5
    rhs = rng.uniform(-1, 1, 5)
    want = np.linalg.solve(B, np.concatenate([rhs, np.zeros(2)]))[:5]
    got = Mc.apply(torch.from_numpy(rhs).cuda()).cpu().numpy()
    assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)


def test_unsorted_rows_and_duplicate_entries():
    """cpddg_pc_create accepts any CSR a LocalOperator could hold: columns in any
    order within a row and duplicate (row, column) entries, which are summed
    (SparseOperator rows are sorted and merged, sparse.hpp:35-46, but the ABI
    does not rely on it).  The pattern analysis takes its general path, the
    reduction still finds the unknown nothing depends on, and the solve equals
    the dense solve."""
    import scipy.sparse as sp
    import torch

    from paper_1909_08734_b200 import api
    rng = np.random.default_rng(11)
    n_ov, n_bc = 300, 3
    n = n_ov + n_bc
    B = sp.random(n, n, density=0.03, random_state=3, format="lil")
    B.setdiag(8.0 + rng.uniform(0, 1, n))
    B = B.toarray()
    B[:, n - 1] = 0.0          # the last closure unknown: only its own row refers to it
    B[n - 1, n - 1] = 3.0
    B[n - 1, :5] = rng.uniform(-1, 1, 5)
    B[n_ov, n_ov + 1] = 0.25   # the other two closure unknowns stay (referenced from overlap rows)
    B[3, n_ov] = -0.5
    B[7, n_ov + 1] = 0.75
    ptr, col, val = [0], [], []
    for r in range(n):
        cs = np.flatnonzero(B[r])
        cs = cs[rng.permutation(cs.size)]            # unsorted
        for c in cs:
            if rng.uniform() < 0.3:                   # a duplicate entry: two halves
                col += [c, c]
                val += [0.5 * B[r, c], 0.5 * B[r, c]]
            else:
                col.append(c)
                val.append(B[r, c])
        ptr.append(len(col))
    idx = np.arange(n_ov, dtype=np.int32)
    loc = dict(n_overlap=n_ov, n_bc=n_bc, overlap=idx, scatter_local=idx, scatter_global=idx,
               ptr=np.asarray(ptr, np.int64), col=np.asarray(col, np.int32), val=np.asarray(val, np.float64))
    mask = api.unreferenced_unknowns(loc)
    assert mask.sum() == 1 and mask[n - 1]
    M = api.SchwarzPreconditioner.from_locals(n_ov, [loc])
    assert M.stats()["n_dropped"] == 1 and M.stats()["n_rows_total"] == n - 1
    rhs = rng.uniform(-1, 1, n_ov)
    want = np.linalg.solve(B, np.concatenate([rhs, np.zeros(n_bc)]))[:n_ov]
    got = M.apply(torch.from_numpy(rhs).cuda()).cpu().numpy()
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
