"""The local-system reduction of the device preconditioner (csrc/cuda/pc.cu,
drop_unreferenced) on the host, no GPU: which closure unknowns are removed,
and that removing them leaves the solution of the remaining unknowns unchanged.

Reference facts it rests on: ghost-type / ring closure nodes "are only ever
referenced by their own transmission row" (proj/include/cpdd/transmission.hpp:84-92);
restrict_residual puts zeros in the closure block (:59-63); only owned overlap
slots are scattered back (:66-69)."""
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spl

from paper_1909_08734_b200 import api, inputs


def _restated_mask(L):
    """Fixed point of: a closure unknown whose column holds nothing but its own
    nonzero diagonal, in rows not yet removed, and that no scatter returns."""
    n = L["n_overlap"] + L["n_bc"]
    ptr, col, val = L["ptr"], L["col"], L["val"]
    rows = np.repeat(np.arange(n), np.diff(ptr))
    diag = np.zeros(n)
    np.add.at(diag, rows[rows == col], val[rows == col])
    fixed = np.zeros(n, bool)
    fixed[L["scatter_local"]] = True
    gone = np.zeros(n, bool)
    while True:
        live = ~gone[rows] & (rows != col)
        ref = np.bincount(col[live], minlength=n)
        cand = (ref == 0) & ~gone & ~fixed & (diag != 0) & np.isfinite(diag)
        cand[: L["n_overlap"]] = False
        if not cand.any():
            return gone
        gone |= cand


def test_reduction_matches_the_restatement_and_keeps_the_solution():
    rng = np.random.default_rng(7)
    for surf, kw, ns, no, method in [("sphere", dict(h=0.1, p=3), 16, 2, "oras"),
                                     ("circle", dict(h=0.025, p=3), 6, 2, "oras"),
                                     ("torus", dict(h=0.08, p=3, major_radius=1.0, minor_radius=0.4), 12, 2, "oras"),
                                     ("sphere", dict(h=0.1, p=3), 16, 2, "ras")]:
        P = api.Problem(surf, **kw)
        part = (inputs.sector_partition(P.active_cp, ns) if surf == "circle"
                else inputs.rcb_partition(P.active_cp, ns))
        P.decompose(part, no, method, 4.0, 40.0)
        dropped_total = 0
        for j in range(P.n_sub):
            L = P.local(j)
            n = L["n_overlap"] + L["n_bc"]
            mask = api.unreferenced_unknowns(L)
            assert np.array_equal(mask, _restated_mask(L)), (surf, method, j)
            assert not mask[: L["n_overlap"]].any() and not mask[L["scatter_local"]].any()
            dropped_total += int(mask.sum())
            if j % 5:
                continue
            # the reference's local solve (restrict_residual: closure block zero) on the whole
            # system and on the reduced one agree on every kept unknown
            A = sp.csr_matrix((L["val"], L["col"], L["ptr"]), shape=(n, n)).tocsc()
            b = np.zeros(n)
            b[: L["n_overlap"]] = rng.uniform(-1, 1, L["n_overlap"])
            z = spl.splu(A).solve(b)
            keep = ~mask
            zr = spl.splu(A[keep][:, keep].tocsc()).solve(b[keep])
            assert np.linalg.norm(z[keep] - zr) <= 1e-11 * np.linalg.norm(z[keep])
            # removed rows referred to nothing that was kept out of their own row only:
            # no kept row refers to a removed column
            assert A[keep][:, mask].nnz == 0
        if method == "oras":
            assert dropped_total > 0  # the Robin ring and the ghost-type closure nodes
