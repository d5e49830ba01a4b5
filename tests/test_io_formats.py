"""On-disk formats byte-identical to the reference's
writers, and the readers' error behaviour (partition.hpp:519-552,
pipeline.hpp:103-117)."""
import os

import numpy as np
import pytest

from conftest import needs_ref

from paper_1909_08734_b200 import api, errors, inputs, io


@needs_ref
def test_writers_byte_identical_to_reference(tmp_path):
    import ref
    R = ref.RefProblem(dict(surface="sphere", h=0.1, p=3, method="oras", n_overlap=2, n_subdomains=4), workers=2)
    B = R.band()
    na = R.n_active
    u = inputs.uniform_vector(na, 3)
    res = np.abs(inputs.uniform_vector(17, 4)) * 1e-3
    t4 = np.array([1.25, 0.5, 2.0, 0.125])
    rdir, odir = tmp_path / "ref", tmp_path / "ours"
    rdir.mkdir()
    odir.mkdir()
    ref.write_outputs(R, str(rdir), u, res, t4, True)
    io.write_solution(str(odir / "solution.csv"), B["x"][:na], u)
    io.write_iterations(str(odir / "iterations.csv"), res)
    io.write_timings(str(odir / "timings.csv"), api.PhaseTimings(*t4), True)
    for f in ("solution.csv", "iterations.csv", "timings.csv"):
        assert (rdir / f).read_bytes() == (odir / f).read_bytes(), f


def test_partition_and_rhs_round_trip(tmp_path):
    P = api.Problem("circle", h=0.05, p=3)
    part = inputs.sector_partition(P.active_cp, 4)
    io.write_partition(str(tmp_path / "p.txt"), part)
    assert np.array_equal(io.read_partition(str(tmp_path / "p.txt"), P.n_active), part)
    b = inputs.rhs_circle(P.active_cp)
    io.write_rhs(str(tmp_path / "b.txt"), b)
    assert np.array_equal(io.read_rhs(str(tmp_path / "b.txt"), P.n_active), b)  # %.17g round trip


def test_reader_errors(tmp_path):
    p = tmp_path / "p.txt"
    p.write_text("0\n1\nx\n")
    with pytest.raises(errors.IoError, match="malformed"):
        io.read_partition(str(p), 3)
    p.write_text("0\n2\n")
    with pytest.raises(errors.ConfigError, match="skip part 1"):
        io.read_partition(str(p), 2)
    p.write_text("0\n1\n")
    with pytest.raises(errors.ConfigError, match="entries but the mesh has"):
        io.read_partition(str(p), 3)
    with pytest.raises(errors.IoError):
        io.read_partition(str(tmp_path / "missing.txt"), 3)
    with pytest.raises(errors.ConfigError, match="values but the mesh has"):
        io.read_rhs(str(p), 5)
