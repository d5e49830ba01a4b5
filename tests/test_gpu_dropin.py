"""The drop-in demonstration (oracle/dropin_demo.cpp): an unmodified reference
pipeline whose hot path is switched to the device through include/cpddg.hpp,
run against the reference's own CPU solve in the same process."""
import json
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
EXE = os.path.join(ROOT, "oracle", "_ref", "dropin_demo")


@pytest.mark.skipif(not os.path.exists(EXE), reason="oracle/_ref/dropin_demo not built (needs /root/reference)")
def test_dropin_matches_reference_solve():
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    rows = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    solves = [x for x in rows if "ref_iters" in x]
    assert len(solves) == 2
    for x in solves:
        assert x["ref_conv"] == 1 and x["dev_conv"] == 1
        assert abs(x["ref_iters"] - x["dev_iters"]) <= 2, x
        assert x["u_rel_diff"] <= 1e-8, x
        assert x["op_rel_diff"] <= 1e-12, x
    errs = [x for x in rows if x["case"].endswith("_error")]
    assert errs and all(x["raised"] == 1 for x in errs)
