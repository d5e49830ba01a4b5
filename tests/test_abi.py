"""The C-ABI library loads and exports every symbol include/cpddg.h declares
(CPU-only: no compute calls)."""
import os
import re

from conftest import ROOT


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "cpddg.h")).read()
    return sorted(set(re.findall(r"\b(cpddg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_1909_08734_b200 import _lib
    assert os.path.exists(_lib.LIB_PATH), "build with __graft_entry__.build()"
    L = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    # the Python binding covers the whole header
    assert set(syms) <= set(_lib.EXPORTED_SYMBOLS)


def test_library_targets_sm100a_only():
    import subprocess

    from paper_1909_08734_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_error_codes_and_messages():
    from paper_1909_08734_b200 import api, errors
    import pytest
    with pytest.raises(errors.ConfigError):
        api.Problem("circle", h=-1.0)
    with pytest.raises(errors.ConfigError):
        api.Problem("sphere", h=0.1, p=9)
    with pytest.raises(errors.ConfigError):
        api.Problem("torus", h=0.1, major_radius=0.3, minor_radius=0.4)
    with pytest.raises(errors.IoError):
        api.Problem("obj", h=0.1, obj_path="/nonexistent/mesh.obj")
    assert api.lib().cpddg_version().decode().startswith("cpddg")
