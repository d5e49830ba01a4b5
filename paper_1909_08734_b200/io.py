"""On-disk formats on either side of the solve path,
byte-compatible with the reference's writers and readers:

  partition file  read_partition / write_partition   partition.hpp:510-552
  rhs file        read_rhs / write_rhs               pipeline.hpp:103-117 (rhs = file:PATH)
  solution.csv    write_solution                     io.hpp:82-95
  iterations.csv  write_iterations                   io.hpp:97-103
  timings.csv     write_timings                      io.hpp:106-115
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .errors import ConfigError, IoError


def _fmt(v: float) -> str:
    return "%.12e" % v


def write_solution(path: str, x: np.ndarray, u: np.ndarray) -> None:
    """x,y,z,u per active node (io.hpp:82-95); x = lattice positions h*ix."""
    x = np.asarray(x, np.float64)
    if x.shape[0] != np.asarray(u).shape[0]:
        from .errors import InternalError
        raise InternalError(_lib.ERR_INTERNAL, "solution size mismatch")
    d = x.shape[1]
    try:
        with open(path, "w") as fh:
            fh.write("x,y,z,u\n")
            for i in range(x.shape[0]):
                cols = [_fmt(x[i, a] if a < d else 0.0) for a in range(3)]
                fh.write(",".join(cols) + "," + _fmt(u[i]) + "\n")
    except OSError as e:
        raise IoError(_lib.ERR_IO, f"cannot open output file: {path}") from e


def write_iterations(path: str, residuals) -> None:
    """iter,residual_2norm (io.hpp:97-103)."""
    try:
        with open(path, "w") as fh:
            fh.write("iter,residual_2norm\n")
            for n, r in enumerate(residuals):
                fh.write(f"{n},{_fmt(r)}\n")
    except OSError as e:
        raise IoError(_lib.ERR_IO, f"cannot open output file: {path}") from e


def write_timings(path: str, timings, gmres_mode: bool) -> None:
    """phase,seconds (io.hpp:106-115)."""
    try:
        with open(path, "w") as fh:
            fh.write("phase,seconds\n")
            fh.write(f"mesh,{_fmt(timings.mesh)}\n")
            fh.write(f"global_matrix,{_fmt(timings.global_matrix)}\n")
            fh.write(f"local_operators,{_fmt(timings.local_operators)}\n")
            fh.write(("preconditioned_solve," if gmres_mode else "solve,") + _fmt(timings.solve) + "\n")
    except OSError as e:
        raise IoError(_lib.ERR_IO, f"cannot open output file: {path}") from e


def write_partition(path: str, part) -> None:
    """One label per line (partition.hpp:510-515)."""
    try:
        with open(path, "w") as fh:
            fh.write("".join(f"{int(p)}\n" for p in part))
    except OSError as e:
        raise IoError(_lib.ERR_IO, f"cannot open partition file for writing: {path}") from e


def read_partition(path: str, n_active: int) -> np.ndarray:
    """load_partition (partition.hpp:519-552): one integer per line, empty lines
    skipped; count == n_active, labels >= 0 and without gaps."""
    try:
        fh = open(path)
    except OSError as e:
        raise IoError(_lib.ERR_IO, f"cannot open partition file: {path}") from e
    part = []
    with fh:
        for line in fh:
            line = line.rstrip("\n")
            if not line:
                continue
            s = line.lstrip()
            j = 0
            if j < len(s) and s[j] in "+-":
                j += 1
            k = j
            while k < len(s) and s[k].isdigit():
                k += 1
            if k == j or s[k:].strip():
                raise IoError(_lib.ERR_IO, f"malformed partition file line: '{line}'")
            part.append(int(s[:k]))
    if len(part) != n_active:
        raise ConfigError(_lib.ERR_CONFIG, f"partition file has {len(part)} entries but the mesh has "
                                           f"{n_active} active nodes")
    if any(v < 0 for v in part):
        raise ConfigError(_lib.ERR_CONFIG, "partition file contains a negative label")
    present = set(part)
    for q in range(max(part) + 1 if part else 0):
        if q not in present:
            raise ConfigError(_lib.ERR_CONFIG, f"partition labels skip part {q}")
    return np.array(part, np.int32)


def write_rhs(path: str, b) -> None:
    """%.17g per line: round-trips exactly through operator>> (pipeline.hpp:108)."""
    try:
        with open(path, "w") as fh:
            fh.write("".join(f"{v:.17g}\n" for v in b))
    except OSError as e:
        raise IoError(_lib.ERR_IO, f"cannot open rhs file: {path}") from e


def read_rhs(path: str, n_active: int) -> np.ndarray:
    """rhs = file:PATH (pipeline.hpp:103-117): whitespace-separated reals, count == n_active."""
    try:
        text = open(path).read()
    except OSError as e:
        raise IoError(_lib.ERR_IO, f"cannot open rhs file: {path}") from e
    try:
        vals = [float(t) for t in text.split()]
    except ValueError as e:
        raise IoError(_lib.ERR_IO, f"malformed rhs file: {path}") from e
    if len(vals) != n_active:
        raise ConfigError(_lib.ERR_CONFIG, f"rhs file has {len(vals)} values but the mesh has {n_active} "
                                           "active nodes")
    return np.array(vals, np.float64)
