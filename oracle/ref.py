"""ORACLE TEST INFRASTRUCTURE -- ctypes wrapper of oracle/_ref/libcpdd_ref.so.

libcpdd_ref.so is the UNMODIFIED reference library (/root/reference/proj/include,
header-only C++20) compiled against the in-repo Eigen/GTest shims by
oracle/Makefile, plus the handle-based driver oracle/ref_driver.cpp that
replaces the CLI11 front end (proj/tools/cpm.cpp).  Only tests/, the smoke
check and bench.py's reference / cpu_baseline legs may use this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libcpdd_ref.so")
_lib = None

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"{LIB_PATH} missing: run `make -C oracle` (needs /root/reference)")
        L = C.CDLL(LIB_PATH)
        L.cref_create.restype = C.c_void_p
        L.cref_create.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_int]
        L.cref_destroy.argtypes = [C.c_void_p]
        L.cref_last_error.argtypes = [C.c_void_p, C.c_char_p, C.c_int]
        L.cref_sizes.argtypes = [C.c_void_p] + [C.POINTER(C.c_int)] * 4 + [C.POINTER(C.c_double)]
        L.cref_phase.restype = C.c_double
        L.cref_phase.argtypes = [C.c_void_p, C.c_int]
        L.cref_band.argtypes = [C.c_void_p, _i32p, _f64p, _f64p, _f64p, _f64p]
        L.cref_nnz.restype = C.c_longlong
        L.cref_nnz.argtypes = [C.c_void_p, C.c_int]
        L.cref_csr.argtypes = [C.c_void_p, C.c_int, _i64p, _i32p, _f64p]
        L.cref_rhs.argtypes = [C.c_void_p, _f64p]
        L.cref_apply_A.argtypes = [C.c_void_p, _f64p, _f64p]
        L.cref_decompose.argtypes = [C.c_void_p, C.c_void_p, _i32p, C.POINTER(C.c_int), C.c_int]
        L.cref_decompose_time.restype = C.c_double
        L.cref_decompose_time.argtypes = [C.c_void_p, C.c_int]
        L.cref_n_sub.argtypes = [C.c_void_p]
        L.cref_sub_counts.argtypes = [C.c_void_p, C.c_int, _i32p]
        L.cref_sub_sets.argtypes = [C.c_void_p, C.c_int, _i32p, _i32p, _i32p, _i32p, _i32p, _f64p]
        L.cref_local_sizes.argtypes = [C.c_void_p, C.c_int, _i64p]
        L.cref_local.argtypes = [C.c_void_p, C.c_int, _i64p, _i32p, _f64p, _i32p, _i32p]
        L.cref_pc_apply.argtypes = [C.c_void_p, _f64p, _f64p]
        L.cref_solve.argtypes = [C.c_void_p, C.c_void_p, _f64p, _f64p, C.c_int,
                                 C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                 C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.cref_run_solve.argtypes = [C.c_void_p, _f64p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                     C.POINTER(C.c_double), _f64p]
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def ini_text(cfg: dict) -> str:
    return "".join(f"{k} = {v}\n" for k, v in cfg.items())


@dataclass
class SubdomainSets:
    disjoint: np.ndarray
    overlap: np.ndarray
    final_layer: np.ndarray
    ghosts: np.ndarray
    bc_int: np.ndarray   # |bc| x (D+4): ix..., global_active, is_ghost_type, cross, fallback
    bc_real: np.ndarray  # |bc| x (4D+1): x, cp, cp_local, conormal, dq
    fallback_count: int
    n_lambda: int


class RefProblem:
    """The reference's BuiltProblem plus the run_solve steps, one call each."""

    def __init__(self, cfg: dict, workers: int = 0):
        L = lib()
        err = C.create_string_buffer(4096)
        self._h = L.cref_create(ini_text(cfg).encode(), int(workers), err, 4096)
        if not self._h:
            msg = err.value.decode()
            code = 2 if msg.startswith("ConfigError") else 4 if msg.startswith("IoError") else 1
            raise RefError(code, msg)
        d, na, ng, p = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        h = C.c_double()
        self._check(L.cref_sizes(self._h, C.byref(d), C.byref(na), C.byref(ng), C.byref(p), C.byref(h)))
        self.dim, self.n_active, self.n_ghost, self.p, self.h = d.value, na.value, ng.value, p.value, h.value
        self.cfg = dict(cfg)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().cref_destroy(self._h)
            self._h = None

    def _check(self, rc: int):
        if rc != 0:
            buf = C.create_string_buffer(4096)
            lib().cref_last_error(self._h, buf, 4096)
            raise RefError(rc, buf.value.decode())

    def phase(self, which: int) -> float:
        return lib().cref_phase(self._h, which)

    def band(self):
        nb, D = self.n_active + self.n_ghost, self.dim
        ix = np.zeros(nb * D, np.int32)
        x, cp, nrm = (np.zeros(nb * D) for _ in range(3))
        dist = np.zeros(nb)
        self._check(lib().cref_band(self._h, ix, x, cp, nrm, dist))
        return dict(ix=ix.reshape(nb, D), x=x.reshape(nb, D), cp=cp.reshape(nb, D),
                    normal=nrm.reshape(nb, D), dist=dist)

    def csr(self, which: str):
        w = {"E": 0, "A": 1}[which]
        nnz = lib().cref_nnz(self._h, w)
        nrows = self.n_active + (self.n_ghost if which == "E" else 0)
        ptr = np.zeros(nrows + 1, np.int64)
        col = np.zeros(nnz, np.int32)
        val = np.zeros(nnz)
        self._check(lib().cref_csr(self._h, w, ptr, col, val))
        return ptr, col, val

    def rhs(self) -> np.ndarray:
        b = np.zeros(self.n_active)
        self._check(lib().cref_rhs(self._h, b))
        return b

    def apply_A(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(self.n_active)
        self._check(lib().cref_apply_A(self._h, x, y))
        return y

    def decompose(self, part=None, factor: bool = True):
        out = np.zeros(self.n_active, np.int32)
        moves = C.c_int()
        if part is not None:
            part = np.ascontiguousarray(part, np.int32)
            ptr = part.ctypes.data_as(C.c_void_p)
        else:
            ptr = None
        self._check(lib().cref_decompose(self._h, ptr, out, C.byref(moves), int(factor)))
        self.n_sub = lib().cref_n_sub(self._h)
        self.decompose_times = (lib().cref_decompose_time(self._h, 0), lib().cref_decompose_time(self._h, 1))
        return out, moves.value

    def subdomain(self, j: int) -> SubdomainSets:
        D = self.dim
        cnt = np.zeros(8, np.int32)
        self._check(lib().cref_sub_counts(self._h, j, cnt))
        arrs = [np.zeros(max(int(c), 1), np.int32) for c in cnt[:4]]
        nbc = int(cnt[4])
        bi = np.zeros(max(nbc, 1) * (D + 4), np.int32)
        br = np.zeros(max(nbc, 1) * (4 * D + 1))
        self._check(lib().cref_sub_sets(self._h, j, *arrs, bi, br))
        arrs = [a[: int(c)] for a, c in zip(arrs, cnt[:4])]
        return SubdomainSets(*arrs, bi[: nbc * (D + 4)].reshape(nbc, D + 4),
                             br[: nbc * (4 * D + 1)].reshape(nbc, 4 * D + 1), int(cnt[5]), int(cnt[6]))

    def local(self, j: int):
        s = np.zeros(4, np.int64)
        self._check(lib().cref_local_sizes(self._h, j, s))
        n_ov, n_bc, nnz, nsc = (int(v) for v in s)
        ptr = np.zeros(n_ov + n_bc + 1, np.int64)
        col = np.zeros(max(nnz, 1), np.int32)
        val = np.zeros(max(nnz, 1))
        scl = np.zeros(max(nsc, 1), np.int32)
        scg = np.zeros(max(nsc, 1), np.int32)
        self._check(lib().cref_local(self._h, j, ptr, col, val, scl, scg))
        return dict(n_overlap=n_ov, n_bc=n_bc, ptr=ptr, col=col[:nnz], val=val[:nnz],
                    scatter_local=scl[:nsc], scatter_global=scg[:nsc])

    def pc_apply(self, r: np.ndarray) -> np.ndarray:
        r = np.ascontiguousarray(r, np.float64)
        z = np.zeros(self.n_active)
        self._check(lib().cref_pc_apply(self._h, r, z))
        return z

    def solve(self, b=None, cap: int = 100000):
        u = np.zeros(self.n_active)
        res = np.zeros(cap)
        nres, iters, conv = C.c_int(), C.c_int(), C.c_int()
        ftrue, secs = C.c_double(), C.c_double()
        bp = None
        if b is not None:
            b = np.ascontiguousarray(b, np.float64)
            bp = b.ctypes.data_as(C.c_void_p)
        self._check(lib().cref_solve(self._h, bp, u, res, cap, C.byref(nres), C.byref(iters),
                                     C.byref(conv), C.byref(ftrue), C.byref(secs)))
        return dict(u=u, residuals=res[: min(cap, nres.value)].copy(), iterations=iters.value,
                    converged=bool(conv.value), final_true_residual=ftrue.value, seconds=secs.value)

    def run_solve(self):
        u = np.zeros(self.n_active)
        iters, conv = C.c_int(), C.c_int()
        frel = C.c_double()
        t = np.zeros(4)
        self._check(lib().cref_run_solve(self._h, u, C.byref(iters), C.byref(conv), C.byref(frel), t))
        return dict(u=u, iterations=iters.value, converged=bool(conv.value),
                    final_relative_residual=frel.value,
                    timings=dict(mesh=t[0], global_matrix=t[1], local_operators=t[2], solve=t[3]))


def _setup_extra(L):
    if getattr(L, "_extra", False):
        return
    PP = C.POINTER(C.c_void_p)
    L.cref_set_locals.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.cref_solve_capped.argtypes = [C.c_void_p, _f64p, C.c_int, C.c_double, C.POINTER(C.c_int),
                                    C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L._extra = True


def set_locals(P: RefProblem, locals_: list):
    """Install LocalOperators (reference struct) from field arrays and factor
    them with the reference DirectSolver on the reference ThreadPool."""
    L = lib()
    _setup_extra(L)
    n = len(locals_)
    keep = []

    def arr(ctype, items):
        a = (ctype * n)(*items)
        keep.append(a)
        return a

    cols = []
    for d in locals_:
        cols.append([np.ascontiguousarray(d["overlap"], np.int32), np.ascontiguousarray(d["scatter_local"], np.int32),
                     np.ascontiguousarray(d["scatter_global"], np.int32), np.ascontiguousarray(d["ptr"], np.int64),
                     np.ascontiguousarray(d["col"], np.int32), np.ascontiguousarray(d["val"], np.float64)])
    keep.append(cols)
    vp = C.c_void_p
    rc = L.cref_set_locals(P._h, n, arr(C.c_int, [int(d["n_overlap"]) for d in locals_]),
                           arr(C.c_int, [int(d["n_bc"]) for d in locals_]),
                           arr(vp, [c[0].ctypes.data for c in cols]),
                           arr(C.c_int, [int(c[1].size) for c in cols]),
                           arr(vp, [c[1].ctypes.data for c in cols]), arr(vp, [c[2].ctypes.data for c in cols]),
                           arr(vp, [c[3].ctypes.data for c in cols]), arr(vp, [c[4].ctypes.data for c in cols]),
                           arr(vp, [c[5].ctypes.data for c in cols]))
    P._check(rc)
    P.locals_seconds = L.cref_decompose_time(P._h, 1)


def solve_capped(P: RefProblem, b, max_iter: int, rel_tol: float):
    L = lib()
    _setup_extra(L)
    it, secs, last = C.c_int(), C.c_double(), C.c_double()
    b = np.ascontiguousarray(b, np.float64)
    P._check(L.cref_solve_capped(P._h, b, int(max_iter), float(rel_tol), C.byref(it), C.byref(secs), C.byref(last)))
    return dict(iterations=it.value, seconds=secs.value, last_residual=last.value)


def write_outputs(P: RefProblem, directory: str, u, residuals, t4, gmres_mode: bool):
    L = lib()
    L.cref_write_outputs.argtypes = [C.c_void_p, C.c_char_p, _f64p, _f64p, C.c_int, _f64p, C.c_int]
    u = np.ascontiguousarray(u, np.float64)
    res = np.ascontiguousarray(residuals, np.float64)
    P._check(L.cref_write_outputs(P._h, directory.encode(), u, res, int(res.size),
                                  np.ascontiguousarray(t4, np.float64), int(gmres_mode)))
