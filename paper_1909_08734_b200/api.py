"""Python host layer over the C ABI (include/cpddg.h).

Mirrors the reference's own operator / partition / solver interface
(proj/include/cpdd/*.hpp) with the same names, argument meaning and error
behaviour, so the parity tests read like the reference's tests:

  reference (C++)                              here
  ------------------------------------------   -------------------------------------
  build_problem (pipeline.hpp:155-168)         Problem(...)
  load_partition + align_interfaces +          Problem.decompose(part, ...)
    build_subdomains + assemble_local
    (pipeline.hpp:186-216)
  SparseOperator::apply on A (sparse.hpp:65)   DeviceHelmholtz.apply(x)
  SchwarzPreconditioner::apply (solve.hpp:69)  SchwarzPreconditioner.apply(r)
  stationary_solve (solve.hpp:95-123)          stationary_solve(A, b, M, rel_tol, max_iter)
  gmres_solve (solve.hpp:128-214)              gmres_solve(A, b, M, rel_tol, max_iter, restart)
  IterationLog / SolveResult (solve.hpp:49-60) IterationLog / SolveResult
  run_solve (pipeline.hpp:183-241)             run_solve(cfg)

Device vectors are torch CUDA tensors (float64); torch is plumbing for device
memory and streams only -- every FLOP of the solve path runs in the sm_100a
kernels of lib/libcpddg.so.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, lib

SURFACES = {"circle": 0, "sphere": 1, "torus": 2, "obj": 3, "trimesh": 3}
METHODS = {"ras": 0, "oras": 1}


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the cpddg solve path needs a CUDA device (no CPU fallback)")
    return torch


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def _stream():
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


# ---------------------------------------------------------------- setup

class Problem:
    """Band, E and A of one configuration (BuiltProblem, pipeline.hpp:73-84),
    plus the decomposition once `decompose` ran.  Bit-exact with the
    reference; device_setup=True builds the band / closest points and the
    alignment / subdomain sets on the GPU (bit-identical to the host path)."""

    def __init__(self, surface: str = "sphere", h: float = 0.05, p: int = 3, c: float = 1.0,
                 radius: float = 1.0, major_radius: float = 2.0 / 3.0, minor_radius: float = 1.0 / 3.0,
                 obj_path: str | None = None, tube_radius: float = 0.0, workers: int = 0,
                 device_setup: bool = False):
        if surface not in SURFACES:
            from .errors import ConfigError
            raise ConfigError(_lib.ERR_CONFIG, f"unknown surface '{surface}'")
        self.surface = surface
        self.dim = 2 if surface == "circle" else 3
        self._obj = obj_path.encode() if obj_path else None
        d = _lib.cpddg_problem_desc(dim=self.dim, surface=SURFACES[surface], radius=radius,
                                    major_radius=major_radius, minor_radius=minor_radius,
                                    obj_path=self._obj, h=h, p=p, tube_radius=tube_radius, c=c,
                                    workers=workers, device_setup=int(bool(device_setup)))
        self.device_setup = bool(device_setup)
        self._h = C.c_void_p()
        self._destroy = lib().cpddg_setup_destroy
        t0 = time.perf_counter()
        check(lib().cpddg_setup_create(C.byref(d), C.byref(self._h)))
        self.timings = {"mesh_and_global_matrix": time.perf_counter() - t0}
        na, ng = C.c_int(), C.c_int()
        ne, nA = C.c_int64(), C.c_int64()
        check(lib().cpddg_setup_sizes(self._h, C.byref(na), C.byref(ng), C.byref(ne), C.byref(nA)))
        self.n_active, self.n_ghost = na.value, ng.value
        self.nnz_E, self.nnz_A = ne.value, nA.value
        self.h, self.p, self.c = h, p, c
        self.n_sub = 0
        self._band = None

    def __del__(self):
        h = getattr(self, "_h", None)
        destroy = getattr(self, "_destroy", None)
        if h is not None and h.value and destroy is not None:
            destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def band(self) -> dict:
        if self._band is None:
            nb, D = self.n_active + self.n_ghost, self.dim
            ix = np.zeros(nb * D, np.int32)
            cp, nrm = np.zeros(nb * D), np.zeros(nb * D)
            dist = np.zeros(nb)
            check(lib().cpddg_setup_band(self._h, ix, cp, nrm, dist))
            self._band = dict(ix=ix.reshape(nb, D), cp=cp.reshape(nb, D), normal=nrm.reshape(nb, D),
                              dist=dist)
        return self._band

    @property
    def active_cp(self) -> np.ndarray:
        return self.band()["cp"][: self.n_active]

    def csr(self, which: str):
        w = {"E": 0, "A": 1}[which]
        rows = self.n_active + (self.n_ghost if which == "E" else 0)
        nnz = self.nnz_E if which == "E" else self.nnz_A
        ptr, col, val = np.zeros(rows + 1, np.int64), np.zeros(nnz, np.int32), np.zeros(nnz)
        check(lib().cpddg_setup_csr(self._h, w, ptr, col, val))
        return ptr, col, val

    def decompose(self, part, n_overlap: int, method: str = "oras", alpha: float = 1.0,
                  alpha_cross: float = -1.0):
        """Partition -> align_interfaces -> build_subdomains -> assemble_local."""
        part = np.ascontiguousarray(part, np.int32)
        out = np.zeros(self.n_active, np.int32)
        moves = C.c_int()
        t0 = time.perf_counter()
        check(lib().cpddg_setup_decompose(self._h, part, int(part.size), int(n_overlap), METHODS[method], float(alpha),
                                          float(alpha_cross), out, C.byref(moves)))
        self.timings["decompose"] = time.perf_counter() - t0
        self.n_sub = lib().cpddg_setup_n_subdomains(self._h)
        self.method = method
        return out, moves.value

    def phase_seconds(self) -> dict:
        """Setup phase times of the native layer (band, E, A, alignment,
        subdomain sets, local systems)."""
        t = np.zeros(6)
        check(lib().cpddg_setup_timings(self._h, t))
        return dict(zip(("band", "E", "A", "align", "sets", "local_systems"), (float(v) for v in t)))

    def subdomain(self, j: int) -> dict:
        D = self.dim
        cnt = np.zeros(8, np.int32)
        check(lib().cpddg_setup_subdomain_counts(self._h, j, cnt))
        arrs = [np.zeros(max(int(c), 1), np.int32) for c in cnt[:4]]
        nbc = int(cnt[4])
        bi = np.zeros(max(nbc, 1) * (D + 4), np.int32)
        br = np.zeros(max(nbc, 1) * (4 * D + 1))
        check(lib().cpddg_setup_subdomain_sets(self._h, j, *arrs, bi, br))
        arrs = [a[: int(c)] for a, c in zip(arrs, cnt[:4])]
        return dict(disjoint=arrs[0], overlap=arrs[1], final_layer=arrs[2], ghosts=arrs[3],
                    bc_int=bi[: nbc * (D + 4)].reshape(nbc, D + 4),
                    bc_real=br[: nbc * (4 * D + 1)].reshape(nbc, 4 * D + 1),
                    fallback_count=int(cnt[5]), n_lambda=int(cnt[6]), n_cross_flagged=int(cnt[7]))

    def fallback_anchors(self) -> int:
        """Sum of Subdomain::fallback_count (pipeline.hpp:203-204)."""
        cnt = np.zeros(8, np.int32)
        total = 0
        for j in range(self.n_sub):
            check(lib().cpddg_setup_subdomain_counts(self._h, j, cnt))
            total += int(cnt[5])
        return total

    def local(self, j: int) -> dict:
        s = np.zeros(4, np.int64)
        check(lib().cpddg_setup_local_sizes(self._h, j, s))
        n_ov, n_bc, nnz, nsc = (int(v) for v in s)
        ptr = np.zeros(n_ov + n_bc + 1, np.int64)
        col, val = np.zeros(max(nnz, 1), np.int32), np.zeros(max(nnz, 1))
        scl, scg = np.zeros(max(nsc, 1), np.int32), np.zeros(max(nsc, 1), np.int32)
        check(lib().cpddg_setup_local(self._h, j, ptr, col, val, scl, scg))
        sub = self.subdomain(j)
        return dict(n_overlap=n_ov, n_bc=n_bc, overlap=sub["overlap"], ptr=ptr, col=col[:nnz],
                    val=val[:nnz], scatter_local=scl[:nsc], scatter_global=scg[:nsc])


# ---------------------------------------------------------------- device operator

class DeviceHelmholtz:
    """Matrix-free A = (c + 2d/h^2) I - h^-2 S E on the device; replaces
    SparseOperator::apply on the assembled A (sparse.hpp:65-75)."""

    def __init__(self, handle: C.c_void_p, n: int):
        self._h = handle
        self._destroy = lib().cpddg_op_destroy
        self.n = n

    @classmethod
    def from_problem(cls, P: Problem) -> "DeviceHelmholtz":
        h = C.c_void_p()
        check(lib().cpddg_op_create_from_setup(P.handle, C.byref(h)))
        return cls(h, P.n_active)

    @classmethod
    def from_band(cls, dim: int, p: int, h: float, c: float, n_active: int, ix, cp) -> "DeviceHelmholtz":
        ix = np.ascontiguousarray(ix, np.int32)
        cp = np.ascontiguousarray(cp, np.float64)
        n_ghost = ix.shape[0] - n_active
        d = _lib.cpddg_band_desc(dim=dim, p=p, n_active=n_active, n_ghost=n_ghost, h=h, c=c,
                                 ix=ix.ctypes.data, cp=cp.ctypes.data)
        hd = C.c_void_p()
        check(lib().cpddg_op_create(C.byref(d), C.byref(hd)))
        return cls(hd, n_active)

    def __del__(self):
        h = getattr(self, "_h", None)
        destroy = getattr(self, "_destroy", None)
        if h is not None and h.value and destroy is not None:
            destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def rows(self) -> int:
        return self.n

    def apply(self, x, out=None):
        torch = _torch()
        if x.numel() != self.n:
            from .errors import InternalError
            raise InternalError(_lib.ERR_INTERNAL, "sparse apply: size mismatch")
        x = x.contiguous()
        y = out if out is not None else torch.empty_like(x)
        check(lib().cpddg_op_apply(self._h, _ptr(x), _ptr(y), _stream()))
        return y

    def residual(self, b, x):
        torch = _torch()
        r = torch.empty_like(b)
        nrm = C.c_double()
        check(lib().cpddg_op_residual(self._h, _ptr(b), _ptr(x), _ptr(r), C.byref(nrm), _stream()))
        return r, nrm.value

    def bytes(self):
        a, s = C.c_int64(), C.c_int64()
        check(lib().cpddg_op_bytes(self._h, C.byref(a), C.byref(s)))
        return a.value, s.value


# ---------------------------------------------------------------- preconditioner

def _local_desc(L: dict):
    """cpddg_local_desc over a LocalOperator-shaped dict (the arrays are returned to keep them alive)."""
    arrs = [np.ascontiguousarray(L["overlap"], np.int32),
            np.ascontiguousarray(L["scatter_local"], np.int32),
            np.ascontiguousarray(L["scatter_global"], np.int32),
            np.ascontiguousarray(L["ptr"], np.int64),
            np.ascontiguousarray(L["col"], np.int32),
            np.ascontiguousarray(L["val"], np.float64)]
    d = _lib.cpddg_local_desc(n_overlap=int(L["n_overlap"]), n_bc=int(L["n_bc"]),
                              overlap=arrs[0].ctypes.data, n_scatter=int(arrs[1].size),
                              scatter_local=arrs[1].ctypes.data, scatter_global=arrs[2].ctypes.data,
                              row_ptr=arrs[3].ctypes.data, col=arrs[4].ctypes.data, val=arrs[5].ctypes.data)
    return d, arrs


def unreferenced_unknowns(L: dict) -> np.ndarray:
    """Mask of the local unknowns the device preconditioner removes before the
    factorisation (closure unknowns only their own row refers to and no scatter
    returns; transmission.hpp:84-92, :66-69).  Host only."""
    d, _keep = _local_desc(L)
    out = np.zeros(int(L["n_overlap"]) + int(L["n_bc"]), np.uint8)
    n = C.c_int()
    check(lib().cpddg_local_unreferenced(C.byref(d), out.ctypes.data_as(C.POINTER(C.c_ubyte)), C.byref(n)))
    assert n.value == int(out.sum())
    return out.astype(bool)


class SchwarzPreconditioner:
    """Device RAS / ORAS preconditioner (SchwarzPreconditioner, solve.hpp:64-86);
    the local factorisations run on the device at construction."""

    def __init__(self, handle: C.c_void_p, n_global: int):
        self._h = handle
        self._destroy = lib().cpddg_pc_destroy
        self.n_global = n_global

    @classmethod
    def from_problem(cls, P: Problem, workers: int = 0) -> "SchwarzPreconditioner":
        opt = _lib.cpddg_pc_options(workers=workers, check_residual=1)
        h = C.c_void_p()
        check(lib().cpddg_pc_create_from_setup(P.handle, C.byref(opt), C.byref(h)))
        return cls(h, P.n_active)

    @classmethod
    def from_locals(cls, n_global: int, locals_: list, workers: int = 0) -> "SchwarzPreconditioner":
        """locals_: dicts with n_overlap, n_bc, overlap, scatter_local,
        scatter_global, ptr, col, val (LocalOperator fields)."""
        keep = []
        descs = (_lib.cpddg_local_desc * len(locals_))()
        for k, L in enumerate(locals_):
            descs[k], arrs = _local_desc(L)
            keep.append(arrs)
        opt = _lib.cpddg_pc_options(workers=workers, check_residual=1)
        h = C.c_void_p()
        check(lib().cpddg_pc_create(int(n_global), len(locals_), descs, C.byref(opt), C.byref(h)))
        return cls(h, n_global)

    def __del__(self):
        h = getattr(self, "_h", None)
        destroy = getattr(self, "_destroy", None)
        if h is not None and h.value and destroy is not None:
            destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def apply(self, r, out=None):
        torch = _torch()
        r = r.contiguous()
        z = out if out is not None else torch.empty_like(r)
        check(lib().cpddg_pc_apply(self._h, _ptr(r), _ptr(z), _stream()))
        return z

    def stats(self) -> dict:
        st = _lib.cpddg_pc_stats()
        check(lib().cpddg_pc_stats_get(self._h, C.byref(st)))
        return {k: getattr(st, k) for k, _ in st._fields_}


# ---------------------------------------------------------------- solvers

@dataclass
class PhaseTimings:
    """solve.hpp:42-47."""
    mesh: float = 0.0
    global_matrix: float = 0.0
    local_operators: float = 0.0
    solve: float = 0.0


@dataclass
class IterationLog:
    """solve.hpp:49-55."""
    residuals: list = field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    final_true_residual: float = -1.0
    timings: PhaseTimings = field(default_factory=PhaseTimings)
    device_seconds: float = 0.0
    kernel_launches: int = 0
    kernel_times: dict = field(default_factory=dict)


@dataclass
class SolveResult:
    """solve.hpp:57-60 (u is a device tensor)."""
    u: object
    log: IterationLog


def _solve(fn, A: DeviceHelmholtz, b, M, rel_tol: float, max_iter: int, restart: int,
           cap: int, profile: bool = False) -> SolveResult:
    torch = _torch()
    b = b.contiguous()
    u = torch.empty_like(b)
    res = (C.c_double * cap)()
    log = _lib.cpddg_log(residuals=C.cast(res, C.POINTER(C.c_double)), capacity=cap)
    prm = _lib.cpddg_solve_params(rel_tol=rel_tol, max_iter=max_iter, restart=restart,
                                  profile_kernels=1 if profile else 0)
    mh = M.handle if M is not None else C.c_void_p()
    check(fn(A.handle, mh, _ptr(b), _ptr(u), C.byref(prm), C.byref(log), _stream()))
    n = min(cap, log.n_residuals)
    out = IterationLog(residuals=list(res[:n]), iterations=log.iterations, converged=bool(log.converged),
                       final_true_residual=log.final_true_residual, device_seconds=log.seconds,
                       kernel_launches=log.kernel_launches)
    out.kernel_times = dict(pc_seconds=log.pc_seconds, pc_launches=log.pc_launches,
                            op_seconds=log.op_seconds, op_launches=log.op_launches)
    out.timings.solve = log.seconds
    return SolveResult(u, out)


def gmres_solve(A: DeviceHelmholtz, b, M: SchwarzPreconditioner | None, rel_tol: float, max_iter: int,
                restart: int = 0, profile: bool = False) -> SolveResult:
    """Right-preconditioned restarted GMRES (solve.hpp:128-214)."""
    return _solve(lib().cpddg_gmres, A, b, M, rel_tol, max_iter, restart, max_iter + 2, profile)


def stationary_solve(A: DeviceHelmholtz, b, M: SchwarzPreconditioner, rel_tol: float,
                     max_iter: int, profile: bool = False) -> SolveResult:
    """Stationary Schwarz iteration u <- u + M^-1 (b - A u) (solve.hpp:95-123)."""
    return _solve(lib().cpddg_stationary, A, b, M, rel_tol, max_iter, 0, max_iter + 2, profile)


def effective_max_iter(mode: str, max_iter: int) -> int:
    """config.hpp:59-62."""
    if max_iter > 0:
        return max_iter
    return 2000 if mode == "gmres" else 5000


def run_solve(cfg: dict, part=None, rhs=None, exact=None) -> dict:
    """run_solve (pipeline.hpp:183-241) on the device path.  cfg keys follow
    RunConfig (config.hpp:19-48): surface, h, p, c, radius, major_radius,
    minor_radius, obj, method, mode, rel_tol, max_iter, gmres_restart,
    n_overlap, n_subdomains, alpha, alpha_cross, tube_radius, workers;
    device_setup (default True: band / closest points and alignment /
    subdomain sets on the GPU, bit-identical to the host).
    `part` (labels) and `rhs` (host array) are required: this path consumes
    partition and right-hand-side files (partition.hpp:519-552,
    pipeline.hpp:103-117), it does not generate them.  `exact`, a function of
    the (n, d) closest points, fills err_inf / err_rms (problems.hpp:93-111);
    the result carries the SolveOutputs fields (pipeline.hpp:171-180) except
    diff_direct (check_direct is a CPU verification aid of the reference)."""
    torch = _torch()
    t = PhaseTimings()
    t0 = time.perf_counter()
    P = Problem(surface=cfg.get("surface", "sphere"), h=float(cfg["h"]), p=int(cfg.get("p", 3)),
                c=float(cfg.get("c", 1.0)), radius=float(cfg.get("radius", 1.0)),
                major_radius=float(cfg.get("major_radius", 2.0 / 3.0)),
                minor_radius=float(cfg.get("minor_radius", 1.0 / 3.0)), obj_path=cfg.get("obj"),
                tube_radius=float(cfg.get("tube_radius", 0.0)), workers=int(cfg.get("workers", 0)),
                device_setup=bool(cfg.get("device_setup", True)))
    t.global_matrix = time.perf_counter() - t0
    from . import io as _io
    if part is None and cfg.get("partition_in"):
        part = _io.read_partition(cfg["partition_in"], P.n_active)
    if rhs is None and str(cfg.get("rhs", "")).startswith("file:"):
        rhs = _io.read_rhs(str(cfg["rhs"])[5:], P.n_active)
    if part is None or rhs is None:
        from .errors import ConfigError
        raise ConfigError(_lib.ERR_CONFIG, "run_solve needs a partition (partition_in) and a right-hand side "
                                           "(rhs = file:PATH)")
    n_sub = int(cfg.get("n_subdomains", int(np.max(part)) + 1))
    if int(np.max(part)) + 1 != n_sub:
        from .errors import ConfigError
        raise ConfigError(_lib.ERR_CONFIG, f"partition file defines {int(np.max(part)) + 1} parts but "
                                           f"n_subdomains = {n_sub}")
    t1 = time.perf_counter()
    aligned, moves = P.decompose(part, int(cfg.get("n_overlap", 4)), cfg.get("method", "oras"),
                                 float(cfg.get("alpha", 1.0)), float(cfg.get("alpha_cross", -1.0)))
    t.mesh = time.perf_counter() - t1
    t2 = time.perf_counter()
    A = DeviceHelmholtz.from_problem(P)
    M = SchwarzPreconditioner.from_problem(P, workers=int(cfg.get("workers", 0)))
    torch.cuda.synchronize()
    t.local_operators = time.perf_counter() - t2
    b = torch.from_numpy(np.ascontiguousarray(rhs, np.float64)).cuda()
    mode = cfg.get("mode", "gmres")
    mi = effective_max_iter(mode, int(cfg.get("max_iter", 0)))
    tol = float(cfg.get("rel_tol", 1e-6))
    if mode == "gmres":
        res = gmres_solve(A, b, M, tol, mi, int(cfg.get("gmres_restart", 0)))
    else:
        res = stationary_solve(A, b, M, tol, mi)
    t.solve = res.log.device_seconds
    res.log.timings = t
    b0 = float(np.linalg.norm(rhs))
    u_host = res.u.cpu().numpy()
    if cfg.get("partition_out"):
        _io.write_partition(cfg["partition_out"], aligned)
    if cfg.get("output_dir"):
        import os
        d = cfg["output_dir"]
        x = P.band()["ix"][: P.n_active] * P.h
        _io.write_solution(os.path.join(d, "solution.csv"), x, u_host)
        _io.write_iterations(os.path.join(d, "iterations.csv"), res.log.residuals)
        _io.write_timings(os.path.join(d, "timings.csv"), t, mode == "gmres")
    err_inf = err_rms = -1.0
    if exact is not None:
        d = u_host - np.asarray(exact(P.active_cp), np.float64)
        err_inf = float(np.max(np.abs(d))) if d.size else 0.0
        err_rms = float(np.sqrt(np.sum(d * d) / max(1, d.size)))
    return dict(u=u_host, log=res.log, part=aligned, align_moves=moves,
                fallback_anchors=P.fallback_anchors(),
                final_relative_residual=res.log.final_true_residual / b0 if b0 > 0 else 0.0,
                err_inf=err_inf, err_rms=err_rms,
                problem=P, operator=A, preconditioner=M)
