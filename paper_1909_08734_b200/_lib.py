"""ctypes binding of lib/libcpddg.so (the C ABI declared in include/cpddg.h).

The library is built in-tree (``python -c "import __graft_entry__ as g; g.build()"``
or ``make -C paper_1909_08734_b200/csrc``).  There is no fallback: if the
library is missing, importing a solver raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CPDDG_LIB") or os.path.join(_HERE, "lib", "libcpddg.so")

OK, ERR_INTERNAL, ERR_CONFIG, ERR_DIVERGENCE, ERR_IO, ERR_CUDA = range(6)

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_vp = C.c_void_p


class cpddg_problem_desc(C.Structure):
    _fields_ = [("dim", C.c_int), ("surface", C.c_int), ("radius", C.c_double),
                ("major_radius", C.c_double), ("minor_radius", C.c_double),
                ("obj_path", C.c_char_p), ("h", C.c_double), ("p", C.c_int),
                ("tube_radius", C.c_double), ("c", C.c_double), ("workers", C.c_int),
                ("device_setup", C.c_int)]


class cpddg_band_desc(C.Structure):
    _fields_ = [("dim", C.c_int), ("p", C.c_int), ("n_active", C.c_int), ("n_ghost", C.c_int),
                ("h", C.c_double), ("c", C.c_double), ("ix", _vp), ("cp", _vp)]


class cpddg_local_desc(C.Structure):
    _fields_ = [("n_overlap", C.c_int), ("n_bc", C.c_int), ("overlap", _vp), ("n_scatter", C.c_int),
                ("scatter_local", _vp), ("scatter_global", _vp), ("row_ptr", _vp), ("col", _vp),
                ("val", _vp)]


class cpddg_pc_options(C.Structure):
    _fields_ = [("workers", C.c_int), ("check_residual", C.c_int)]


class cpddg_pc_stats(C.Structure):
    _fields_ = [("n_sub", C.c_int), ("n_reduced", C.c_int), ("n_rows_total", C.c_int64),
                ("factor_entries", C.c_int64), ("profile_entries", C.c_int64), ("factor_bytes", C.c_int64),
                ("algorithmic_bytes", C.c_int64), ("max_rows", C.c_int),
                ("factor_seconds", C.c_double), ("analyse_seconds", C.c_double),
                ("max_probe_residual", C.c_double), ("apply_mode", C.c_int), ("n_pivoted", C.c_int),
                ("win_cuts", C.c_int), ("win_lpt_efficiency", C.c_double), ("win_bal_efficiency", C.c_double),
                ("n_dropped", C.c_int64)]


class cpddg_solve_params(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("max_iter", C.c_int), ("restart", C.c_int),
                ("profile_kernels", C.c_int)]


class cpddg_log(C.Structure):
    _fields_ = [("residuals", C.POINTER(C.c_double)), ("capacity", C.c_int),
                ("n_residuals", C.c_int), ("iterations", C.c_int), ("converged", C.c_int),
                ("final_true_residual", C.c_double), ("seconds", C.c_double),
                ("kernel_launches", C.c_int64), ("pc_seconds", C.c_double), ("pc_launches", C.c_int64),
                ("op_seconds", C.c_double), ("op_launches", C.c_int64)]


_SIGS = {
    "cpddg_last_error": (C.c_int, [C.c_char_p, C.c_size_t]),
    "cpddg_version": (C.c_char_p, []),
    "cpddg_setup_create": (C.c_int, [C.POINTER(cpddg_problem_desc), C.POINTER(_vp)]),
    "cpddg_setup_destroy": (C.c_int, [_vp]),
    "cpddg_setup_sizes": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "cpddg_setup_band": (C.c_int, [_vp, _i32p, _f64p, _f64p, _f64p]),
    "cpddg_setup_csr": (C.c_int, [_vp, C.c_int, _i64p, _i32p, _f64p]),
    "cpddg_setup_decompose": (C.c_int, [_vp, _i32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                        _i32p, C.POINTER(C.c_int)]),
    "cpddg_setup_n_subdomains": (C.c_int, [_vp]),
    "cpddg_setup_timings": (C.c_int, [_vp, _f64p]),
    "cpddg_pc_debug_zero_stats": (C.c_int, [_vp, _i64p]),
    "cpddg_setup_subdomain_counts": (C.c_int, [_vp, C.c_int, _i32p]),
    "cpddg_setup_subdomain_sets": (C.c_int, [_vp, C.c_int, _i32p, _i32p, _i32p, _i32p, _i32p, _f64p]),
    "cpddg_setup_local_sizes": (C.c_int, [_vp, C.c_int, _i64p]),
    "cpddg_setup_local": (C.c_int, [_vp, C.c_int, _i64p, _i32p, _f64p, _i32p, _i32p]),
    "cpddg_op_create": (C.c_int, [C.POINTER(cpddg_band_desc), C.POINTER(_vp)]),
    "cpddg_op_create_from_setup": (C.c_int, [_vp, C.POINTER(_vp)]),
    "cpddg_op_apply": (C.c_int, [_vp, _vp, _vp, _vp]),
    "cpddg_op_residual": (C.c_int, [_vp, _vp, _vp, _vp, C.POINTER(C.c_double), _vp]),
    "cpddg_op_size": (C.c_int, [_vp]),
    "cpddg_op_bytes": (C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "cpddg_op_destroy": (C.c_int, [_vp]),
    "cpddg_pc_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(cpddg_local_desc),
                                  C.POINTER(cpddg_pc_options), C.POINTER(_vp)]),
    "cpddg_pc_create_from_setup": (C.c_int, [_vp, C.POINTER(cpddg_pc_options), C.POINTER(_vp)]),
    "cpddg_local_unreferenced": (C.c_int, [C.POINTER(cpddg_local_desc), C.POINTER(C.c_ubyte), C.POINTER(C.c_int)]),
    "cpddg_pc_apply": (C.c_int, [_vp, _vp, _vp, _vp]),
    "cpddg_pc_stats_get": (C.c_int, [_vp, C.POINTER(cpddg_pc_stats)]),
    "cpddg_pc_destroy": (C.c_int, [_vp]),
    "cpddg_gmres": (C.c_int, [_vp, _vp, _vp, _vp, C.POINTER(cpddg_solve_params),
                              C.POINTER(cpddg_log), _vp]),
    "cpddg_stationary": (C.c_int, [_vp, _vp, _vp, _vp, C.POINTER(cpddg_solve_params),
                                   C.POINTER(cpddg_log), _vp]),
    # development / profiling entry points (last section of include/cpddg.h)
    "cpddg_pc_apply_mode": (C.c_int, [_vp, _vp, _vp, C.c_int, _vp]),
    "cpddg_dev_trace": (C.c_int, [_vp]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


def lib():
    """Load lib/libcpddg.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                               "(no CPU fallback exists for the solve path)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class CpddgError(RuntimeError):
    """Failure reported through the C ABI; `code` follows include/cpddg.h."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def check(rc: int) -> None:
    if rc != OK:
        buf = C.create_string_buffer(4096)
        lib().cpddg_last_error(buf, 4096)
        raise error_for(rc, buf.value.decode(errors="replace"))


def error_for(code: int, msg: str) -> Exception:
    from . import errors
    cls = {ERR_CONFIG: errors.ConfigError, ERR_DIVERGENCE: errors.DivergenceError,
           ERR_IO: errors.IoError, ERR_INTERNAL: errors.InternalError,
           ERR_CUDA: errors.CudaError}.get(code, CpddgError)
    return cls(code, msg)
