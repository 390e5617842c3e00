"""ctypes binding of the C-ABI library ``librbns.so`` (declared in include/rbns.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``python -m paper_1807_11866_b200.build``).  There
is no fallback: if the shared object is missing or fails to load, every entry point raises ``NativeError``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import NativeError

LIB_PATH = Path(os.environ.get("RBNS_LIB", Path(__file__).resolve().parent / "librbns.so"))

MAX_TERMS = 256
MAX_GROUPS = 4
NU_LINEAR = 1
STOP_ABSOLUTE = 2
STATUS_NAMES = {0: "CONVERGED", 1: "NON_CONVERGED", 2: "SINGULAR_SYSTEM", 3: "SINGULAR_RECOVERY", 4: "NONFINITE"}

# every symbol include/rbns.h declares (checked by tests/test_abi.py)
EXPORTED_SYMBOLS = (
    "rbns_model_create", "rbns_model_create2", "rbns_model_terms", "rbns_model_destroy", "rbns_model_info",
    "rbns_model_device_bytes", "rbns_model_contraction_slices", "rbns_model_attached", "rbns_solve", "rbns_solve_ex", "rbns_solve_host",
    "rbns_solve_host_ex", "rbns_reduced_operator", "rbns_recover_pressure", "rbns_reconstruct_pressure",
    "rbns_get_stats", "rbns_project_convection", "rbns_error_string", "rbns_last_error_message",
    "rbns_abi_version",
)
ABI_VERSION = 3
ERR_NO_ATTACHED = 6


class ThetaTermC(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("k", ctypes.c_int32), ("m", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("scale", ctypes.c_double)]


class ModelDescC(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("q", ctypes.c_int32), ("n_p", ctypes.c_int32),
                ("reserved", ctypes.c_int32),
                ("A", ctypes.c_void_p), ("C", ctypes.c_void_p), ("f", ctypes.c_void_p),
                ("Mp", ctypes.c_void_p), ("Bq", ctypes.c_void_p), ("theta", ctypes.POINTER(ThetaTermC))]


class TermFamilyC(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int32), ("reserved", ctypes.c_int32), ("data", ctypes.c_void_p),
                ("theta", ctypes.POINTER(ThetaTermC))]


class ModelDesc2C(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("n_p", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("n_stop", ctypes.c_int32), ("linear", TermFamilyC), ("quadratic", TermFamilyC),
                ("load", TermFamilyC), ("coupling", TermFamilyC), ("Mp", ctypes.c_void_p),
                ("n_att", ctypes.c_int32), ("reserved2", ctypes.c_int32), ("P_att", ctypes.c_void_p)]


class StatsC(ctypes.Structure):
    _fields_ = [("sample_iterations", ctypes.c_int64), ("contraction_iterations", ctypes.c_int64),
                ("newton_rounds", ctypes.c_int32), ("kernel_launches", ctypes.c_int32),
                ("gemm_launches", ctypes.c_int32), ("lu_launches", ctypes.c_int32),
                ("ms_gemm", ctypes.c_double), ("ms_lu", ctypes.c_double), ("ms_recovery", ctypes.c_double),
                ("ms_total", ctypes.c_double), ("ms_assembly", ctypes.c_double),
                ("pivot_fallbacks", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None


def load(path: os.PathLike | None = None) -> ctypes.CDLL:
    """Load (once) and type the library; raises NativeError when it is absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise NativeError(f"CUDA library {p} not built: run __graft_entry__.build() "
                          "(there is no CPU fallback for the online solver)")
    try:
        lib = ctypes.CDLL(str(p))
    except OSError as exc:  # pragma: no cover - depends on the box
        raise NativeError(f"failed to load {p}: {exc}") from exc
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    lib.rbns_model_create.argtypes = [ctypes.POINTER(ModelDescC), ctypes.c_int, ctypes.POINTER(vp)]
    lib.rbns_model_create2.argtypes = [ctypes.POINTER(ModelDesc2C), ctypes.c_int, ctypes.POINTER(vp)]
    lib.rbns_model_terms.argtypes = [vp, ctypes.POINTER(i32)]
    lib.rbns_model_destroy.argtypes = [vp]
    lib.rbns_model_info.argtypes = [vp] + [ctypes.POINTER(i32)] * 4
    lib.rbns_model_device_bytes.argtypes = [vp]
    lib.rbns_model_device_bytes.restype = i64
    lib.rbns_model_contraction_slices.argtypes = [vp]
    lib.rbns_model_contraction_slices.restype = ctypes.c_int
    solve_args = [vp, vp, i64, dbl, i32, vp, vp, vp, vp, vp, vp]
    lib.rbns_solve.argtypes = solve_args
    lib.rbns_solve_host.argtypes = solve_args
    solve_ex_args = [vp, vp, i64, dbl, i32, vp, vp, vp, vp, vp, ctypes.POINTER(StatsC), vp]
    lib.rbns_solve_ex.argtypes = solve_ex_args
    lib.rbns_solve_host_ex.argtypes = solve_ex_args
    lib.rbns_reconstruct_pressure.argtypes = [vp, vp, i64, vp, vp]
    lib.rbns_model_attached.argtypes = [vp, ctypes.POINTER(i32)]
    lib.rbns_reduced_operator.argtypes = [vp, vp, vp, i64, vp, vp, vp]
    lib.rbns_recover_pressure.argtypes = [vp, vp, vp, i64, vp, vp, vp]
    lib.rbns_get_stats.argtypes = [vp, ctypes.POINTER(StatsC)]
    lib.rbns_project_convection.argtypes = [vp, vp, vp, vp, i64, i32, vp, i32, vp]
    lib.rbns_error_string.argtypes = [ctypes.c_int]
    lib.rbns_error_string.restype = ctypes.c_char_p
    lib.rbns_last_error_message.argtypes = []
    lib.rbns_last_error_message.restype = ctypes.c_char_p
    lib.rbns_abi_version.restype = ctypes.c_int
    if lib.rbns_abi_version() != ABI_VERSION:
        raise NativeError(f"{p}: ABI version {lib.rbns_abi_version()}, this package binds {ABI_VERSION} "
                          "(rebuild with __graft_entry__.build())")
    for name in EXPORTED_SYMBOLS:
        if name not in ("rbns_model_device_bytes", "rbns_error_string", "rbns_last_error_message",
                        "rbns_abi_version"):
            getattr(lib, name).restype = ctypes.c_int
    if path is None:
        _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        lib = load()
        msg = lib.rbns_error_string(rc).decode()
        detail = lib.rbns_last_error_message().decode()
        raise NativeError(f"{what} failed ({rc}: {msg}): {detail}")
