"""ctypes binding of the C ABI in ``include/fe_b200.h`` (libfeb200.so).

The reference loads its generated kernels the same way
(``/root/reference/pkg/src/fevec/jit.py:90-111``: ``ctypes.CDLL`` on the
compiled object).  There is no fallback: if the library is missing, or no
CUDA device is present when a kernel is launched, the call raises.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FE_LIB_PATH") or os.path.join(HERE, "libfeb200.so")

FORMS = {
    "mass": 0, "helmholtz": 1, "laplacian": 2, "elasticity": 3,
    "laplacian_scalar": 4, "elasticity_lame": 5, "neohookean": 6, "neohookean_tangent": 7,
}
CELLS = {"triangle": 0, "quadrilateral": 1, "tetrahedron": 2, "hexahedron": 3}

FE_PTR_HOST = 0
FE_PTR_DEVICE = 1
FE_APPLY_ACCUMULATE = 0
FE_APPLY_OVERWRITE = 1
FE_PLAN_GENERIC = 1          # plan flag: force the generic quadrature kernel

ERRORS = {1: "EINVAL", 2: "EUNSUPPORTED", 3: "ECUDA", 4: "ENOMESH", 5: "ENOMEM"}

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int32)


class ElementDesc(ctypes.Structure):
    _fields_ = [
        ("form", ctypes.c_int32), ("cell", ctypes.c_int32),
        ("degree", ctypes.c_int32), ("value_size", ctypes.c_int32),
        ("ndof", ctypes.c_int32), ("nvert", ctypes.c_int32), ("nq", ctypes.c_int32),
        ("qweights", _dp), ("phi", _dp), ("dphi", _dp), ("gphi", _dp), ("gdphi", _dp),
        ("q1d", ctypes.c_int32),
        ("B1d", _dp), ("D1d", _dp), ("w1d", _dp), ("x1d", _dp), ("lex", _ip),
        ("params", ctypes.c_double * 4),
        ("nq_aux", ctypes.c_int32), ("qw_aux", _dp), ("dphi_aux", _dp),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("kernel", ctypes.c_char * 64),
        ("threads_per_cell", ctypes.c_int32),
        ("block", ctypes.c_int32),
        ("launches_per_apply", ctypes.c_int32),
        ("ncells", ctypes.c_int64),
        ("nglobal", ctypes.c_int64),
    ]


class FeError(RuntimeError):
    """A failed call across the C ABI (carries fe_last_error())."""


# every symbol include/fe_b200.h declares
EXPORTS = (
    "fe_abi_version", "fe_plan_create", "fe_plan_bind_mesh", "fe_apply", "fe_wrap",
    "fe_wrap_host", "fe_plan_get_info", "fe_plan_destroy", "fe_last_error", "fe_diagonal",
    "fe_eval_log", "fe_launch_count",
)

_lib = None


def load():
    """Load libfeb200.so (built by ``make`` / ``__graft_entry__.build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FeError(
            f"{LIB_PATH} is missing: build the sm_100a extension with `make` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    vp = ctypes.c_void_p
    lib.fe_abi_version.restype = ctypes.c_int
    lib.fe_last_error.restype = ctypes.c_char_p
    lib.fe_plan_create.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(ElementDesc), ctypes.c_uint32]
    lib.fe_plan_bind_mesh.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                      vp, vp, vp, ctypes.c_uint32, vp]
    lib.fe_apply.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, vp, vp, vp, vp,
                             ctypes.c_uint32, vp]
    lib.fe_wrap.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, vp, vp, vp, vp, vp, vp, vp, vp]
    lib.fe_diagonal.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, vp, vp, vp, ctypes.c_uint32, vp]
    lib.fe_wrap_host.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, vp, vp, vp, vp, vp, vp, vp]
    lib.fe_plan_get_info.argtypes = [vp, ctypes.POINTER(PlanInfo)]
    lib.fe_eval_log.argtypes = [vp, vp, ctypes.c_int64, vp]
    lib.fe_launch_count.restype = ctypes.c_int64
    lib.fe_launch_count.argtypes = []
    lib.fe_plan_destroy.argtypes = [vp]
    lib.fe_plan_destroy.restype = None
    for name in ("fe_plan_create", "fe_plan_bind_mesh", "fe_apply", "fe_wrap",
                 "fe_wrap_host", "fe_plan_get_info"):
        getattr(lib, name).restype = ctypes.c_int
    if lib.fe_abi_version() != 1:
        raise FeError("libfeb200.so ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().fe_last_error().decode(errors="replace")
        raise FeError(f"{what}: {ERRORS.get(rc, rc)}: {msg}")
