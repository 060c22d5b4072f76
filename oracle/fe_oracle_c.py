"""ctypes binding of oracle/fe_oracle.c -- TEST / BASELINE INFRASTRUCTURE ONLY.

The compiled restatement of the reference's generated cell loop; used by
bench.py's cpu_baseline and --impl reference legs (timed on the host cores)
and cross-checked against the numpy oracle in tests/test_oracle_c.py.
"""

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
FORMS = {"mass": 0, "helmholtz": 1, "laplacian": 2, "elasticity": 3, "laplacian_scalar": 4,
         "elasticity_lame": 5, "neohookean": 6, "neohookean_tangent": 7}
_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} missing: run `make oracle`")
        _lib = ctypes.CDLL(LIB)
        for name in ("fe_oracle_apply", "fe_oracle_apply_mt"):
            getattr(_lib, name).restype = None
    return _lib


def _p(a, t=ctypes.c_double):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(t))


def assemble(P, coords, cell2vert, cell2dof, u, mu=None, lam=None, start=0, end=None,
             threads=1, out=None, state=None):
    """Same contract as fe_oracle.assemble, computed by the C loop
    (``state``: the linearisation point u0 of neohookean_tangent)."""
    lib = load()
    coords = np.ascontiguousarray(coords, np.float64)
    c2v = np.ascontiguousarray(cell2vert, np.int32)
    c2d = np.ascontiguousarray(cell2dof, np.int32)
    u = np.ascontiguousarray(u, np.float64)
    end = len(c2d) if end is None else end
    y = np.zeros_like(u) if out is None else out
    tabs = [np.ascontiguousarray(a, np.float64) for a in (P.qw, P.phi, P.dphi, P.gphi, P.gdphi)]
    if mu is not None:
        mu = np.ascontiguousarray(mu, np.float64)
        lam = np.ascontiguousarray(lam, np.float64)
    if P.form == "neohookean_tangent":
        if state is None:
            raise ValueError("neohookean_tangent needs the state u0")
        mu, lam = np.ascontiguousarray(state, np.float64), None   # passed as the dof field mu
    affine = 1 if P.kind in ("triangle", "tetrahedron") else 0
    p0, p1 = (P.params + (0.0, 0.0))[:2] if P.params else (0.0, 0.0)
    args = [FORMS[P.form], P.d, P.nv, P.nd, P.vs, len(P.qw), affine] + [_p(t) for t in tabs] + [
        ctypes.c_double(p0), ctypes.c_double(p1), int(start), int(end), _p(y), _p(coords), _p(u),
        _p(c2d, ctypes.c_int32), _p(c2v, ctypes.c_int32), _p(mu), _p(lam)]
    if threads > 1:
        lib.fe_oracle_apply_mt(*args, int(threads))
    else:
        lib.fe_oracle_apply(*args)
    return y
