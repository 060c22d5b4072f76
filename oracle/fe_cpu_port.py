"""ctypes binding of oracle/fe_cpu_port.cpp -- BASELINE INFRASTRUCTURE ONLY.

The SIMD-batched, per-(form, cell, degree, rule) specialised CPU port of the
reference's cell loop (the paper's cross-element vectorisation).  Used by
bench.py's cpu_baseline and --impl reference legs (timed on the host cores)
and pinned to the oracle in tests/test_cpu_port.py; the product never
imports it.
"""

import ctypes
import os

import numpy as np

from . import fe_oracle_c as foc

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libcpuport.so")
_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} missing: run `make oracle`")
        lib = ctypes.CDLL(LIB)
        d, i, i64, vp = ctypes.c_double, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
        lib.fe_cpu_supported.argtypes = [i] * 7
        lib.fe_cpu_apply.argtypes = [i] * 7 + [vp] * 5 + [d, d, i64, i64, vp, i64] + [vp] * 6 + [i]
        _lib = lib
    return _lib


def _key(P):
    affine = 1 if P.kind in ("triangle", "tetrahedron") else 0
    return (foc.FORMS[P.form], P.d, P.nv, P.nd, P.vs, len(P.qw), affine)


def supported(P) -> bool:
    return P.form in foc.FORMS and bool(load().fe_cpu_supported(*_key(P)))


def assemble(P, coords, cell2vert, cell2dof, u, mu=None, lam=None, start=0, end=None,
             threads=1, out=None, state=None):
    """Same contract as fe_oracle.assemble (accumulates into ``out``)."""
    lib = load()
    keep = []

    def ptr(a, dt=np.float64):
        if a is None:
            return None
        a = np.ascontiguousarray(a, dt)
        keep.append(a)
        return ctypes.c_void_p(a.ctypes.data)

    u = np.ascontiguousarray(u, np.float64)
    y = np.zeros_like(u) if out is None else out
    end = len(cell2dof) if end is None else end
    c0, c1 = mu, lam
    if P.form == "neohookean_tangent":
        if state is None:
            raise ValueError("neohookean_tangent needs the state u0")
        c0, c1 = state, None
    p0, p1 = (tuple(P.params) + (0.0, 0.0))[:2] if P.params else (0.0, 0.0)
    rc = lib.fe_cpu_apply(*_key(P), ptr(P.qw), ptr(P.phi), ptr(P.dphi), ptr(P.gphi), ptr(P.gdphi),
                          p0, p1, int(start), int(end), ctypes.c_void_p(y.ctypes.data), y.size,
                          ptr(coords), ptr(u), ptr(cell2dof, np.int32), ptr(cell2vert, np.int32),
                          ptr(c0), ptr(c1), int(threads))
    if rc != 0:
        raise ValueError(f"no CPU port specialisation for {P.form} {P.kind} p{P.k} nq={len(P.qw)}")
    return y
