"""Operator plans behind the reference's ``emit_for`` / ``compile_and_load`` /
``KernelHandle`` interface.

Reference (``/root/reference/pkg/src/fevec``):

* ``bench.emit_for(spec, target, rule)`` (``bench.py:81-91``) emits C for one
  (form, cell, degree) and ``jit.compile_and_load(unit)`` (``jit.py:90-111``)
  compiles and dlopens it;
* ``KernelHandle.__call__(start, end, bindings)`` (``jit.py:71-87``) looks up
  the named buffers ``dat0, dat1, dat2, map0, map1``, checks dtypes
  (``TypeError``; ``KeyError`` for a missing binding) and calls
  ``wrap_<form>``.

Here ``emit_for`` returns a :class:`PlanUnit` (the tables the reference would
bake into the emitted source) and ``compile_and_load`` creates an sm_100a
plan in ``libfeb200.so`` whose kernel was compiled ahead of time.  The
returned :class:`GpuKernelHandle` is called exactly like ``KernelHandle``:

* with numpy bindings it is the drop-in host path (``fe_wrap_host``: upload,
  apply, download, accumulate into ``dat0``);
* with CUDA torch tensors it stays on the device (``fe_wrap`` on the current
  stream);
* ``handle.apply(u, y, ...)`` is the device fast path used by the benchmark.

The mesh (``dat1``/``map0``/``map1``) is re-laid out for the GPU once and
cached by buffer identity (the reference's builders return read-only arrays,
``mesh.py:58-60,114``); call :meth:`GpuKernelHandle.rebind` after mutating
mesh buffers in place.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .elements import (OperatorSpec, QuadratureRule, integrand_degree, quadrature_rule,
                       stiffness_modes, tabulate, tensor_factors)

__all__ = ["Target", "PlanUnit", "emit_for", "compile_and_load", "GpuKernelHandle",
           "ToolchainError", "KernelError"]


class ToolchainError(Exception):
    """No sm_100a kernel exists for the requested unit (reference jit.py:30-31)."""


KernelError = _lib.FeError


@dataclass(frozen=True)
class Target:
    """Compilation target.  The only target is sm_100a; ``generic`` forces the
    reference-structured quadrature kernel instead of the specialised one."""
    kind: str = "sm100a"
    generic: bool = False


@dataclass(frozen=True)
class PlanUnit:
    spec: OperatorSpec
    rule: QuadratureRule
    target: Target
    entry: str
    args: tuple = field(default=())


def _wrapper_args(spec: OperatorSpec) -> tuple:
    """Argument list of wrap_<form> in reference order (codegen.py:375-394):
    start, end, the dats in local-kernel argument order, then the maps."""
    args = [("start", "int32", "read"), ("end", "int32", "read"),
            ("dat0", "real64", "inc"), ("dat1", "real64", "read"),
            ("dat2", "real64", "read")]
    if spec.coefficient_fields:
        args += [("dat3", "real64", "read"), ("dat4", "real64", "read")]
    elif spec.has_state:
        args += [("dat3", "real64", "read")]
    args += [("map0", "int32", "read"), ("map1", "int32", "read")]
    return tuple(args)


def emit_for(spec: OperatorSpec, target: Target = None, rule: QuadratureRule = None) -> PlanUnit:
    if target is None:
        target = Target()
    if rule is None:
        rule = quadrature_rule(spec.cell, integrand_degree(spec))
    if rule.cell.kind != spec.cell.kind:
        raise ValueError(f"operator on {spec.cell.kind} with a {rule.cell.kind} quadrature rule")
    return PlanUnit(spec, rule, target, f"wrap_{spec.form}", _wrapper_args(spec))


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _dptr(a):
    return ctypes.cast(a.ctypes.data, ctypes.POINTER(ctypes.c_double))


class GpuKernelHandle:
    """A loaded sm_100a operator plan, callable like the reference's
    ``KernelHandle`` (``jit.py:47-87``)."""

    def __init__(self, unit: PlanUnit):
        self.unit = unit
        self.spec = spec = unit.spec
        rule = unit.rule
        lib = _lib.load()
        el, geo, cell = spec.element, spec.geometry, spec.cell
        tab = tabulate(el, rule)
        gtab = tabulate(geo, rule)
        keep = {
            "qw": np.ascontiguousarray(rule.weights, dtype=np.float64),
            "phi": np.ascontiguousarray(tab.values, dtype=np.float64),
            "dphi": np.ascontiguousarray(tab.grads, dtype=np.float64),
            "gphi": np.ascontiguousarray(gtab.values, dtype=np.float64),
            "gdphi": np.ascontiguousarray(gtab.grads, dtype=np.float64),
        }
        d = _lib.ElementDesc()
        d.form = _lib.FORMS[spec.form]
        d.cell = _lib.CELLS[cell.kind]
        d.degree = el.degree
        d.value_size = el.value_size
        d.ndof = el.ndof_scalar
        d.nvert = cell.nvertices
        d.nq = rule.npoints
        d.qweights = _dptr(keep["qw"])
        d.phi = _dptr(keep["phi"])
        d.dphi = _dptr(keep["dphi"])
        d.gphi = _dptr(keep["gphi"])
        d.gdphi = _dptr(keep["gdphi"])
        d.q1d = 0
        if not cell.simplex:
            tf = tensor_factors(el, rule)
            keep["B"] = np.ascontiguousarray(tf.B)
            keep["D"] = np.ascontiguousarray(tf.D)
            keep["w"] = np.ascontiguousarray(tf.w)
            keep["x"] = np.ascontiguousarray(tf.x)
            keep["lex"] = np.ascontiguousarray(tf.lex, dtype=np.int32)
            d.q1d = rule.npoints_1d
            d.B1d = _dptr(keep["B"])
            d.D1d = _dptr(keep["D"])
            d.w1d = _dptr(keep["w"])
            d.x1d = _dptr(keep["x"])
            d.lex = ctypes.cast(keep["lex"].ctypes.data, ctypes.POINTER(ctypes.c_int32))
        for i, v in enumerate(spec.params[:4]):
            d.params[i] = v
        d.nq_aux = 0
        if cell.simplex and spec.form in ("helmholtz", "laplacian_scalar"):
            qw_aux, dphi_aux = stiffness_modes(el, cell)
            keep["qw_aux"] = qw_aux
            keep["dphi_aux"] = dphi_aux
            d.nq_aux = qw_aux.shape[0]
            d.qw_aux = _dptr(keep["qw_aux"])
            d.dphi_aux = _dptr(keep["dphi_aux"])
        plan = ctypes.c_void_p()
        flags = _lib.FE_PLAN_GENERIC if unit.target.generic else 0
        rc = lib.fe_plan_create(ctypes.byref(plan), ctypes.byref(d), flags)
        if rc == 2:
            raise ToolchainError(lib.fe_last_error().decode())
        _lib.check(rc, "fe_plan_create")
        self._lib = lib
        self._plan = plan
        self._bound = None
        self._keep_mesh = None

    # -- plan info ---------------------------------------------------------

    @property
    def info(self) -> dict:
        i = _lib.PlanInfo()
        _lib.check(self._lib.fe_plan_get_info(self._plan, ctypes.byref(i)), "fe_plan_get_info")
        return {"kernel": i.kernel.decode(), "block": i.block, "ncells": i.ncells,
                "nglobal": i.nglobal, "launches_per_apply": i.launches_per_apply}

    @property
    def value_size(self) -> int:
        return self.spec.element.value_size

    # -- mesh binding --------------------------------------------------------

    def bind(self, coords, map0, map1=None, nglobal=None, stream=None):
        """Upload + re-lay out the mesh.  numpy arrays -> host pointers; CUDA
        torch tensors -> device pointers."""
        nd = self.spec.element.ndof_scalar
        nv = self.spec.cell.nvertices
        dim = self.spec.cell.dim
        dev = _is_cuda(map0)
        if dev:
            ncells = map0.numel() // nd
            nverts = coords.numel() // dim
            ptrs = (coords.data_ptr(), map0.data_ptr(), map1.data_ptr() if map1 is not None else None)
            flags = _lib.FE_PTR_DEVICE
            if stream is None:
                import torch
                stream = torch.cuda.current_stream().cuda_stream
        else:
            coords = _host(coords, np.float64, "dat1")
            map0 = _host(map0, np.int32, "map0")
            map1 = _host(map1, np.int32, "map1") if map1 is not None else None
            ncells = map0.size // nd
            nverts = coords.size // dim
            ptrs = (coords.ctypes.data, map0.ctypes.data, map1.ctypes.data if map1 is not None else None)
            flags = _lib.FE_PTR_HOST
        if nglobal is None:
            raise ValueError("nglobal (scalar dof count) is required")
        rc = self._lib.fe_plan_bind_mesh(self._plan, ncells, nverts, int(nglobal),
                                         ctypes.c_void_p(ptrs[0]), ctypes.c_void_p(ptrs[1]),
                                         ctypes.c_void_p(ptrs[2]) if ptrs[2] else None,
                                         flags, ctypes.c_void_p(stream) if stream else None)
        _lib.check(rc, "fe_plan_bind_mesh")
        self._bound = (flags, ptrs, ncells, int(nglobal))
        self._keep_mesh = (coords, map0, map1)

    def rebind(self):
        self._bound = None

    @property
    def ncells(self) -> int:
        return self._bound[2] if self._bound else 0

    # -- calls ---------------------------------------------------------------

    def __call__(self, start: int, end: int, bindings: dict) -> None:
        names = [a[0] for a in self.unit.args[2:]]
        bufs = {}
        for name in names:
            try:
                bufs[name] = bindings[name]
            except KeyError:
                raise KeyError(f"no binding for kernel argument {name!r}") from None
        vs = self.value_size
        if _is_cuda(bufs["dat0"]):
            self._call_device(start, end, bufs, vs)
        else:
            self._call_host(start, end, bufs, vs)

    def _ensure_bound(self, flags, coords, map0, map1, nglobal, stream=None):
        if flags == _lib.FE_PTR_DEVICE:
            ptrs = (coords.data_ptr(), map0.data_ptr(), map1.data_ptr())
        else:
            ptrs = (coords.ctypes.data, map0.ctypes.data, map1.ctypes.data)
        b = self._bound
        if b is None or b[0] != flags or b[1] != ptrs or b[3] != nglobal:
            self.bind(coords, map0, map1, nglobal=nglobal, stream=stream)

    def _call_host(self, start, end, bufs, vs):
        out = bufs["dat0"]
        if not isinstance(out, np.ndarray) or out.dtype != np.float64:
            raise TypeError(f"binding 'dat0' has dtype {getattr(out, 'dtype', type(out))}, expected float64")
        if not (out.flags.c_contiguous and out.flags.writeable):
            raise ValueError("binding 'dat0' must be a writeable C-contiguous array "
                             "(the output is accumulated in place)")
        conv = {}
        for name, buf in bufs.items():
            want = np.int32 if name.startswith("map") else np.float64
            conv[name] = _host(buf, want, name)
        nglobal = conv["dat2"].size // vs
        if conv["dat0"].size != conv["dat2"].size:
            raise ValueError("dat0 and dat2 sizes differ")
        self._ensure_bound(_lib.FE_PTR_HOST, conv["dat1"], conv["map0"], conv["map1"], nglobal)
        rc = self._lib.fe_wrap_host(
            self._plan, int(start), int(end), _ptr(conv["dat0"]), _ptr(conv["dat1"]),
            _ptr(conv["dat2"]), _ptr(conv.get("dat3")), _ptr(conv.get("dat4")),
            _ptr(conv["map0"]), _ptr(conv["map1"]))
        _lib.check(rc, "fe_wrap_host")

    def _call_device(self, start, end, bufs, vs):
        import torch
        for name, buf in bufs.items():
            want = torch.int32 if name.startswith("map") else torch.float64
            if buf.dtype != want:
                raise TypeError(f"binding {name!r} has dtype {buf.dtype}, expected {want}")
            if not buf.is_contiguous():
                raise ValueError(f"binding {name!r} must be contiguous")
        stream = torch.cuda.current_stream().cuda_stream
        nglobal = bufs["dat2"].numel() // vs
        self._ensure_bound(_lib.FE_PTR_DEVICE, bufs["dat1"], bufs["map0"], bufs["map1"], nglobal, stream)
        p = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
        rc = self._lib.fe_wrap(self._plan, int(start), int(end), p(bufs["dat0"]), p(bufs["dat1"]),
                               p(bufs["dat2"]), p(bufs.get("dat3")), p(bufs.get("dat4")),
                               p(bufs["map0"]), p(bufs["map1"]), ctypes.c_void_p(stream))
        _lib.check(rc, "fe_wrap")

    def apply(self, u, y, start=0, end=None, coef=None, overwrite=False, stream=None):
        """Device fast path on the bound mesh: y (+)= A(u) over [start, end).
        ``u``/``y`` are CUDA float64 tensors (or raw device pointers)."""
        if self._bound is None:
            raise _lib.FeError("no mesh bound: call bind() first")
        end = self._bound[2] if end is None else end
        ptr = lambda t: None if t is None else ctypes.c_void_p(t if isinstance(t, int) else t.data_ptr())
        c0, c1 = (None, None) if coef is None else coef
        if stream is None:
            import torch
            stream = torch.cuda.current_stream().cuda_stream
        rc = self._lib.fe_apply(self._plan, int(start), int(end), ptr(y), ptr(u), ptr(c0), ptr(c1),
                                _lib.FE_APPLY_OVERWRITE if overwrite else _lib.FE_APPLY_ACCUMULATE,
                                ctypes.c_void_p(stream) if stream else None)
        _lib.check(rc, "fe_apply")

    def diagonal(self, coef=None, out=None, start=0, end=None, stream=None):
        """Operator diagonal on the bound mesh (fe_diagonal): a CUDA float64
        tensor of vs*nglobal entries, e.g. the Jacobi preconditioner of
        ``solver.cg``.  Linear forms (and the tangent at its state) only."""
        import torch
        if self._bound is None:
            raise _lib.FeError("no mesh bound: call bind() first")
        end = self._bound[2] if end is None else end
        if out is None:
            out = torch.zeros(self.value_size * self._bound[3], dtype=torch.float64, device="cuda")
        ptr = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())
        c0, c1 = (None, None) if coef is None else coef
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        rc = self._lib.fe_diagonal(self._plan, int(start), int(end), ptr(out), ptr(c0), ptr(c1),
                                   _lib.FE_APPLY_ACCUMULATE, ctypes.c_void_p(stream))
        _lib.check(rc, "fe_diagonal")
        return out

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan:
            try:
                self._lib.fe_plan_destroy(plan)
            except Exception:
                pass
            self._plan = None


def compile_and_load(unit: PlanUnit, toolchain=None) -> GpuKernelHandle:
    """Create the sm_100a plan for ``unit`` (reference ``jit.py:90-111``).
    ``toolchain`` is accepted for signature compatibility and ignored: the
    kernels are compiled ahead of time by ``make``."""
    return GpuKernelHandle(unit)


def _is_cuda(a) -> bool:
    return getattr(a, "is_cuda", False) is True


def _host(a, dtype, name):
    a = np.asarray(a)
    if a.dtype != dtype:
        raise TypeError(f"binding {name!r} has dtype {a.dtype}, expected {np.dtype(dtype)}")
    if not a.flags.c_contiguous:
        a = np.ascontiguousarray(a)
    return a.ravel()
