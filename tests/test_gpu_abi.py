"""The C ABI called directly, the way a reference-side ctypes binding would
call wrap_<form> (codegen.py:375-394, jit.py:71-87): the mesh arrives with
every call, no sizes, no explicit bind.  fe_wrap / fe_wrap_host must (re-)bind
the mesh from the buffers they are given (include/fe_b200.h), reject an
out-of-range [start, end) before queueing any copy, and leave dat0 untouched
on error."""

import ctypes
import math

import numpy as np
import pytest

import paper_1903_08243_b200 as fe
from paper_1903_08243_b200 import _lib
from paper_1903_08243_b200 import configs as C
from oracle import fe_oracle as fo

pytestmark = pytest.mark.gpu
TOL = 1e-12
vp = ctypes.c_void_p


def _problem(name, n, seed):
    return C.build_problem(C.get_config(name, n), seed)


def _oracle(prob):
    P = fo.Problem(prob.spec.form, prob.spec.cell.kind, prob.spec.element.degree,
                   prob.rule.exactness_degree, prob.spec.params)
    return fo.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u,
                       prob.mu, prob.lam, state=prob.state)


def _host_arrays(prob):
    return dict(dat1=np.ascontiguousarray(prob.mesh.coords, np.float64).ravel(),
                dat2=np.ascontiguousarray(prob.u),
                map0=np.ascontiguousarray(prob.dofmap.cell2dof, np.int32).ravel(),
                map1=np.ascontiguousarray(prob.mesh.cell2vert, np.int32).ravel(),
                dat3=None if prob.mu is None else np.ascontiguousarray(prob.mu),
                dat4=None if prob.lam is None else np.ascontiguousarray(prob.lam))


def _p(a):
    return None if a is None else vp(a.ctypes.data)


@pytest.mark.parametrize("name,n1,n2", [("C2-P2", 3, 4), ("C4-quad-Q2", 5, 7), ("C3-Q3", 2, 3)])
def test_fe_wrap_host_rebinds_a_second_mesh(name, n1, n2):
    lib = _lib.load()
    h = fe.compile_and_load(fe.emit_for(_problem(name, n1, 0).spec, fe.Target(),
                                        _problem(name, n1, 0).rule))
    for n, seed in ((n1, 1), (n2, 2), (n1, 3)):      # new buffers every call
        prob = _problem(name, n, seed)
        a = _host_arrays(prob)
        out = np.zeros(prob.ndofs)
        rc = lib.fe_wrap_host(h._plan, 0, prob.mesh.ncells, _p(out), _p(a["dat1"]), _p(a["dat2"]),
                              _p(a["dat3"]), _p(a["dat4"]), _p(a["map0"]), _p(a["map1"]))
        assert rc == 0, lib.fe_last_error()
        assert fo.rel_l2(out, _oracle(prob)) <= TOL, (name, n)
        assert h.info["ncells"] == prob.mesh.ncells


def test_fe_wrap_device_rebinds_a_second_mesh():
    import torch
    lib = _lib.load()
    p1 = _problem("C2-P3", 3, 0)
    h = fe.compile_and_load(fe.emit_for(p1.spec, fe.Target(), p1.rule))
    for n, seed in ((3, 0), (4, 5)):
        prob = _problem("C2-P3", n, seed)
        d = {k: (None if v is None else torch.as_tensor(v, device="cuda"))
             for k, v in _host_arrays(prob).items()}
        out = torch.zeros(prob.ndofs, dtype=torch.float64, device="cuda")
        t = lambda x: None if x is None else vp(x.data_ptr())
        rc = lib.fe_wrap(h._plan, 0, prob.mesh.ncells, t(out), t(d["dat1"]), t(d["dat2"]), None, None,
                         t(d["map0"]), t(d["map1"]), vp(torch.cuda.current_stream().cuda_stream))
        assert rc == 0, lib.fe_last_error()
        torch.cuda.synchronize()
        assert fo.rel_l2(out.cpu().numpy(), _oracle(prob)) <= TOL


def test_fe_wrap_host_implicit_bind_grows_with_end():
    """An implicitly bound mesh covers [0, end) of the call that bound it; a
    later call with the same buffers and a larger end re-binds."""
    lib = _lib.load()
    prob = _problem("C2-P2", 3, 0)
    h = fe.compile_and_load(fe.emit_for(prob.spec, fe.Target(), prob.rule))
    a = _host_arrays(prob)
    out = np.zeros(prob.ndofs)
    half = prob.mesh.ncells // 2
    args = lambda s, e: (h._plan, s, e, _p(out), _p(a["dat1"]), _p(a["dat2"]), None, None,
                         _p(a["map0"]), _p(a["map1"]))
    assert lib.fe_wrap_host(*args(0, half)) == 0
    assert lib.fe_wrap_host(*args(half, prob.mesh.ncells)) == 0, lib.fe_last_error()
    assert fo.rel_l2(out, _oracle(prob)) <= TOL


@pytest.mark.parametrize("start,end", [(0, None), (-1, 4), (5, 4)])
def test_fe_wrap_host_rejects_bad_range_without_touching_dat0(start, end):
    lib = _lib.load()
    prob = _problem("C2-P2", 3, 0)
    h = fe.compile_and_load(fe.emit_for(prob.spec, fe.Target(), prob.rule))
    a = _host_arrays(prob)
    h.bind(a["dat1"], a["map0"], a["map1"], nglobal=prob.dofmap.ndofs_global)   # explicit bind
    end = prob.mesh.ncells + 1 if end is None else end
    out = np.full(prob.ndofs, 7.0)
    rc = lib.fe_wrap_host(h._plan, start, end, _p(out), _p(a["dat1"]), _p(a["dat2"]), None, None,
                          _p(a["map0"]), _p(a["map1"]))
    assert rc == 1   # FE_EINVAL
    assert b"range" in lib.fe_last_error()
    assert np.all(out == 7.0)
    # the numpy-binding path raises like the torch path does
    with pytest.raises(_lib.FeError):
        h(start, end, fe.make_bindings(prob.mesh, prob.dofmap, prob.u, out))


def test_concurrent_applies_on_one_plan_from_threads():
    """Parameter blocks are built per launch: two host threads applying one
    plan on disjoint outputs and different ranges give the serial result."""
    import threading
    import torch
    prob = _problem("C4-quad-Q1", 12, 0)
    h = fe.compile_and_load(fe.emit_for(prob.spec, fe.Target(), prob.rule))
    dev = lambda x: torch.as_tensor(x, device="cuda")
    h.bind(dev(np.asarray(prob.mesh.coords).ravel()), dev(np.asarray(prob.dofmap.cell2dof, np.int32).ravel()),
           dev(np.asarray(prob.mesh.cell2vert, np.int32).ravel()), nglobal=prob.dofmap.ndofs_global)
    u, coef = dev(prob.u), (dev(prob.mu), dev(prob.lam))
    nc = prob.mesh.ncells
    ys = [torch.zeros(prob.ndofs, dtype=torch.float64, device="cuda") for _ in range(2)]
    ranges = [(0, nc // 3), (nc // 3, nc)]

    def work(i):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(50):
                ys[i].zero_()
                h.apply(u, ys[i], *ranges[i], coef=coef)
        s.synchronize()

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    [t.start() for t in th]
    [t.join() for t in th]
    torch.cuda.synchronize()
    ref = _oracle(prob)
    assert fo.rel_l2((ys[0] + ys[1]).cpu().numpy(), ref) <= TOL


def test_fast_log_special_values():
    import torch
    lib = _lib.load()
    inf, nan = math.inf, math.nan
    x = np.array([1.0, 2.0, 0.5, 1e-300, 5e-324, 2.2250738585072014e-308 / 3, 1e308, inf, 0.0, -0.0,
                  -1.0, nan, 1.0000001, 0.9999999, 3.3, 0.1])
    xd = torch.as_tensor(x, device="cuda")
    yd = torch.empty_like(xd)
    assert lib.fe_eval_log(vp(xd.data_ptr()), vp(yd.data_ptr()), x.size, None) == 0
    torch.cuda.synchronize()
    y = yd.cpu().numpy()
    with np.errstate(divide="ignore", invalid="ignore"):
        ref = np.log(x)
    finite = np.isfinite(ref)
    assert np.all(np.abs(y[finite] - ref[finite]) <= 4e-16 * np.maximum(1.0, np.abs(ref[finite])))
    assert np.array_equal(np.isnan(y), np.isnan(ref))
    assert np.array_equal(y[np.isinf(ref)], ref[np.isinf(ref)])
