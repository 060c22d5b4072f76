"""The C-ABI boundary without a GPU: the library loads, exports every symbol
include/fe_b200.h declares, and rejects bad calls with the reference's error
behaviour (jit.py:71-87: KeyError for a missing binding, TypeError for a wrong
dtype) before any kernel is launched."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1903_08243_b200 import _lib
import paper_1903_08243_b200 as fe

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "fe_b200.h")).read()
    return sorted(set(re.findall(r"\b(fe_[a-z_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert set(syms) == set(_lib.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.fe_abi_version() == 1


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


def test_null_arguments_are_rejected():
    lib = _lib.load()
    assert lib.fe_plan_create(None, None, 0) == 1
    assert b"null" in lib.fe_last_error()
    assert lib.fe_apply(None, 0, 0, None, None, None, None, 0, None) == 1


def test_unsupported_degree_raises_at_construction():
    with pytest.raises(ValueError, match="degree"):
        fe.operator_spec("mass", "tri", 5)


def test_apply_without_mesh_is_an_error():
    spec = fe.operator_spec("mass", "tri", 2)
    h = fe.compile_and_load(fe.emit_for(spec))        # element-tensor plan: no device work yet
    assert h.info["kernel"].startswith("element_tensor")
    with pytest.raises(_lib.FeError, match="mesh"):
        h.apply(0, 0)


def test_binding_errors_mirror_reference():
    spec = fe.operator_spec("mass", "tri", 2)
    h = fe.compile_and_load(fe.emit_for(spec))
    mesh = fe.build_mesh("tri", 2, 2)
    dm = fe.build_dof_map(mesh, spec.element)
    u = np.ones(dm.ndofs_global)
    b = fe.make_bindings(mesh, dm, u, np.zeros_like(u))
    del b["map1"]
    with pytest.raises(KeyError, match="map1"):
        h(0, mesh.ncells, b)
    b = fe.make_bindings(mesh, dm, u, np.zeros_like(u))
    b["dat2"] = u.astype(np.float32)
    with pytest.raises(TypeError, match="dat2"):
        h(0, mesh.ncells, b)
    b = fe.make_bindings(mesh, dm, u, np.zeros((2, u.size))[:, 0])
    with pytest.raises(ValueError, match="dat0"):
        h(0, mesh.ncells, b)


def test_wrapper_argument_order_matches_reference():
    # codegen.py:375-394: start, end, dats in local-kernel order, then maps
    unit = fe.emit_for(fe.operator_spec("helmholtz", "tri", 1))
    assert [a[0] for a in unit.args] == ["start", "end", "dat0", "dat1", "dat2", "map0", "map1"]
    assert unit.entry == "wrap_helmholtz"
    unit = fe.emit_for(fe.operator_spec("elasticity_lame", "hex", 1))
    assert [a[0] for a in unit.args][2:7] == ["dat0", "dat1", "dat2", "dat3", "dat4"]


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1903_08243_b200")
    pat = re.compile(r"^\s*(from|import)\s+[\w.]*oracle", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                assert not pat.search(open(os.path.join(dirpath, f)).read()), f
