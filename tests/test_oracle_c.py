"""The C restatement of the reference loop (oracle/fe_oracle.c) agrees with
the numpy oracle, single- and multi-threaded (it is the timed CPU baseline)."""

import numpy as np
import pytest

from oracle import fe_oracle as fo
from oracle import fe_oracle_c as foc
from paper_1903_08243_b200 import configs as C


@pytest.mark.parametrize("name,n", [("C1", 6), ("C2-P1", 3), ("C2-P3", 2), ("C3-Q2", 3),
                                    ("C4-quad-Q2", 5), ("C4-hex-Q1", 3), ("C5", 2), ("C6", 2)])
@pytest.mark.parametrize("threads", [1, 4])
def test_c_oracle_matches_numpy_oracle(name, n, threads):
    prob = C.build_problem(C.get_config(name, n), seed=3)
    P = fo.Problem(prob.spec.form, prob.spec.cell.kind, prob.spec.element.degree,
                   prob.rule.exactness_degree, prob.spec.params)
    args = (P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u, prob.mu, prob.lam)
    st = prob.state
    ref = fo.assemble(*args, state=st)
    got = foc.assemble(*args, threads=threads, state=st)
    assert fo.rel_l2(got, ref) <= 1e-13
    sub = foc.assemble(*args, start=1, end=prob.mesh.ncells - 2, threads=threads, state=st)
    assert fo.rel_l2(sub, fo.assemble(*args, start=1, end=prob.mesh.ncells - 2, state=st)) <= 1e-13


def test_c_oracle_matches_reference_golden(golden2d):
    for name in golden2d["names"]:
        form, cell, deg = str(name).split("_")
        g = lambda k: golden2d[f"{name}/{k}"]
        P = fo.Problem(form, cell, int(deg))
        y = foc.assemble(P, g("coords"), g("cell2vert"), g("cell2dof"), g("u"))
        assert fo.rel_l2(y, g("y")) <= 1e-13, name
