"""The SIMD-batched CPU port (oracle/fe_cpu_port.cpp: the paper's
cross-element vectorisation, the timed CPU baseline) equals the oracle on
every BASELINE operator -- ragged batch remainders, sub-ranges and several
thread counts included -- so the baseline computes the same operator."""

import numpy as np
import pytest

from oracle import fe_cpu_port as fcp
from oracle import fe_oracle as fo
from paper_1903_08243_b200 import configs as C
from paper_1903_08243_b200.distributed import build_slab

CASES = [("C1", (5, 3)), ("C2-P1", (3, 2, 2)), ("C2-P2", (2, 2, 3)), ("C2-P3", (2, 2, 2)),
         ("C2-P4", (2, 1, 2)), ("C3-Q1", (3, 2, 2)), ("C3-Q2", (2, 2, 2)), ("C3-Q3", (2, 2, 1)),
         ("C3-Q4", (2, 1, 1)), ("C3-Q5", (1, 2, 1)), ("C3-Q6", (1, 1, 2)),
         ("C4-quad-Q1", (5, 4)), ("C4-quad-Q2", (4, 3)), ("C4-quad-Q3", (3, 3)), ("C4-quad-Q4", (2, 3)),
         ("C4-hex-Q1", (3, 2, 2)), ("C4-hex-Q2", (2, 2, 1)), ("C4-hex-Q3", (1, 2, 1)),
         ("C5", (2, 2, 2)), ("C6", (2, 2, 2))]


@pytest.mark.parametrize("name,n", CASES)
@pytest.mark.parametrize("threads", [1, 3])
def test_cpu_port_matches_oracle(name, n, threads):
    cfg = C.get_config(name, n)
    s = build_slab(cfg, 4, 0, n[-1], n[-1])
    P = fo.Problem(s.spec.form, s.spec.cell.kind, s.spec.element.degree, s.rule.exactness_degree,
                   s.spec.params)
    assert fcp.supported(P)
    args = (P, s.mesh.coords, s.mesh.cell2vert, s.dofmap.cell2dof, s.u, s.mu, s.lam)
    nc = s.mesh.ncells
    for a, b in ((0, nc), (1, nc - 2), (3, 3 + min(nc - 3, 11))):
        ref = fo.assemble(*args, start=a, end=b, state=s.state)
        got = fcp.assemble(*args, start=a, end=b, threads=threads, state=s.state)
        assert fo.rel_l2(got, ref) <= 1e-13, (a, b, fo.rel_l2(got, ref))


def test_cpu_port_accumulates_and_rejects_unknown():
    cfg = C.get_config("C2-P2", (2, 2, 2))
    s = build_slab(cfg, 0, 0, 2, 2)
    P = fo.Problem(s.spec.form, s.spec.cell.kind, 2, s.rule.exactness_degree)
    args = (P, s.mesh.coords, s.mesh.cell2vert, s.dofmap.cell2dof, s.u)
    out = np.ones(s.ndofs)
    fcp.assemble(*args, out=out, threads=2)
    assert fo.rel_l2(out - 1.0, fo.assemble(*args)) <= 1e-13
    Q = fo.Problem("helmholtz", "tetrahedron", 2, 6)           # a rule the port does not specialise
    assert not fcp.supported(Q)
    with pytest.raises(ValueError):
        fcp.assemble(Q, s.mesh.coords, s.mesh.cell2vert, s.dofmap.cell2dof, s.u)
