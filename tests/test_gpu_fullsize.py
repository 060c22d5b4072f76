"""BASELINE configs at their full sizes, checked through size-independent
properties (the CPU oracle would take minutes there) plus a sub-range of
cells against the oracle:

* symmetry  v.(A u) = u.(A v) for the linear symmetric forms;
* linearity A(a u + b v) = a A u + b A v;
* constants / rigid motions in the kernel (gradient forms, elasticity,
  neo-Hookean translation invariance);
* the first cells of the full mesh against the oracle (parity at scale,
  64-bit address arithmetic exercised at 10^7 cells).
"""

import numpy as np
import pytest

import paper_1903_08243_b200 as fe
from paper_1903_08243_b200 import configs as C
from oracle import fe_oracle as fo

pytestmark = pytest.mark.gpu


def _setup(name):
    import torch
    prob = C.build_problem(C.get_config(name), seed=0)
    h = fe.compile_and_load(fe.emit_for(prob.spec, fe.Target(), prob.rule))
    dev = torch.device("cuda")
    h.bind(torch.tensor(np.asarray(prob.mesh.coords).ravel(), device=dev),
           torch.tensor(np.asarray(prob.dofmap.cell2dof, np.int32).ravel(), device=dev),
           torch.tensor(np.asarray(prob.mesh.cell2vert, np.int32).ravel(), device=dev),
           nglobal=prob.dofmap.ndofs_global)
    coef = None
    if prob.coef() is not None:
        coef = tuple(None if c is None else torch.tensor(c, device=dev) for c in prob.coef())

    def A(u):
        y = torch.zeros_like(u)
        h.apply(u, y, coef=coef, overwrite=True)
        return y
    return prob, h, A, dev, coef


def _subrange_parity(prob, h, dev, coef, ncheck=2048):
    import torch
    u = torch.tensor(prob.u, device=dev)
    y = torch.zeros_like(u)
    h.apply(u, y, 0, ncheck, coef=coef, overwrite=True)
    P = fo.Problem(prob.spec.form, prob.spec.cell.kind, prob.spec.element.degree,
                   prob.rule.exactness_degree, prob.spec.params)
    ref = fo.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u,
                      prob.mu, prob.lam, 0, ncheck, state=prob.state)
    return fo.rel_l2(y.cpu().numpy(), ref)


@pytest.mark.parametrize("name", ["C2-P4", "C3-Q3", "C3-Q6", "C4-quad-Q4", "C4-hex-Q3", "C6"])
def test_full_size_symmetry_linearity_and_parity(name):
    import torch
    prob, h, A, dev, coef = _setup(name)
    g = torch.Generator(device="cpu").manual_seed(1)
    u = torch.tensor(prob.u, device=dev)
    v = (torch.rand(u.numel(), generator=g, dtype=torch.float64) * 2 - 1).to(dev)
    Au, Av = A(u), A(v)
    vAu, uAv = float(v @ Au), float(u @ Av)
    scale = float(torch.linalg.norm(u) * torch.linalg.norm(Av))
    assert abs(vAu - uAv) <= 1e-12 * scale
    lin = A(2.5 * u - 0.75 * v)
    assert float(torch.linalg.norm(lin - (2.5 * Au - 0.75 * Av))) <= 1e-13 * float(torch.linalg.norm(lin))
    assert _subrange_parity(prob, h, dev, coef) <= 1e-12


@pytest.mark.parametrize("name", ["C3-Q6", "C2-P3"])
def test_full_size_constants(name):
    import torch
    prob, h, A, dev, coef = _setup(name)
    ones = torch.ones(prob.ndofs, dtype=torch.float64, device=dev)
    y = A(ones)
    if prob.spec.form == "laplacian_scalar":
        ref = float(torch.linalg.norm(A(torch.tensor(prob.u, device=dev))))
        assert float(torch.linalg.norm(y)) <= 1e-12 * ref
    else:
        # helmholtz: grad 1 = 0 leaves the mass term; sum = volume of the unit
        # cube.  The stiffness term cancels only to round-off of the (shared)
        # reference matrices' row sums, a SYSTEMATIC ~1e-15 |S| per cell that
        # adds up over 1.6M cells weighted by |K| ~ h: tolerance 1e-9.
        assert abs(float(y.sum()) - 1.0) <= 1e-9


def test_full_size_neohookean_translation_invariance_and_parity():
    import torch
    prob, h, A, dev, coef = _setup("C5")
    u = torch.tensor(prob.u, device=dev)
    shift = torch.tensor([1e-3, -2e-3, 0.5e-3], dtype=torch.float64, device=dev).repeat(prob.nglobal)
    r0, r1 = A(u), A(u + shift)
    assert float(torch.linalg.norm(r1 - r0)) <= 1e-11 * float(torch.linalg.norm(r0))
    assert _subrange_parity(prob, h, dev, coef) <= 1e-12
