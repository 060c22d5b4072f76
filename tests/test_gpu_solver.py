"""Operator diagonal (fe_diagonal) and the matrix-free CG driver on the
B200."""

import numpy as np
import pytest

import paper_1903_08243_b200 as fe
from paper_1903_08243_b200 import configs as C
from paper_1903_08243_b200.solver import cg, jacobi
from oracle import fe_oracle as fo

pytestmark = pytest.mark.gpu


def _bound(prob):
    import torch
    h = fe.compile_and_load(fe.emit_for(prob.spec, fe.Target(), prob.rule))
    dev = torch.device("cuda")
    h.bind(torch.tensor(np.asarray(prob.mesh.coords).ravel(), device=dev),
           torch.tensor(np.asarray(prob.dofmap.cell2dof, np.int32).ravel(), device=dev),
           torch.tensor(np.asarray(prob.mesh.cell2vert, np.int32).ravel(), device=dev),
           nglobal=prob.dofmap.ndofs_global)
    coef = None
    if prob.coef() is not None:
        coef = tuple(None if c is None else torch.tensor(c, device=dev) for c in prob.coef())
    return h, coef


def _oracle_diagonal(prob):
    """diag(A) column by column through the oracle (small meshes only)."""
    P = fo.Problem(prob.spec.form, prob.spec.cell.kind, prob.spec.element.degree,
                   prob.rule.exactness_degree, prob.spec.params)
    n = prob.ndofs
    d = np.empty(n)
    for i in range(n):
        e = np.zeros(n)
        e[i] = 1.0
        d[i] = fo.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, e,
                           prob.mu, prob.lam, state=prob.state)[i]
    return d


@pytest.mark.parametrize("name,n", [("C2-P2", 2), ("C2-P3", 1), ("C4-hex-Q1", 2),
                                    ("C3-Q2", 2), ("C6", 1)])
def test_diagonal_matches_oracle(name, n):
    prob = C.build_problem(C.get_config(name, n), seed=3)
    h, coef = _bound(prob)
    d = h.diagonal(coef=coef).cpu().numpy()
    assert fo.rel_l2(d, _oracle_diagonal(prob)) <= 1e-12


def test_diagonal_of_the_residual_is_rejected():
    prob = C.build_problem(C.get_config("C5", 1), seed=3)
    h, coef = _bound(prob)
    with pytest.raises(fe.KernelError):
        h.diagonal(coef=coef)


@pytest.mark.parametrize("name,n,precond", [("C2-P2", 6, True), ("C2-P2", 6, False),
                                            ("C4-hex-Q1", 4, True)])
def test_cg_recovers_manufactured_solution(name, n, precond):
    import torch
    prob = C.build_problem(C.get_config(name, n), seed=4)
    h, coef = _bound(prob)
    A = lambda u, y: h.apply(u, y, coef=coef, overwrite=True)
    u = torch.tensor(prob.u, device="cuda")
    b = torch.empty_like(u)
    A(u, b)
    if prob.spec.form == "elasticity_lame":
        # pure-traction elasticity is singular (rigid modes): shift by the mass-like identity
        A0 = A
        A = lambda v, y: (A0(v, y), y.add_(1e-3 * v))
        b.add_(1e-3 * u)
    M = jacobi(h.diagonal(coef=coef)) if precond else None
    x, info = cg(A, b, rtol=1e-12, maxiter=2000, precond=M)
    assert info.converged, info.residuals[-3:]
    assert float((x - u).abs().max()) <= 1e-7 * float(u.abs().max())


@pytest.mark.parametrize("n", [2, 8])
def test_gpu_newton_neohookean_residual_and_tangent(n):
    """Newton on the B200: the C5 residual kernel and the C6 tangent kernel
    inside solver.newton (CG per step), Dirichlet data u = A x on the cube
    boundary -> the exact homogeneous deformation at every node."""
    import torch
    from paper_1903_08243_b200.solver import newton
    from test_solver import newton_problem
    s, exact, free = newton_problem(n)
    dev = torch.device("cuda")
    hr = fe.compile_and_load(fe.emit_for(fe.operator_spec("neohookean", "tetrahedron", 2), fe.Target(), s.rule))
    ht = fe.compile_and_load(fe.emit_for(fe.operator_spec("neohookean_tangent", "tetrahedron", 2), fe.Target(),
                                         s.rule))
    mesh = (torch.tensor(np.asarray(s.mesh.coords).ravel(), device=dev),
            torch.tensor(np.asarray(s.dofmap.cell2dof, np.int32).ravel(), device=dev),
            torch.tensor(np.asarray(s.mesh.cell2vert, np.int32).ravel(), device=dev))
    for h in (hr, ht):
        h.bind(*mesh, nglobal=s.dofmap.ndofs_global)
    residual = lambda u, r: hr.apply(u, r, overwrite=True)
    tangent = lambda u0: (lambda du, y: ht.apply(du, y, coef=(u0, None), overwrite=True))
    fr = torch.tensor(free, device=dev)
    u = torch.tensor(exact * (1.0 - free), device=dev)
    u, info = newton(residual, tangent, u, free=fr, rtol=1e-12, maxiter=10, cg_rtol=1e-13)
    assert info.converged, info.residuals
    assert info.iterations <= 8
    rel = np.array(info.residuals) / info.residuals[0]
    assert rel[-1] <= 1e-12 and rel[-2] <= 1e-5          # quadratic tail
    assert float((u.cpu() - torch.tensor(exact)).abs().max()) <= 1e-11
