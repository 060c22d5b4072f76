"""Matrix-free CG driver on CPU: the generic iteration
against a dense solve, and the slab-partitioned CG over gloo (world 2)
against the single-domain run with the oracle as the local operator."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1903_08243_b200 import configs as C
from paper_1903_08243_b200.distributed import DistributedOperator, build_slab, slab_range
from paper_1903_08243_b200.solver import SlabDot, cg
from oracle import fe_oracle as fo


def test_cg_matches_dense_solve():
    rng = np.random.default_rng(0)
    M = rng.standard_normal((40, 40))
    A = torch.tensor(M @ M.T + 40 * np.eye(40))
    b = torch.tensor(rng.standard_normal(40))
    x, info = cg(lambda u, y: y.copy_(A @ u), b, rtol=1e-13, maxiter=200)
    assert info.converged
    assert torch.allclose(x, torch.linalg.solve(A, b), rtol=0, atol=1e-11)
    # Jacobi (tensor) and callable preconditioners converge to the same x
    d = torch.diagonal(A)
    xj, ij = cg(lambda u, y: y.copy_(A @ u), b, rtol=1e-13, precond=1.0 / d)
    xc, ic = cg(lambda u, y: y.copy_(A @ u), b, rtol=1e-13, precond=lambda r: r / d)
    assert ij.converged and ic.converged and ij.iterations == ic.iterations
    assert torch.allclose(xj, x, atol=1e-11)


def _oracle_apply(slab):
    P = fo.Problem(slab.spec.form, slab.spec.cell.kind, slab.spec.element.degree,
                   slab.rule.exactness_degree, slab.spec.params)

    def apply(u, y):
        y.copy_(torch.from_numpy(fo.assemble(P, slab.mesh.coords, slab.mesh.cell2vert,
                                             slab.dofmap.cell2dof, u.numpy(), slab.mu, slab.lam,
                                             state=slab.state)))
    return apply


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _solve(slab, rank, world):
    op = DistributedOperator(slab, _oracle_apply(slab), rank, world)
    u_exact = torch.from_numpy(slab.u.copy())
    b = torch.zeros_like(u_exact)
    op.apply(u_exact, b)
    x, info = cg(op.apply, b, rtol=1e-12, maxiter=500, dot=SlabDot(slab, rank, world))
    return x, info, u_exact


def _worker(rank, world, port, name, nz, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    z0, z1, nzg = slab_range(rank, world, nz)
    slab = build_slab(C.get_config(name, (3, 2, nz)), 5, z0, z1, nzg)
    x, info, u_exact = _solve(slab, rank, world)
    q.put((rank, info.iterations, info.converged, float((x - u_exact).abs().max())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["C2-P1", "C2-P2"])
def test_distributed_cg_equals_single_domain(name):
    world, nz = 2, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, nz, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    glob = build_slab(C.get_config(name, (3, 2, nz * world)), 5, 0, nz * world, nz * world)
    _, info1, _ = _solve(glob, 0, 1)
    for rank, its, conv, err in res:
        assert conv and err < 1e-8, (rank, err)
        assert abs(its - info1.iterations) <= 1, (its, info1.iterations)   # same Krylov sequence


def _node_coords(slab):
    """Physical position of every scalar dof (affine simplices: the nodes'
    reference coordinates mapped by each cell's vertices)."""
    X = slab.mesh.coords[slab.mesh.cell2vert]                       # [c][4][3]
    ref = np.array(slab.spec.element.nodes, float)                   # [nd][3]
    pts = X[:, None, 0, :] + np.einsum("ia,cad->cid", ref, X[:, 1:, :] - X[:, None, 0, :])
    out = np.empty((slab.dofmap.ndofs_global, 3))
    out[np.asarray(slab.dofmap.cell2dof).ravel()] = pts.reshape(-1, 3)
    return out


def newton_problem(n=2):
    """Neo-Hookean P2 on the C5 mesh family, Dirichlet data u = A x on the
    cube's boundary: the homogeneous deformation x -> (I + A) x is an exact
    equilibrium (no body force) and P2 interpolates it exactly, so Newton
    must land on u = A x at every node."""
    cfg = C.get_config("C5", (n, n, n))
    s = build_slab(cfg, 0, 0, n, n)
    xyz = _node_coords(s)
    A = np.array([[0.02, -0.01, 0.005], [0.01, 0.03, -0.02], [-0.015, 0.0, 0.01]])
    exact = (xyz @ A.T).ravel()
    on_bnd = np.any((np.abs(xyz) < 1e-12) | (np.abs(xyz - 1.0) < 1e-12), axis=1)
    free = np.repeat(~on_bnd, 3).astype(float)
    return s, exact, free


def test_newton_recovers_homogeneous_deformation():
    from paper_1903_08243_b200.solver import newton
    s, exact, free = newton_problem(2)
    Pr = fo.Problem("neohookean", "tetrahedron", 2, 4)
    Pt = fo.Problem("neohookean_tangent", "tetrahedron", 2, 4)
    geo = (s.mesh.coords, s.mesh.cell2vert, s.dofmap.cell2dof)

    def residual(u, r):
        r.copy_(torch.from_numpy(fo.assemble(Pr, *geo, u.numpy())))

    def tangent(u0):
        st = u0.numpy().copy()
        return lambda du, y: y.copy_(torch.from_numpy(fo.assemble(Pt, *geo, du.numpy(), state=st)))

    u = torch.from_numpy(exact * (1.0 - free))          # boundary data, interior 0
    u, info = newton(residual, tangent, u, free=torch.from_numpy(free), rtol=1e-13, maxiter=8)
    assert info.converged, info.residuals
    assert info.iterations <= 5
    # quadratic convergence: each step squares the (relative) residual
    rel = np.array(info.residuals) / info.residuals[0]
    assert rel[2] <= 10 * rel[1] ** 2 + 1e-14
    assert np.abs(u.numpy() - exact).max() <= 1e-12
