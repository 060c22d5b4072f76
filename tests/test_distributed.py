"""Multi-rank element partition + halo sums on CPU (gloo, world_size 2 and 3).

The local slab action is the CPU oracle here (the GPU path plugs the sm_100a
plan into the same DistributedOperator); the test checks the partition
logic, slab-local numbering, seeded per-plane inputs and the interface
exchange: gathered distributed y == single-domain y (reference
test_reference.py:72-89 partition independence, SURVEY.md 8e parity)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1903_08243_b200 import configs as C
from paper_1903_08243_b200.distributed import (DistributedOperator, build_slab, global_dof_index,
                                               slab_range, slab_split)
from oracle import fe_oracle as fo


def _oracle_apply(slab):
    P = fo.Problem(slab.spec.form, slab.spec.cell.kind, slab.spec.element.degree,
                   slab.rule.exactness_degree, slab.spec.params)

    def apply(u, y):
        y.copy_(torch.from_numpy(fo.assemble(P, slab.mesh.coords, slab.mesh.cell2vert,
                                             slab.dofmap.cell2dof, u.numpy(), slab.mu, slab.lam,
                                             state=slab.state)))

    def range_apply(u, y, start, end, overwrite):
        part = torch.from_numpy(fo.assemble(P, slab.mesh.coords, slab.mesh.cell2vert,
                                            slab.dofmap.cell2dof, u.numpy(), slab.mu, slab.lam,
                                            start, end, state=slab.state))
        if overwrite:
            y.copy_(part)
        else:
            y += part
    return apply, range_apply


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, nz, q, overlap=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = C.get_config(name, (3, 2, nz))
    z0, z1, nzg = slab_range(rank, world, nz)
    slab = build_slab(cfg, 11, z0, z1, nzg)
    apply, range_apply = _oracle_apply(slab)
    op = DistributedOperator(slab, apply, rank, world, range_apply if overlap else None)
    u = torch.from_numpy(slab.u.copy())
    y = torch.zeros_like(u)
    op.apply(u, y)
    st = None if slab.state is None else slab.state.copy()
    q.put((rank, global_dof_index(slab), y.numpy().copy(), slab.u.copy(), st))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world,nz,overlap", [
    ("C2-P2", 2, 2, False), ("C5", 2, 2, False), ("C3-Q2", 3, 2, False), ("C4-hex-Q1", 2, 2, False),
    # boundary layers first, exchange overlapping the interior layers
    ("C2-P2", 3, 3, True), ("C4-hex-Q1", 2, 4, True), ("C6", 2, 2, True)])
def test_distributed_equals_single_domain(name, world, nz, overlap):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, nz, q, overlap))
             for r in range(world)]
    for p in procs:
        p.start()
    results = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = C.get_config(name, (3, 2, nz))
    glob = build_slab(cfg, 11, 0, nz * world, nz * world)
    P = fo.Problem(glob.spec.form, glob.spec.cell.kind, glob.spec.element.degree,
                   glob.rule.exactness_degree, glob.spec.params)
    y_glob = fo.assemble(P, glob.mesh.coords, glob.mesh.cell2vert, glob.dofmap.cell2dof, glob.u,
                         glob.mu, glob.lam, state=glob.state)
    for rank, idx, y, u, st in results:
        assert np.array_equal(u, glob.u[idx])                       # consistent inputs
        if glob.state is not None:                                  # (and state planes)
            assert np.array_equal(st, glob.state[idx])
        assert fo.rel_l2(y, y_glob[idx]) <= 1e-14, rank


def _strong_worker(rank, world, port, name, n, q, boundary_first=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = C.get_config(name, n)
    z0, z1, nzg = slab_split(rank, world, cfg.n[-1])
    slab = build_slab(cfg, 5, z0, z1, nzg, boundary_first=boundary_first)
    apply, range_apply = _oracle_apply(slab)
    op = DistributedOperator(slab, apply, rank, world, range_apply)
    u = torch.from_numpy(slab.u.copy())
    y = torch.zeros_like(u)
    op.apply(u, y)
    q.put((rank, global_dof_index(slab), y.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world,n,bfirst", [
    # strong scaling: ONE fixed mesh split into world slabs (bench.py --gpus N)
    ("C5", 2, (2, 2, 6), False), ("C2-P3", 2, (2, 2, 5), False), ("C3-Q2", 3, (2, 3, 7), False),
    ("C1", 2, (4, 6), False), ("C4-quad-Q2", 3, (3, 7), False), ("C4-hex-Q1", 2, (2, 2, 4), False),
    # the cell order bench.py uses at N > 1: both boundary layers first (one launch)
    ("C5", 2, (2, 2, 8), True), ("C3-Q2", 3, (2, 3, 10), True), ("C4-quad-Q2", 2, (3, 8), True)])
def test_strong_split_equals_single_domain(name, world, n, bfirst):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_strong_worker, args=(r, world, port, name, n, q, bfirst)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = C.get_config(name, n)
    glob = build_slab(cfg, 5, 0, cfg.n[-1], cfg.n[-1])
    P = fo.Problem(glob.spec.form, glob.spec.cell.kind, glob.spec.element.degree,
                   glob.rule.exactness_degree, glob.spec.params)
    y_glob = fo.assemble(P, glob.mesh.coords, glob.mesh.cell2vert, glob.dofmap.cell2dof, glob.u,
                         glob.mu, glob.lam, state=glob.state)
    covered = np.zeros(y_glob.size, bool)
    for rank, idx, y in results:
        assert fo.rel_l2(y, y_glob[idx]) <= 1e-14, rank
        covered[idx] = True
    assert covered.all()


@pytest.mark.parametrize("name,n", [("C1", (3, 4)), ("C4-quad-Q3", (2, 3)), ("C4-quad-Q1", (4, 4))])
def test_2d_slab_is_a_valid_mesh(name, n):
    """2D slabs (rows of squares): positive orientation, conforming lattice
    numbering (every lattice node used, shared nodes agree), and the
    single-slab operator equals the oracle on the reference-built mesh up to
    the node permutation when there is no jitter."""
    cfg = C.get_config(name, n)
    s = build_slab(cfg, 0, 0, n[-1], n[-1])
    X = s.mesh.coords[s.mesh.cell2vert]
    if cfg.cell == "triangle":
        det = np.linalg.det(X[:, 1:] - X[:, :1])
    else:
        det = np.linalg.det(np.stack([X[:, 1] - X[:, 0], X[:, 2] - X[:, 0]], axis=1))
    assert (det > 0).all()
    assert s.mesh.ncells == cfg.ncells
    k = s.spec.element.degree
    assert s.dofmap.ndofs_global == (k * n[0] + 1) * (k * n[1] + 1)
    assert np.unique(s.dofmap.cell2dof).size == s.dofmap.ndofs_global
    # the lattice node of each local dof sits at the mapped physical point (unjittered copy)
    import dataclasses
    flat = build_slab(dataclasses.replace(cfg, jitter=False), 0, 0, n[-1], n[-1])
    from paper_1903_08243_b200.distributed import vertex_first_ids
    Lx, Ly = k * n[0] + 1, k * n[1] + 1
    J, I = np.meshgrid(np.arange(Ly), np.arange(Lx), indexing="ij")
    pts = np.stack([I.ravel(), J.ravel()], axis=-1)
    ids = vertex_first_ids(pts, n, k)
    assert np.array_equal(np.sort(ids), np.arange(Lx * Ly))          # a permutation of the lattice
    lat = np.empty((Lx * Ly, 2), np.int64)
    lat[ids] = pts
    d = flat.dofmap.cell2dof
    gx, gy = lat[d, 0] / (k * n[0]), lat[d, 1] / (k * n[1])
    assert np.array_equal(d[:, :flat.spec.cell.nvertices], flat.mesh.cell2vert)   # vertex dofs first
    nodes = np.asarray(flat.spec.element.nodes)
    Xc = flat.mesh.coords[flat.mesh.cell2vert]
    if cfg.cell == "triangle":
        phys = Xc[:, None, 0, :] + np.einsum("ia,cad->cid", nodes, Xc[:, 1:, :] - Xc[:, None, 0, :])
    else:
        phys = Xc[:, None, 0, :] + nodes[None, :, :] * (Xc[:, None, 3, :] - Xc[:, None, 0, :])
    assert np.allclose(phys[..., 0], gx) and np.allclose(phys[..., 1], gy)


def test_slab_split_is_balanced_and_covers():
    for nz, world in ((128, 8), (64, 3), (7, 7), (256, 4)):
        parts = [slab_split(r, world, nz) for r in range(world)]
        assert parts[0][0] == 0 and parts[-1][1] == nz
        assert all(a[1] == b[0] for a, b in zip(parts[:-1], parts[1:]))
        sizes = [p[1] - p[0] for p in parts]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        slab_split(0, 9, 8)


def test_slab_of_whole_mesh_matches_config_shape():
    cfg = C.get_config("C2-P1", (4, 4, 4))
    s = build_slab(cfg, 0, 0, 4, 4)
    assert s.mesh.ncells == cfg.ncells
    assert s.dofmap.ndofs_global == 5 ** 3
    # positive orientation everywhere
    X = s.mesh.coords[s.mesh.cell2vert]
    det = np.linalg.det(X[:, 1:] - X[:, :1])
    assert (det > 0).all()


def test_loopback_exchange_matches_distributed_semantics():
    """Three slabs in one process: after exchange_loopback both copies of
    every interface node hold the sum, every other entry is untouched."""
    from paper_1903_08243_b200.distributed import exchange_loopback
    cfg = C.get_config("C2-P2", (2, 2, 3))
    slabs = [build_slab(cfg, 0, *slab_split(r, 3, 3)) for r in range(3)]
    ys = [torch.arange(s.ndofs, dtype=torch.float64) + 1000 * r for r, s in enumerate(slabs)]
    before = [y.clone() for y in ys]
    exchange_loopback(ys, slabs)
    for r, (s, y, y0) in enumerate(zip(slabs, ys, before)):
        touched = np.zeros(s.ndofs, bool)
        for side, nb in (("below", r - 1), ("above", r + 1)):
            if not 0 <= nb < 3:
                continue
            other = "above" if side == "below" else "below"
            for (a, b), (c, d) in zip(s.interface_ranges(side), slabs[nb].interface_ranges(other)):
                assert torch.equal(y[a:b], y0[a:b] + before[nb][c:d])
                touched[a:b] = True
        assert torch.equal(y[~torch.from_numpy(touched)], y0[~torch.from_numpy(touched)])
    # interface nodes sit at the same physical points on both sides
    for lo, hi in zip(slabs[:-1], slabs[1:]):
        for (a, b), (c, d) in zip(lo.interface_ranges("above"), hi.interface_ranges("below")):
            assert np.array_equal(lo.global_index[a:b], hi.global_index[c:d])
