"""The multi-GPU data path on one GPU: several z-slabs of one global mesh,
each applied by its own sm_100a plan on its slab-local numbering, interface
planes summed in process (exchange_loopback: the same arithmetic the NCCL
path does between ranks) -- equals the single-domain oracle."""

import numpy as np
import pytest

import paper_1903_08243_b200 as fe
from paper_1903_08243_b200 import configs as C
from paper_1903_08243_b200.distributed import build_slab, exchange_loopback, global_dof_index, slab_range
from oracle import fe_oracle as fo

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,world,nz,split", [
    ("C2-P2", 2, 2, False), ("C2-P4", 3, 2, False), ("C3-Q3", 2, 2, False), ("C4-hex-Q2", 2, 2, False),
    ("C5", 4, 2, False),
    # the overlapped order of DistributedOperator: boundary layers, then interior
    ("C2-P3", 3, 3, True), ("C3-Q2", 2, 4, True), ("C4-hex-Q1", 2, 3, True),
    # boundary-first cell order (bench.py at N > 1): both boundary layers in one range
    ("C5", 2, 4, "bfirst"), ("C3-Q3", 2, 3, "bfirst"), ("C4-hex-Q2", 2, 4, "bfirst")])
def test_slabs_on_gpu_equal_single_domain(name, world, nz, split):
    import torch
    cfg = C.get_config(name, (3, 2, nz))
    dev = torch.device("cuda")
    ys, slabs = [], []
    for r in range(world):
        z0, z1, nzg = slab_range(r, world, nz)
        s = build_slab(cfg, 9, z0, z1, nzg, boundary_first=(split == "bfirst"))
        h = fe.compile_and_load(fe.emit_for(s.spec, fe.Target(), s.rule))
        h.bind(torch.tensor(np.asarray(s.mesh.coords).ravel(), device=dev),
               torch.tensor(np.asarray(s.dofmap.cell2dof, np.int32).ravel(), device=dev),
               torch.tensor(np.asarray(s.mesh.cell2vert, np.int32).ravel(), device=dev),
               nglobal=s.dofmap.ndofs_global)
        u = torch.tensor(s.u, device=dev)
        y = torch.zeros_like(u)
        coef = None if s.mu is None else (torch.tensor(s.mu, device=dev), torch.tensor(s.lam, device=dev))
        if split == "bfirst":
            nc = s.mesh.ncells
            lc = nc // nz
            h.apply(u, y, 0, 2 * lc, coef=coef, overwrite=True)
            h.apply(u, y, 2 * lc, nc, coef=coef)
        elif split:
            nc = s.mesh.ncells
            lc = nc // nz
            h.apply(u, y, 0, lc, coef=coef, overwrite=True)
            h.apply(u, y, nc - lc, nc, coef=coef)
            h.apply(u, y, lc, nc - lc, coef=coef)
        else:
            h.apply(u, y, coef=coef, overwrite=True)
        ys.append(y)
        slabs.append(s)
    exchange_loopback(ys, slabs)
    torch.cuda.synchronize()
    glob = build_slab(cfg, 9, 0, nz * world, nz * world)
    P = fo.Problem(glob.spec.form, glob.spec.cell.kind, glob.spec.element.degree,
                   glob.rule.exactness_degree, glob.spec.params)
    yg = fo.assemble(P, glob.mesh.coords, glob.mesh.cell2vert, glob.dofmap.cell2dof, glob.u,
                     glob.mu, glob.lam)
    for s, y in zip(slabs, ys):
        y = y.cpu().numpy()
        assert fo.rel_l2(y, yg[global_dof_index(s)]) <= 1e-12
