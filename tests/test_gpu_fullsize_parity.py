"""Every operator at its FULL BASELINE size against the C oracle, whole
vector (north star: relative L2 <= 1e-12 in FP64).

All 20 operators -- C1..C5 (19) and the C6 tangent -- on exactly the
problem bench.py times (the single-domain slab of the fixed mesh,
``build_slab(cfg, 0, 0, nz, nz)``), applied on the GPU through the C ABI
and compared with oracle/fe_oracle.c on every host core (the C restatement
of the reference cell loop, itself pinned to the reference's golden vectors
and the numpy oracle: tests/test_oracle_c.py).  The reference-numbered C1
mesh is compared with the reference's own full-size output in
tests/test_gpu_parity.py.
"""

import os

import numpy as np
import pytest

import paper_1903_08243_b200 as fe
from paper_1903_08243_b200 import configs as C
from paper_1903_08243_b200.distributed import build_slab
from oracle import fe_oracle as fo
from oracle import fe_oracle_c as foc

pytestmark = pytest.mark.gpu
TOL = 1e-12
ALL = (["C1"] + [f"C2-P{k}" for k in range(1, 5)] + [f"C3-Q{k}" for k in range(1, 7)]
       + [f"C4-quad-Q{k}" for k in range(1, 5)] + [f"C4-hex-Q{k}" for k in range(1, 4)] + ["C5", "C6"])


@pytest.mark.parametrize("name", ALL)
def test_full_size_operator_matches_c_oracle(name):
    import torch
    cfg = C.get_config(name)
    prob = build_slab(cfg, 0, 0, cfg.n[-1], cfg.n[-1])
    h = fe.compile_and_load(fe.emit_for(prob.spec, fe.Target(), prob.rule))
    dev = torch.device("cuda")
    h.bind(torch.tensor(np.asarray(prob.mesh.coords).ravel(), device=dev),
           torch.tensor(np.asarray(prob.dofmap.cell2dof, np.int32).ravel(), device=dev),
           torch.tensor(np.asarray(prob.mesh.cell2vert, np.int32).ravel(), device=dev),
           nglobal=prob.dofmap.ndofs_global)
    coef = None
    if prob.coef() is not None:
        coef = tuple(None if c is None else torch.tensor(c, device=dev) for c in prob.coef())
    u = torch.tensor(prob.u, device=dev)
    y = torch.full_like(u, 3.0)                      # overwrite: the fill must not survive
    h.apply(u, y, coef=coef, overwrite=True)
    torch.cuda.synchronize()
    got = y.cpu().numpy()
    P = fo.Problem(prob.spec.form, prob.spec.cell.kind, prob.spec.element.degree,
                   prob.rule.exactness_degree, prob.spec.params)
    ref = foc.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u,
                       prob.mu, prob.lam, threads=len(os.sched_getaffinity(0)), state=prob.state)
    err = fo.rel_l2(got, ref)
    print(f"{name}: kernel={h.info['kernel']} cells={prob.mesh.ncells} dofs={prob.ndofs} rel_l2={err:.3e}")
    assert err <= TOL, (name, h.info["kernel"], err)
    assert fe.harness.rel_err(got, ref) <= TOL                      # the reference's own metric too
