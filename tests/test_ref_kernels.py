"""The reference's own generated C (oracle/_ref, built from /root/reference by
oracle/build_ref.py) agrees with the golden vectors and the oracles; it is the
CPU baseline of the reference-supported configs."""

import numpy as np
import pytest

from oracle import fe_oracle as fo
from oracle import ref_c
from paper_1903_08243_b200 import configs as C
import paper_1903_08243_b200 as fe

pytestmark = pytest.mark.skipif(not ref_c.manifest(), reason="oracle/_ref not built")


def test_reference_c1_kernel_matches_golden(golden_c1):
    prob = C.build_problem(C.get_config("C1"), 0)
    for target in ("scalar", "vector-ext"):
        k = ref_c.RefKernel("mass", "tri", 2, target)
        out = np.zeros(prob.ndofs)
        b = fe.make_bindings(prob.mesh, prob.dofmap, prob.u, out)
        k(0, prob.mesh.ncells, b)
        assert fo.rel_l2(out, golden_c1["y"]) <= 1e-14
        y = k.run_threads(prob.mesh.ncells, b, 4)
        assert fo.rel_l2(y, golden_c1["y"]) <= 1e-14


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_reference_elasticity_is_lame_with_half_zero(k):
    prob = C.build_problem(C.get_config(f"C4-quad-Q{k}", 6), 0)
    ker = ref_c.RefKernel("elasticity", "quad", k)
    out = np.zeros(prob.ndofs)
    ker(0, prob.mesh.ncells, fe.make_bindings(prob.mesh, prob.dofmap, prob.u, out))
    P = fo.Problem("elasticity_lame", "quadrilateral", k)
    nv = prob.mesh.nvertices
    ref = fo.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u,
                      np.full(nv, 0.5), np.zeros(nv))
    assert fo.rel_l2(out, ref) <= 1e-12
