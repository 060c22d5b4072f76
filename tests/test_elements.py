"""Host-side element machinery that the kernels consume (no GPU)."""

import numpy as np
import pytest

from paper_1903_08243_b200.elements import (quadrature_rule, reference_element, stiffness_modes,
                                            tabulate)


@pytest.mark.parametrize("cell,k", [(c, k) for c in ("triangle", "tetrahedron") for k in (1, 2, 3, 4)])
def test_stiffness_modes_factor_the_reference_stiffness_tensor(cell, k):
    """S_ab = sum_r w_r G[r,:,a] G[r,:,b]^T with m = dim P_{k-1} modes: the
    modal split / modal DMMA kernels' tables reproduce every reference
    stiffness matrix the quadrature loop (kernels.py:205-220) integrates."""
    el = reference_element(cell, k)
    w, G = stiffness_modes(el)
    d = el.cell.dim
    m = {2: k * (k + 1) // 2, 3: k * (k + 1) * (k + 2) // 6}[d]
    assert G.shape == (m, el.ndof_scalar, d) and np.all(w == 1.0)
    rule = quadrature_rule(cell, 2 * k)   # any rule exact for the integrand
    g = tabulate(el, rule).grads
    S = np.einsum("q,qia,qjb->aibj", rule.weights, g, g)
    S2 = np.einsum("r,ria,rjb->aibj", w, G, G)
    assert np.abs(S - S2).max() <= 1e-13 * np.abs(S).max()


def test_stiffness_modes_reject_tensor_cells():
    with pytest.raises(ValueError):
        stiffness_modes(reference_element("hexahedron", 2))
