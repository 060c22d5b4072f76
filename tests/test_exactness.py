"""Exactness pins for the 3D element machinery the headline operators run on.

* Quadrature: the collapsed GL x GJ(1,0) x GJ(2,0) tetrahedron rule and the
  GL^3 hexahedron rule -- both the product's (``elements.quadrature_rule``)
  and the oracle's (``oracle.fe_oracle.quadrature``) -- integrate every
  monomial up to the requested degree exactly (restating the reference's
  test_elements.py:104-118 for 3D, degrees 0..12; degree 8 is what C2-P4
  needs), with the exact integrals pinned against sympy (restating
  test_elements.py:135-145).
* Single-cell oracles (restating test_kernels.py:36-104 for the operators
  of the headline configs): helmholtz on tetrahedra P3 and P4, the scalar
  Laplacian on an affine hexahedron Q3 and Lame elasticity (Q1 mu/lambda
  fields) on an affine hexahedron Q2, each on a perturbed physical cell with
  rational coordinates.  The symbolic side shares nothing numerical with
  the oracle: the simplex basis is the closed-form barycentric Lagrange
  basis (no Vandermonde solve), the hexahedron basis a product of 1D
  Lagrange polynomials, and the integrals are exact rational sums of
  monomial integrals (affine cells: constant J, polynomial integrands).
"""

import math
from fractions import Fraction
from itertools import product

import numpy as np
import pytest
import sympy
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import fe_oracle as fo
from paper_1903_08243_b200 import configs as C
from paper_1903_08243_b200.elements import monomial_integral, quadrature_rule, reference_cell

X, Y, Z = sympy.symbols("X Y Z")


def _exact(kind, a, b, c):
    if kind == "tetrahedron":
        return Fraction(math.factorial(a) * math.factorial(b) * math.factorial(c),
                        math.factorial(a + b + c + 3))
    return Fraction(1, (a + 1) * (b + 1) * (c + 1))


def _monos(kind, d):
    if kind == "tetrahedron":
        return [(a, b, c) for a in range(d + 1) for b in range(d + 1 - a) for c in range(d + 1 - a - b)]
    return list(product(range(d + 1), repeat=3))


def _check_rule(kind, d, pts, wts):
    assert (np.asarray(wts) > 0).all()
    x, y, z = (np.asarray(pts)[:, i] for i in range(3))
    worst = 0.0
    for a, b, c in _monos(kind, d):
        approx = float((wts * x ** a * y ** b * z ** c).sum())
        exact = float(_exact(kind, a, b, c))
        worst = max(worst, abs(approx - exact) / exact)
    assert worst <= 1e-12, (kind, d, worst)


@pytest.mark.parametrize("kind", ["tetrahedron", "hexahedron"])
@pytest.mark.parametrize("d", range(0, 13))
def test_product_rule_is_exact(kind, d):
    r = quadrature_rule(kind, d)
    assert r.points.shape[1] == 3 and r.exactness_degree == d
    _check_rule(kind, d, r.points, r.weights)


@pytest.mark.parametrize("kind", ["tetrahedron", "hexahedron"])
@pytest.mark.parametrize("d", range(0, 13))
def test_oracle_rule_is_exact(kind, d):
    pts, wts = fo.quadrature(kind, d)
    _check_rule(kind, d, pts, wts)


@pytest.mark.parametrize("kind,d", [("tetrahedron", 13), ("tetrahedron", 15), ("hexahedron", 15)])
def test_rule_degree_is_not_overstated(kind, d):
    """n = (d+2)//2 points per direction: exact to 2n-1, and NOT beyond --
    a monomial of degree 2n (in the GL direction) is integrated inexactly,
    so the exactness claim above is not vacuous."""
    r = quadrature_rule(kind, d)
    n = (d + 2) // 2
    e = 2 * n
    x = r.points[:, 0]
    approx = float((r.weights * x ** e).sum())
    assert abs(approx - float(_exact(kind, e, 0, 0))) > 1e-10 * float(_exact(kind, e, 0, 0))


def test_weight_sums_are_cell_measures():
    for kind, vol in (("tetrahedron", 1 / 6), ("hexahedron", 1.0)):
        for d in (2, 4, 8, 12):
            assert math.isclose(quadrature_rule(kind, d).weights.sum(), vol, rel_tol=1e-14)
            assert math.isclose(fo.quadrature(kind, d)[1].sum(), vol, rel_tol=1e-14)


@given(a=st.integers(0, 5), b=st.integers(0, 5), c=st.integers(0, 5),
       kind=st.sampled_from(["tetrahedron", "hexahedron"]))
@settings(max_examples=30, deadline=None)
def test_monomial_integrals_match_sympy(a, b, c, kind):
    f = X ** a * Y ** b * Z ** c
    if kind == "tetrahedron":
        exact = sympy.integrate(f, (Z, 0, 1 - X - Y), (Y, 0, 1 - X), (X, 0, 1))
    else:
        exact = sympy.integrate(f, (Z, 0, 1), (Y, 0, 1), (X, 0, 1))
    want = Fraction(int(exact.p), int(exact.q))
    assert _exact(kind, a, b, c) == want
    assert monomial_integral(reference_cell(kind), (a, b, c)) == want


# ---------------------------------------------------------------------------
# exact single-cell residuals
# ---------------------------------------------------------------------------


def _poly(e):
    return sympy.Poly(e, X, Y, Z, domain="QQ")


def _integrate(p, kind):
    """Exact integral of a polynomial over the reference cell."""
    s = Fraction(0)
    for (a, b, c), coef in p.terms():
        s += Fraction(int(coef.p), int(coef.q)) * _exact(kind, a, b, c)
    return s


def _basis(kind, k):
    """Nodal basis in the oracle's node order, built independently:
    simplex -- barycentric Lagrange phi_alpha = prod_i prod_{m<alpha_i}
    (k lambda_i - m)/(m + 1), alpha = k lambda(node); hexahedron -- products
    of 1D equispaced Lagrange polynomials."""
    out = []
    for n in fo.nodes(kind, k):
        if kind == "tetrahedron":
            lam = [1 - n[0] - n[1] - n[2], n[0], n[1], n[2]]
            lvar = [1 - X - Y - Z, X, Y, Z]
            alpha = [int(l * k) for l in lam]
            assert sum(alpha) == k and all(Fraction(al, k) == l for al, l in zip(alpha, lam))
            e = sympy.Integer(1)
            for i in range(4):
                for m in range(alpha[i]):
                    e *= (k * lvar[i] - m) / sympy.Integer(m + 1)
        else:
            e = sympy.Integer(1)
            for s, xn in zip((X, Y, Z), n):
                j = int(xn * k)
                for m in range(k + 1):
                    if m != j:
                        e *= (s - sympy.Rational(m, k)) / sympy.Rational(j - m, k)
        out.append(_poly(e))
    return out


def _exact_residual(form, kind, k, coords, w, mu=None, lam=None):
    """A_e on an AFFINE physical cell (tet, or parallelepiped hexahedron)."""
    nodes_v = [[sympy.Rational(v).limit_denominator(10 ** 6) for v in row] for row in coords]
    V0 = sympy.Matrix(nodes_v[0])
    if kind == "tetrahedron":
        cols = [sympy.Matrix(nodes_v[i]) - V0 for i in (1, 2, 3)]
    else:  # tensor vertex order (0,0,0),(1,0,0),(0,1,0),(1,1,0),(0,0,1),...
        cols = [sympy.Matrix(nodes_v[i]) - V0 for i in (1, 2, 4)]
    J = sympy.Matrix.hstack(*cols)
    det = J.det()
    assert det > 0
    Ji = J.inv()
    basis = _basis(kind, k)
    grads = [[_poly(sum(Ji[b, a] * sympy.diff(p.as_expr(), s) for b, s in enumerate((X, Y, Z))))
              for a in range(3)] for p in basis]
    w = [sympy.Rational(v).limit_denominator(10 ** 6) for v in w]
    nd = len(basis)
    integ = lambda p: _integrate(p, kind) * Fraction(int(sympy.Rational(det).p), int(sympy.Rational(det).q))
    if form in ("helmholtz", "laplacian_scalar", "mass"):
        u = sum((w[i] * basis[i] for i in range(nd)), _poly(0))
        gu = [sum((w[i] * grads[i][a] for i in range(nd)), _poly(0)) for a in range(3)]
        out = []
        for j in range(nd):
            f = _poly(0)
            if form != "mass":
                f = f + sum((gu[a] * grads[j][a] for a in range(3)), _poly(0))
            if form != "laplacian_scalar":
                f = f + u * basis[j]
            out.append(float(integ(f)))
        return np.array(out)
    assert form == "elasticity_lame"
    gb = _basis(kind, 1)
    muf = sum((sympy.Rational(mu[v]).limit_denominator(10 ** 6) * gb[v] for v in range(len(gb))), _poly(0))
    lf = sum((sympy.Rational(lam[v]).limit_denominator(10 ** 6) * gb[v] for v in range(len(gb))), _poly(0))
    G = [[sum((w[3 * i + d] * grads[i][a] for i in range(nd)), _poly(0)) for a in range(3)]
         for d in range(3)]                                   # G[d][a] = du_d/dx_a
    tr = G[0][0] + G[1][1] + G[2][2]
    sig = [[muf * (G[d][a] + G[a][d]) + (lf * tr if a == d else _poly(0)) for a in range(3)]
           for d in range(3)]
    out = []
    for j in range(nd):
        for d in range(3):
            out.append(float(integ(sum((sig[d][a] * grads[j][a] for a in range(3)), _poly(0)))))
    return np.array(out)


CASES = [("C2-P3", "helmholtz", "tetrahedron", 3), ("C2-P4", "helmholtz", "tetrahedron", 4),
         ("C3-Q3", "laplacian_scalar", "hexahedron", 3), ("C4-hex-Q2", "elasticity_lame", "hexahedron", 2)]


@pytest.mark.parametrize("config,form,kind,k", CASES)
def test_oracle_matches_exact_single_cell(config, form, kind, k):
    """The oracle with the config's own quadrature rule (C2: exact for 2k,
    C3: k+1 GL points, C4: k+2) equals the exact residual on a perturbed
    affine cell to 1e-13 relative."""
    rng = np.random.default_rng(11 + k)
    if kind == "tetrahedron":
        coords = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
        coords = coords + np.round(rng.uniform(-0.2, 0.2, (4, 3)) * 16) / 16
    else:
        e = [np.array([1, 0.125, -0.0625]), np.array([0.25, 0.875, 0.0]), np.array([0.0625, 0.125, 1.0])]
        coords = np.array([i * e[0] + j * e[1] + l * e[2] for l in (0, 1) for j in (0, 1) for i in (0, 1)])
    cfg = C.get_config(config)
    P = fo.Problem(form, kind, k, cfg.qdegree)
    w = np.round(rng.uniform(-1, 1, P.nd * P.vs) * 16) / 16
    mu = lam = None
    if form == "elasticity_lame":
        mu = np.round(rng.uniform(0.5, 2, P.nv) * 16) / 16
        lam = np.round(rng.uniform(0.5, 2, P.nv) * 16) / 16
    got = fo.local_residual(P, coords, w, mu, lam)
    want = _exact_residual(form, kind, k, coords, w, mu, lam)
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max(), np.abs(got - want).max()


@pytest.mark.parametrize("config,form,kind,k", CASES)
def test_product_tables_match_exact_single_cell(config, form, kind, k):
    """The PRODUCT's tables (elements.tabulate on elements.quadrature_rule,
    what fe_plan_create uploads to the GPU) reproduce the exact residual
    too: a quadrature-loop restatement over those tables on the same cell."""
    import paper_1903_08243_b200 as fe
    from paper_1903_08243_b200.elements import tabulate
    cfg = C.get_config(config)
    spec = fe.operator_spec(form, kind, k)
    rule = quadrature_rule(kind, cfg.qdegree)
    tab = tabulate(spec.element, rule)
    gtab = tabulate(fe.operator_spec("mass", kind, 1).element, rule)
    rng = np.random.default_rng(5 + k)
    if kind == "tetrahedron":
        coords = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
        coords = coords + np.round(rng.uniform(-0.2, 0.2, (4, 3)) * 16) / 16
    else:
        e = [np.array([1, 0.0, 0.125]), np.array([-0.125, 1.0, 0.0]), np.array([0.0, 0.25, 0.875])]
        coords = np.array([i * e[0] + j * e[1] + l * e[2] for l in (0, 1) for j in (0, 1) for i in (0, 1)])
    vs = spec.element.value_size
    nd = spec.element.ndof_scalar
    w = np.round(rng.uniform(-1, 1, nd * vs) * 16) / 16
    mu = lam = None
    J = np.einsum("va,qvb->qab", coords, gtab.grads)
    det = np.linalg.det(J)
    Ji = np.linalg.inv(J)
    tw = rule.weights * np.abs(det)
    gx = np.einsum("qba,qib->qia", Ji, tab.grads)              # physical gradients
    if vs == 1:
        uq = tab.values @ w
        gu = np.einsum("qia,i->qa", gx, w)
        got = np.einsum("q,qa,qja->j", tw, gu, gx)
        if form == "helmholtz":
            got += np.einsum("q,q,qj->j", tw, uq, tab.values)
    else:
        mu = np.round(rng.uniform(0.5, 2, 8) * 16) / 16
        lam = np.round(rng.uniform(0.5, 2, 8) * 16) / 16
        muq, lq = gtab.values @ mu, gtab.values @ lam
        G = np.einsum("qia,id->qda", gx, w.reshape(nd, vs))
        tr = np.einsum("qdd->q", G)
        sig = muq[:, None, None] * (G + np.swapaxes(G, 1, 2)) + (lq * tr)[:, None, None] * np.eye(3)
        got = np.einsum("q,qda,qja->jd", tw, sig, gx).ravel()
    want = _exact_residual(form, kind, k, coords, w, mu, lam)
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max(), np.abs(got - want).max()
