"""Pin the CPU oracle before trusting it.

* 2D: bitwise against golden vectors produced by the REAL reference
  (tests/golden/make_golden.py -> fevec.reference.assemble_reference);
* the reference's known-answer tests (test_kernels.py:107-124);
* 3D / new forms: sympy single-cell oracles and the reference's physics
  identities (test_reference.py:24-89) re-expressed for tets/hexes, vs=3,
  mu/lambda fields and the neo-Hookean residual.
"""

import hashlib

import numpy as np
import pytest
import sympy

from oracle import fe_oracle as fo
from paper_1903_08243_b200 import configs as C


@pytest.mark.parametrize("idx", range(32))
def test_oracle_matches_reference_golden_bitwise(golden2d, idx):
    name = str(golden2d["names"][idx])
    form, cell, deg = name.split("_")
    P = fo.Problem(form, cell, int(deg))
    g = lambda k: golden2d[f"{name}/{k}"]
    assert np.array_equal(P.pts, g("qpoints")) and np.array_equal(P.qw, g("qweights"))
    y = fo.assemble(P, g("coords"), g("cell2vert"), g("cell2dof"), g("u"))
    assert np.array_equal(y, g("y")), (name, fo.rel_l2(y, g("y")))


def test_oracle_c1_full_size_matches_reference(golden_c1):
    prob = C.build_problem(C.get_config("C1"), seed=0)
    h = hashlib.sha256()
    for a in (np.asarray(prob.mesh.coords), np.asarray(prob.dofmap.cell2dof, np.int32), prob.u):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(golden_c1["input_digest"])   # our builders == reference inputs
    P = fo.Problem("mass", "triangle", 2)
    y = fo.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u)
    assert fo.rel_l2(y, golden_c1["y"]) <= 1e-15


def test_known_answer_helmholtz_p1():
    # reference test_kernels.py:112-124: u = y on the reference triangle
    P = fo.Problem("helmholtz", "tri", 1)
    A = fo.local_residual(P, [[0, 0], [1, 0], [0, 1]], [0.0, 0.0, 1.0])
    assert np.abs(A - np.array([-11 / 24, 1 / 24, 7 / 12])).max() < 1e-14


def test_known_answer_mass_p1():
    P = fo.Problem("mass", "tri", 1)
    A = fo.local_residual(P, [[0, 0], [1, 0], [0, 1]], np.ones(3))
    assert np.abs(A - 1 / 6).max() < 1e-15


# ---------------------------------------------------------------------------
# sympy single-cell oracle for 3D cells (restating test_kernels.py:36-104)
# ---------------------------------------------------------------------------

X, Y, Z = sympy.symbols("X Y Z")


def _sym_basis(kind, k):
    nodes = fo.nodes(kind, k)
    if kind == "hexahedron":
        # 1D Lagrange products
        def l1(j, s):
            e = sympy.Integer(1)
            for m in range(k + 1):
                if m != j:
                    e *= (s - sympy.Rational(m, k)) / sympy.Rational(j - m, k)
            return e
        return [sympy.expand(l1(int(n[0] * k), X) * l1(int(n[1] * k), Y) * l1(int(n[2] * k), Z))
                for n in nodes]
    exps = [(a, b, c) for a in range(k + 1) for b in range(k + 1 - a) for c in range(k + 1 - a - b)]
    V = sympy.Matrix([[n[0] ** a * n[1] ** b * n[2] ** c for (a, b, c) in exps] for n in nodes])
    Ci = V.inv()
    return [sympy.expand(sum(Ci[m, i] * X ** a * Y ** b * Z ** c for m, (a, b, c) in enumerate(exps)))
            for i in range(len(nodes))]


def _sym_residual(form, kind, k, coords, w, mu=None, lam=None):
    basis = _sym_basis(kind, k)
    gb = _sym_basis(kind, 1)
    coords = sympy.Matrix([[sympy.Rational(v) for v in row] for row in coords])
    xm = [sum(coords[v, a] * gb[v] for v in range(len(gb))) for a in range(3)]
    J = sympy.Matrix([[sympy.diff(xm[a], s) for s in (X, Y, Z)] for a in range(3)])
    detJ = J.det()
    Jinv = J.inv()

    def grad(f):
        return Jinv.T * sympy.Matrix([sympy.diff(f, s) for s in (X, Y, Z)])

    def integrate(f):
        if kind == "hexahedron":
            return sympy.integrate(f, (Z, 0, 1), (Y, 0, 1), (X, 0, 1))
        return sympy.integrate(f, (Z, 0, 1 - X - Y), (Y, 0, 1 - X), (X, 0, 1))

    vs = 3 if form in fo.VECTOR_FORMS else 1
    w = [sympy.Rational(v) for v in w]
    out = []
    if vs == 1:
        u = sum(w[i] * basis[i] for i in range(len(basis)))
        gu = grad(u)
        for j in range(len(basis)):
            if form == "mass":
                f = u * basis[j]
            elif form == "helmholtz":
                f = gu.dot(grad(basis[j])) + u * basis[j]
            else:
                f = gu.dot(grad(basis[j]))
            out.append(integrate(sympy.expand(f * detJ)))
        return np.array([float(v) for v in out])
    uc = [sum(w[3 * i + d] * basis[i] for i in range(len(basis))) for d in range(3)]
    G = sympy.Matrix([[grad(uc[d])[a] for a in range(3)] for d in range(3)])  # G[d][a]
    eps = (G + G.T) / 2
    if form == "elasticity_lame":
        muf = sum(sympy.Rational(mu[v]) * gb[v] for v in range(len(gb)))
        lf = sum(sympy.Rational(lam[v]) * gb[v] for v in range(len(gb)))
        sig = 2 * muf * eps + lf * eps.trace() * sympy.eye(3)
    elif form == "laplacian":
        sig = G
    else:
        sig = eps
    for j in range(len(basis)):
        gv = grad(basis[j])
        for d in range(3):
            f = sum(sig[d, a] * gv[a] for a in range(3))
            out.append(integrate(sympy.expand(f * detJ)))
    return np.array([float(v) for v in out])


TET = [[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]]


@pytest.mark.parametrize("form,kind,k", [
    ("mass", "tetrahedron", 2), ("helmholtz", "tetrahedron", 1), ("helmholtz", "tetrahedron", 2),
    ("laplacian_scalar", "tetrahedron", 2), ("elasticity_lame", "tetrahedron", 1),
    ("helmholtz", "hexahedron", 1), ("laplacian_scalar", "hexahedron", 2),
])
def test_oracle_matches_sympy_single_cell(form, kind, k):
    rng = np.random.default_rng(7)
    if kind == "tetrahedron":
        coords = np.array(TET, float) + np.round(rng.uniform(-0.2, 0.2, (4, 3)) * 8) / 8
    else:
        # a parallelepiped (affine hexahedron): polynomial integrands, exact rule
        e1, e2, e3 = np.array([1, 0.125, 0]), np.array([0.25, 1, 0]), np.array([0, 0.125, 1])
        coords = np.array([i * e1 + j * e2 + l * e3 for l in (0, 1) for j in (0, 1) for i in (0, 1)])
    P = fo.Problem(form, kind, k)
    nd = P.nd
    w = np.round(rng.uniform(-1, 1, nd * P.vs) * 8) / 8
    mu = lam = None
    if form == "elasticity_lame":
        mu = np.round(rng.uniform(0.5, 2, 4) * 8) / 8
        lam = np.round(rng.uniform(0.5, 2, 4) * 8) / 8
    got = fo.local_residual(P, coords, w, mu, lam)
    want = _sym_residual(form, kind, k, coords.tolist(), w.tolist(), mu, lam)
    assert np.abs(got - want).max() < 1e-12 * max(1.0, np.abs(want).max())


# ---------------------------------------------------------------------------
# identities (reference test_reference.py:24-89, re-expressed in 3D)
# ---------------------------------------------------------------------------


def _problem(name, n, seed=0):
    return C.build_problem(C.get_config(name, n), seed)


def _asm(prob, u=None, start=0, end=None, form=None):
    P = fo.Problem(form or prob.spec.form, prob.spec.cell.kind, prob.spec.element.degree,
                   prob.rule.exactness_degree, prob.spec.params)
    return fo.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof,
                       prob.u if u is None else u, prob.mu, prob.lam, start, end,
                       state=prob.state)


@pytest.mark.parametrize("name", ["C2-P1", "C2-P2", "C2-P3", "C3-Q1", "C3-Q3"])
def test_mass_of_one_is_volume(name):
    prob = _problem(name, 3)
    y = _asm(prob, np.ones(prob.nglobal), form="mass")
    assert abs(y.sum() - 1.0) < 1e-13


@pytest.mark.parametrize("name", ["C2-P2", "C3-Q2"])
def test_gradient_forms_annihilate_constants(name):
    prob = _problem(name, 3)
    y = _asm(prob, np.ones(prob.nglobal))
    if prob.spec.form == "helmholtz":
        assert np.abs(y - _asm(prob, np.ones(prob.nglobal), form="mass")).max() < 1e-14
    else:
        assert np.abs(y).max() < 1e-13


@pytest.mark.parametrize("name", ["C4-hex-Q1", "C4-hex-Q2", "C4-quad-Q2", "C5"])
def test_vector_forms_annihilate_translations(name):
    prob = _problem(name, 3)
    d = prob.mesh.dim
    u = np.tile(np.array([0.3, -0.7, 0.2][:d]) * (0.01 if name == "C5" else 1.0), prob.nglobal)
    y = _asm(prob, u)
    assert np.abs(y).max() < 1e-14


def _dof_positions(prob):
    from paper_1903_08243_b200.elements import tabulate_points
    el = prob.spec.element
    pts = np.array([[float(c) for c in n] for n in el.nodes])
    gphi = tabulate_points(prob.spec.geometry, pts).values       # [nd][nv]
    X = np.einsum("iv,cva->cia", gphi, prob.mesh.coords[prob.mesh.cell2vert])
    d = prob.mesh.dim
    xnode = np.zeros((prob.nglobal, d))
    xnode[prob.dofmap.cell2dof.ravel()] = X.reshape(-1, d)
    return xnode


def _rigid_rotation(prob, angle):
    """u = (R - I) x at every dof node (exact in any Lagrange space)."""
    xnode = _dof_positions(prob)
    d = prob.mesh.dim
    c, s = np.cos(angle), np.sin(angle)
    R = np.eye(d)
    R[0, 0], R[0, 1], R[1, 0], R[1, 1] = c, -s, s, c
    return (xnode @ R.T - xnode).ravel()


@pytest.mark.parametrize("name", ["C4-hex-Q1", "C4-quad-Q1", "C4-hex-Q2"])
def test_lame_elasticity_annihilates_infinitesimal_rotation(name):
    # reference test_reference.py:51-69: u = W x with W skew gives eps(u) = 0
    prob = _problem(name, 3)
    d = prob.mesh.dim
    W = np.zeros((d, d))
    W[0, 1], W[1, 0] = -1.0, 1.0
    if d == 3:
        W[1, 2], W[2, 1] = -0.5, 0.5
    u = (_dof_positions(prob) @ W.T).ravel()
    y = _asm(prob, u)
    assert np.abs(y).max() < 1e-13
    # the vector laplacian does NOT annihilate it
    assert np.abs(_asm(prob, u, form="laplacian")).max() > 1e-3


def test_neohookean_rigid_rotation_is_stress_free():
    prob = _problem("C5", 3)
    u = _rigid_rotation(prob, 0.3)           # finite rotation: F = R, P(R) = 0
    y = _asm(prob, u)
    assert np.abs(y).max() < 1e-13


def test_neohookean_is_gradient_of_strain_energy():
    """r(u; v) = dPi/du with Pi = int mu/2 (tr C - 3) - mu ln J + lam/2 (ln J)^2:
    central finite differences of Pi along random directions."""
    prob = _problem("C5", 2)
    P = fo.Problem("neohookean", "tetrahedron", 2, 4)
    coords, c2v, c2d = prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof
    mu_c, lam_c = P.params

    def energy(u):
        X = coords[c2v]
        J = np.einsum("cva,qvb->cqab", X, P.gdphi)
        det, Jinv = fo._det_inv(J)
        tw = P.qw[None, :] * np.abs(det)
        gphix = np.einsum("cqba,qib->cqia", Jinv, P.dphi)
        w = u.reshape(-1, 3)[c2d]
        G = np.einsum("cqia,cid->cqda", gphix, w)
        F = np.eye(3) + G
        Jf, _ = fo._det_inv(F)
        trC = np.einsum("cqda,cqda->cq", F, F)
        psi = mu_c / 2 * (trC - 3) - mu_c * np.log(Jf) + lam_c / 2 * np.log(Jf) ** 2
        return float((tw * psi).sum())

    y = _asm(prob)
    rng = np.random.default_rng(3)
    for _ in range(3):
        v = rng.uniform(-1, 1, prob.u.shape) * 0.01 / 2
        h = 1e-4
        fd = (energy(prob.u + h * v) - energy(prob.u - h * v)) / (2 * h)
        assert abs(fd - y @ v) < 1e-7 * max(1.0, abs(fd))


def test_neohookean_small_strain_limit_is_lame_elasticity():
    prob = _problem("C5", 2)
    u = prob.u * 1e-3
    y_nh = _asm(prob, u)
    # linearisation at F = I: P ~ mu (G + G^T) + lambda tr(G) I = 2 mu eps + lambda tr eps I
    P = fo.Problem("elasticity_lame", "tetrahedron", 2, 4)
    nv = prob.mesh.nvertices
    y_lin = fo.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, u,
                        np.full(nv, 1.0), np.full(nv, 10.0))
    assert fo.rel_l2(y_nh, y_lin) < 1e-3 * 5


@pytest.mark.parametrize("name", ["C2-P2", "C3-Q2", "C4-hex-Q1", "C5"])
def test_partition_independence(name):
    """reference test_reference.py:72-89: cell sub-ranges assembled
    separately and summed equal the whole (template of the multi-GPU test)."""
    prob = _problem(name, 3)
    whole = _asm(prob)
    nc = prob.mesh.ncells
    cuts = [0, nc // 3 + 1, 2 * nc // 3 - 1, nc]
    total = sum(_asm(prob, start=a, end=b) for a, b in zip(cuts[:-1], cuts[1:]))
    assert np.abs(total - whole).max() <= 1e-13 * max(1.0, np.abs(whole).max())


def test_elasticity_lame_half_zero_equals_reference_elasticity():
    """2 mu eps:eps + lambda div div with mu = 1/2, lambda = 0
    is the reference elasticity form eps(u):grad v."""
    prob = _problem("C4-quad-Q2", 4)
    nv = prob.mesh.nvertices
    P = fo.Problem("elasticity_lame", "quadrilateral", 2)
    a = fo.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u,
                    np.full(nv, 0.5), np.zeros(nv))
    Pr = fo.Problem("elasticity", "quadrilateral", 2)
    b = fo.assemble(Pr, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u)
    assert fo.rel_l2(a, b) < 1e-15


# ---------------------------------------------------------------------------
# neohookean_tangent: the linearised residual at a state u0
# ---------------------------------------------------------------------------


def _tangent(prob_c6, du, state):
    P = fo.Problem("neohookean_tangent", "tetrahedron", 2, 4)
    return fo.assemble(P, prob_c6.mesh.coords, prob_c6.mesh.cell2vert, prob_c6.dofmap.cell2dof,
                       du, state=state)


def _residual(prob, u):
    P = fo.Problem("neohookean", "tetrahedron", 2, 4)
    return fo.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, u)


def test_neohookean_tangent_is_derivative_of_residual():
    """a(u0; du, v) = d/de r(u0 + e du; v): central differences of the
    residual (error O(e^2)) along the configured direction."""
    prob = _problem("C6", 2)
    a = _tangent(prob, prob.u, prob.state)
    h = 1e-3 * 0.01 / 2          # step relative to the state's scale
    fd = (_residual(prob, prob.state + h * prob.u) - _residual(prob, prob.state - h * prob.u)) / (2 * h)
    assert fo.rel_l2(a, fd) < 1e-6


def test_neohookean_tangent_is_symmetric():
    """Hyperelastic tangent: v . A(u0) du = du . A(u0) v."""
    prob = _problem("C6", 2)
    rng = np.random.default_rng(11)
    v = rng.uniform(-1, 1, prob.u.shape)
    lhs = v @ _tangent(prob, prob.u, prob.state)
    rhs = prob.u @ _tangent(prob, v, prob.state)
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


def test_neohookean_tangent_at_zero_state_is_lame_elasticity():
    """At u0 = 0 (F = I) the tangent is exactly 2 mu eps : eps(v) + lambda
    div div with mu = 1, lambda = 10."""
    prob = _problem("C6", 2)
    y = _tangent(prob, prob.u, np.zeros_like(prob.u))
    P = fo.Problem("elasticity_lame", "tetrahedron", 2, 4)
    nv = prob.mesh.nvertices
    y_lin = fo.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u,
                        np.full(nv, 1.0), np.full(nv, 10.0))
    assert fo.rel_l2(y, y_lin) < 1e-13


def test_neohookean_tangent_annihilates_translations():
    prob = _problem("C6", 2)
    t = np.tile([0.3, -0.2, 0.7], prob.u.size // 3)
    y = _tangent(prob, t, prob.state)
    assert np.abs(y).max() < 1e-13
