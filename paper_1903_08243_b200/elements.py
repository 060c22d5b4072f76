"""Reference cells, Lagrange elements, quadrature rules and tabulation.

Host-side setup for the B200 operator plans.  Mirrors the reference
``fevec.elements`` API (``/root/reference/pkg/src/fevec/elements.py``) and
extends it to the cells, degrees and value sizes the B200 path needs:

* cells ``triangle``/``quadrilateral`` (reference, ``elements.py:31-72``) plus
  ``tetrahedron``/``hexahedron``;
* degrees 1..4 on simplices, 1..6 on tensor cells (reference: 1..4,
  ``elements.py:26,140-143``);
* value sizes 1..3 (reference: 1..2, ``elements.py:144-145``);
* forms ``mass``, ``helmholtz``, ``laplacian`` (vector, reference semantics),
  ``elasticity`` (reference eps(u):grad v), plus ``laplacian_scalar``,
  ``elasticity_lame`` (2 mu eps:eps + lambda div div, vertex-valued mu/lambda)
  and ``neohookean`` (compressible neo-Hookean residual P(F):grad v).

Node ordering follows the reference convention (``elements.py:93-115``):
vertices, then edge nodes (edges ordered by vertex pairs, nodes from the low
to the high vertex), then (3D) face-interior nodes, then cell-interior nodes
sorted lexicographically.

Basis functions: on simplices and on quadrilaterals up to Q4 the nodal basis
is solved from a monomial Vandermonde system exactly as the reference does
(``elements.py:136-156``), so 2D tables match the reference's bit for bit.
On hexahedra (and Q5/Q6 quads) it is the product of 1D equispaced Lagrange
polynomials: the same nodal basis (Q_k is the tensor-product space and the
nodes are the tensor lattice), but well conditioned up to Q6, where the 3D
monomial Vandermonde matrix is not.

Quadrature (``elements.py:176-208``): n = (d + 2) // 2 points per direction;
Gauss-Legendre tensor rules on quadrilaterals/hexahedra (x slowest, as the
reference orders them) and collapsed (Duffy) rules on simplices: GL x
Gauss-Jacobi(1,0) on triangles (reference) and GL x GJ(1,0) x GJ(2,0) on
tetrahedra (extension).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction
from functools import lru_cache

import numpy as np
from scipy.special import roots_jacobi, roots_legendre

__all__ = [
    "ReferenceCell",
    "ReferenceElement",
    "QuadratureRule",
    "Tabulation",
    "OperatorSpec",
    "OPERATOR_FORMS",
    "reference_cell",
    "reference_element",
    "lagrange_nodes",
    "cell_edges",
    "quadrature_rule",
    "tabulate",
    "monomial_integral",
    "operator_spec",
    "integrand_degree",
    "tensor_factors",
    "stiffness_modes",
    "MAX_QUADRATURE_DEGREE",
]

MAX_QUADRATURE_DEGREE = 20
MAX_SIMPLEX_DEGREE = 4
MAX_TENSOR_DEGREE = 6

# Reference forms first (elements.py:28), then the B200 extensions.
OPERATOR_FORMS = (
    "mass",
    "helmholtz",
    "laplacian",
    "elasticity",
    "laplacian_scalar",
    "elasticity_lame",
    "neohookean",
    "neohookean_tangent",
)


@dataclass(frozen=True)
class ReferenceCell:
    kind: str          # 'triangle' | 'quadrilateral' | 'tetrahedron' | 'hexahedron'
    vertices: tuple    # canonical vertex coordinates (Fractions)
    measure: Fraction

    @property
    def dim(self) -> int:
        return len(self.vertices[0])

    @property
    def nvertices(self) -> int:
        return len(self.vertices)

    @property
    def simplex(self) -> bool:
        return self.kind in ("triangle", "tetrahedron")


F0, F1 = Fraction(0), Fraction(1)
_TRIANGLE = ReferenceCell("triangle", ((F0, F0), (F1, F0), (F0, F1)), Fraction(1, 2))
# tensor vertex order (elements.py:51-61): x fastest
_QUAD = ReferenceCell(
    "quadrilateral", ((F0, F0), (F1, F0), (F0, F1), (F1, F1)), Fraction(1)
)
_TET = ReferenceCell(
    "tetrahedron",
    ((F0, F0, F0), (F1, F0, F0), (F0, F1, F0), (F0, F0, F1)),
    Fraction(1, 6),
)
_HEX = ReferenceCell(
    "hexahedron",
    tuple((Fraction(x), Fraction(y), Fraction(z))
          for z in (0, 1) for y in (0, 1) for x in (0, 1)),
    Fraction(1),
)

_CELLS = {
    "triangle": _TRIANGLE, "tri": _TRIANGLE,
    "quadrilateral": _QUAD, "quad": _QUAD,
    "tetrahedron": _TET, "tet": _TET,
    "hexahedron": _HEX, "hex": _HEX,
}


def reference_cell(kind) -> ReferenceCell:
    if isinstance(kind, ReferenceCell):
        return kind
    try:
        return _CELLS[kind]
    except KeyError:
        raise ValueError(
            f"unsupported cell {kind!r}; expected one of "
            "'triangle', 'quadrilateral', 'tetrahedron', 'hexahedron'"
        ) from None


def cell_edges(cell: ReferenceCell) -> tuple:
    """Edges as vertex-index pairs, ordered lexicographically
    (reference ``elements.py:74-78`` for 2D)."""
    verts = cell.vertices
    pairs = []
    for a in range(len(verts)):
        for b in range(a + 1, len(verts)):
            if cell.simplex:
                pairs.append((a, b))
            else:
                # tensor cell: an edge joins vertices differing in one coordinate
                diff = sum(1 for x, y in zip(verts[a], verts[b]) if x != y)
                if diff == 1:
                    pairs.append((a, b))
    return tuple(pairs)


def cell_faces(cell: ReferenceCell) -> tuple:
    """2D faces of a 3D cell as sorted vertex tuples, lexicographic order.
    Simplex faces list (a, b, c); hexahedron faces (a, b, c, d) in tensor
    order, so the face is parametrised from vertex a along b-a and c-a."""
    if cell.dim != 3:
        return ()
    nv = cell.nvertices
    if cell.simplex:
        return tuple((a, b, c) for a in range(nv) for b in range(a + 1, nv)
                     for c in range(b + 1, nv))
    faces = []
    verts = cell.vertices
    for axis in range(3):
        for val in (F0, F1):
            faces.append(tuple(i for i in range(nv) if verts[i][axis] == val))
    return tuple(sorted(faces))


# ---------------------------------------------------------------------------
# Lagrange elements
# ---------------------------------------------------------------------------


def _monomials(cell: ReferenceCell, k: int) -> list:
    d = cell.dim
    if cell.simplex:
        if d == 2:
            return [(a, b) for a in range(k + 1) for b in range(k + 1 - a)]
        return [(a, b, c) for a in range(k + 1) for b in range(k + 1 - a)
                for c in range(k + 1 - a - b)]
    if d == 2:
        return [(a, b) for a in range(k + 1) for b in range(k + 1)]
    return [(a, b, c) for a in range(k + 1) for b in range(k + 1) for c in range(k + 1)]


def lagrange_nodes(cell: ReferenceCell, k: int) -> list:
    """Equispaced nodes: vertices, edges (low to high vertex), face
    interiors (3D), cell interior sorted lexicographically.  Identical to the
    reference for 2D cells (``elements.py:93-115``)."""
    cell = reference_cell(cell)
    verts = cell.vertices
    d = cell.dim
    nodes = [tuple(v) for v in verts]
    for a, b in cell_edges(cell):
        va, vb = verts[a], verts[b]
        for i in range(1, k):
            t = Fraction(i, k)
            nodes.append(tuple(va[c] + t * (vb[c] - va[c]) for c in range(d)))
    for face in cell_faces(cell):
        va, vb, vc = verts[face[0]], verts[face[1]], verts[face[2]]
        fnodes = []
        for i in range(1, k):
            for j in range(1, k):
                if cell.simplex and i + j > k - 1:
                    continue
                s, t = Fraction(i, k), Fraction(j, k)
                fnodes.append(tuple(va[c] + s * (vb[c] - va[c]) + t * (vc[c] - va[c])
                                    for c in range(d)))
        fnodes.sort()
        nodes.extend(fnodes)
    interior = []
    rng = range(1, k)
    if d == 2:
        for i in rng:
            for j in rng:
                if cell.simplex and i + j > k - 1:
                    continue
                interior.append((Fraction(i, k), Fraction(j, k)))
    else:
        for i in rng:
            for j in rng:
                for l in rng:
                    if cell.simplex and i + j + l > k - 1:
                        continue
                    interior.append((Fraction(i, k), Fraction(j, k), Fraction(l, k)))
    interior.sort()
    nodes.extend(interior)
    return nodes


@dataclass(frozen=True)
class ReferenceElement:
    cell: ReferenceCell
    degree: int
    value_size: int
    nodes: tuple                                # reference coordinates (Fractions)
    coeffs: np.ndarray = field(compare=False)   # simplex: [nmono][ndof]; tensor: None
    exponents: tuple = ()

    @property
    def ndof_scalar(self) -> int:
        return len(self.nodes)

    @property
    def ndof(self) -> int:
        return self.ndof_scalar * self.value_size


def reference_element(cell, degree: int, value_size: int = 1) -> ReferenceElement:
    """Equispaced Lagrange element (reference ``elements.py:136-156``)."""
    cell = reference_cell(cell)
    maxdeg = MAX_SIMPLEX_DEGREE if cell.simplex else MAX_TENSOR_DEGREE
    if not 1 <= degree <= maxdeg:
        raise ValueError(
            f"unsupported degree {degree}; supported range is 1..{maxdeg}"
        )
    if value_size not in (1, 2, 3):
        raise ValueError(f"value_size must be 1, 2 or 3, got {value_size}")
    nodes = lagrange_nodes(cell, degree)
    exps = _monomials(cell, degree)
    coeffs = None
    # the reference solves the monomial Vandermonde system (elements.py:146-
    # 156); we do the same wherever it is well conditioned so that tables
    # match the reference's to the last bit, and use the 1D product otherwise
    if cell.simplex or (cell.kind == "quadrilateral" and degree <= 4):
        V = np.array([[math.prod(float(x) ** e for x, e in zip(node, ex)) for ex in exps]
                      for node in nodes])
        coeffs = np.linalg.solve(V, np.eye(len(nodes)))
        resid = np.abs(V @ coeffs - np.eye(len(nodes))).max()
        if resid >= 1e-10:
            raise ValueError(f"ill-conditioned Vandermonde system (residual {resid:.2e})")
        coeffs.setflags(write=False)
    return ReferenceElement(cell, degree, value_size, tuple(nodes), coeffs, tuple(exps))


# ---------------------------------------------------------------------------
# Quadrature
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class QuadratureRule:
    cell: ReferenceCell
    points: np.ndarray = field(compare=False)   # [nq][dim]
    weights: np.ndarray = field(compare=False)  # [nq]
    exactness_degree: int
    npoints_1d: int = 0

    @property
    def npoints(self) -> int:
        return len(self.weights)


@lru_cache(maxsize=None)
def _gauss_01(n: int, alpha: float = 0.0):
    if alpha == 0.0:
        x, w = roots_legendre(n)
    else:
        x, w = roots_jacobi(n, alpha, 0.0)
    return (x + 1.0) / 2.0, w


def quadrature_rule(cell, required_degree: int) -> QuadratureRule:
    """A rule exact for polynomials up to ``required_degree``
    (reference ``elements.py:176-208``; tetrahedra per SURVEY.md A.4)."""
    cell = reference_cell(cell)
    if required_degree < 0:
        raise ValueError("required_degree must be >= 0")
    if required_degree > MAX_QUADRATURE_DEGREE:
        raise ValueError(
            f"quadrature degree {required_degree} above the implemented maximum "
            f"{MAX_QUADRATURE_DEGREE}"
        )
    n = (required_degree + 2) // 2
    x01, wg = _gauss_01(n)
    w01 = wg / 2.0
    if cell.kind == "quadrilateral":
        pts = np.array([(x, y) for x in x01 for y in x01])
        wts = np.array([wx * wy for wx in w01 for wy in w01])
    elif cell.kind == "hexahedron":
        pts = np.array([(x, y, z) for x in x01 for y in x01 for z in x01])
        wts = np.array([wx * wy * wz for wx in w01 for wy in w01 for wz in w01])
    elif cell.kind == "triangle":
        v01, wj = _gauss_01(n, 1.0)
        wv = wj / 4.0
        pts = np.array([(u * (1.0 - v), v) for u in x01 for v in v01])
        wts = np.array([wu * w for wu in w01 for w in wv])
    else:
        t01, wj1 = _gauss_01(n, 1.0)
        r01, wj2 = _gauss_01(n, 2.0)
        wt, wr = wj1 / 4.0, wj2 / 8.0
        pts = np.array([(s * (1.0 - t) * (1.0 - r), t * (1.0 - r), r)
                        for s in x01 for t in t01 for r in r01])
        wts = np.array([ws * w1 * w2 for ws in w01 for w1 in wt for w2 in wr])
    pts.setflags(write=False)
    wts.setflags(write=False)
    return QuadratureRule(cell, pts, wts, required_degree, n)


def monomial_integral(cell, exps) -> Fraction:
    """Exact integral of prod x_i^{e_i} over the reference cell."""
    cell = reference_cell(cell)
    if not cell.simplex:
        out = Fraction(1)
        for e in exps:
            out /= (e + 1)
        return out
    num = math.prod(math.factorial(e) for e in exps)
    return Fraction(num, math.factorial(sum(exps) + cell.dim))


# ---------------------------------------------------------------------------
# Tabulation
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Tabulation:
    values: np.ndarray   # [nq][ndof_scalar]
    grads: np.ndarray    # [nq][ndof_scalar][dim]


def _lagrange_1d(k: int, x: np.ndarray):
    """Values and derivatives of the k+1 equispaced 1D Lagrange polynomials
    (nodes j/k) at points x: arrays [len(x)][k+1]."""
    nodes = np.arange(k + 1) / k
    x = np.asarray(x, dtype=float)
    val = np.ones((len(x), k + 1))
    der = np.zeros((len(x), k + 1))
    for j in range(k + 1):
        others = [m for m in range(k + 1) if m != j]
        denom = np.prod([nodes[j] - nodes[m] for m in others])
        for m in others:
            val[:, j] *= (x - nodes[m])
        for skip in others:
            term = np.ones(len(x))
            for m in others:
                if m != skip:
                    term *= (x - nodes[m])
            der[:, j] += term
        val[:, j] /= denom
        der[:, j] /= denom
    return val, der


def _tensor_index(element: ReferenceElement) -> np.ndarray:
    """For each local node, its 1D lattice indices [ndof][dim]."""
    k = element.degree
    return np.array([[int(x * k) for x in node] for node in element.nodes])


def tabulate_points(element: ReferenceElement, pts) -> Tabulation:
    """Values and reference gradients of the scalar basis at given points."""
    pts = np.asarray(pts, dtype=float)
    cell = element.cell
    d = cell.dim
    nq = len(pts)
    if element.coeffs is not None:
        exps = element.exponents
        nm = len(exps)
        mono = np.empty((nq, nm))
        dmono = np.zeros((nq, nm, d))
        for m, ex in enumerate(exps):
            t = pts[:, 0] ** ex[0]
            for c in range(1, d):
                t = t * pts[:, c] ** ex[c]
            mono[:, m] = t
            for a in range(d):
                if ex[a]:
                    # evaluation order of elements.py:246-247
                    t = ex[a] * (pts[:, 0] ** (ex[0] - 1) if a == 0 else pts[:, 0] ** ex[0])
                    for c in range(1, d):
                        t = t * (pts[:, c] ** (ex[c] - 1) if c == a else pts[:, c] ** ex[c])
                    dmono[:, m, a] = t
        values = mono @ element.coeffs
        grads = np.einsum("qma,mi->qia", dmono, element.coeffs)
    else:
        idx = _tensor_index(element)
        vals1 = []
        ders1 = []
        for c in range(d):
            v, dv = _lagrange_1d(element.degree, pts[:, c])
            vals1.append(v)
            ders1.append(dv)
        nd = element.ndof_scalar
        values = np.ones((nq, nd))
        grads = np.ones((nq, nd, d))
        for c in range(d):
            values *= vals1[c][:, idx[:, c]]
            for a in range(d):
                f = ders1[c] if a == c else vals1[c]
                grads[:, :, a] *= f[:, idx[:, c]]
    return Tabulation(values, grads)


def tabulate(element: ReferenceElement, rule: QuadratureRule) -> Tabulation:
    """Values and first derivatives of each scalar basis function at every
    quadrature point (reference ``elements.py:233-254``)."""
    if element.cell.kind != rule.cell.kind:
        raise ValueError(
            f"element on {element.cell.kind} tabulated with {rule.cell.kind} rule"
        )
    tab = tabulate_points(element, rule.points)
    tab.values.setflags(write=False)
    tab.grads.setflags(write=False)
    return tab


@dataclass(frozen=True)
class TensorFactors:
    """1D factors of a tensor-product element and rule: B[q][p] values and
    D[q][p] derivatives of the 1D basis at the 1D Gauss points, weights w[q],
    and ``lex[i]`` = local node index of the tensor node with lattice indices
    (i % p, (i // p) % p, i // p**2) (x fastest)."""
    B: np.ndarray
    D: np.ndarray
    w: np.ndarray
    x: np.ndarray
    lex: np.ndarray


def tensor_factors(element: ReferenceElement, rule: QuadratureRule) -> TensorFactors:
    cell = element.cell
    if cell.simplex:
        raise ValueError("tensor factors exist only on quadrilaterals/hexahedra")
    n = rule.npoints_1d
    x01, wg = _gauss_01(n)
    B, D = _lagrange_1d(element.degree, x01)
    p = element.degree + 1
    d = cell.dim
    idx = _tensor_index(element)
    lin = idx[:, 0] + p * idx[:, 1] + (p * p * idx[:, 2] if d == 3 else 0)
    lex = np.empty(p ** d, dtype=np.int32)
    lex[lin] = np.arange(len(lin), dtype=np.int32)
    return TensorFactors(B, D, wg / 2.0, x01, lex)


def stiffness_modes(element: ReferenceElement, cell=None):
    """Minimal-rank factorisation of the reference stiffness tensor of a
    simplex element: tables (w, G) with m = dim P_{k-1} "modes" such that

        S_ab[i][j] = int dphi_i/dxi_a dphi_j/dxi_b = sum_r w_r G[r,i,a] G[r,j,b]

    (w = 1).  The reference gradients of P_k lie in P_{k-1}; G[:, :, a] are
    their coefficients in an L2-orthonormal basis of P_{k-1}, obtained as the
    rank-m SVD factor of the square-root-weighted gradient table on the rule
    exact for degree 2k-2.  This is the reference's quadrature with the
    smallest possible number of points (m instead of k^d: 4 vs 8 for P2
    tetrahedra, 20 vs 64 for P4); the kernels that consume it treat the modes
    exactly like quadrature points.  Exact on affine cells."""
    cell = element.cell
    if not cell.simplex:
        raise ValueError("stiffness modes are defined for simplices")
    k, d, nd = element.degree, cell.dim, element.ndof_scalar
    rule = quadrature_rule(cell, max(2 * k - 2, 0))
    grads = tabulate(element, rule).grads                     # [nq][nd][d]
    Q = np.sqrt(rule.weights)[:, None] * grads.transpose(0, 2, 1).reshape(rule.npoints, d * nd)
    _, sig, vt = np.linalg.svd(Q, full_matrices=False)
    m = 1
    for j in range(k - 1):
        m = m * (d + k - 1 - j) // (j + 1)                    # C(k-1+d, d)
    if len(sig) < m or (len(sig) > m and sig[m] > 1e-12 * sig[0]):
        raise ValueError("stiffness tensor rank differs from dim P_{k-1}")
    G = (sig[:m, None] * vt[:m]).reshape(m, d, nd).transpose(0, 2, 1)
    return np.ones(m), np.ascontiguousarray(G)


# ---------------------------------------------------------------------------
# Operator specification
# ---------------------------------------------------------------------------


def form_value_size(form: str, dim: int) -> int:
    if form in ("laplacian", "elasticity", "elasticity_lame", "neohookean", "neohookean_tangent"):
        return dim
    return 1


@dataclass(frozen=True)
class OperatorSpec:
    """Which weak form, over which (identical) coefficient/test space
    (reference ``elements.py:262-286``).  ``params`` carries scalar material
    constants (neohookean: mu, lambda)."""

    form: str
    element: ReferenceElement
    geometry: ReferenceElement
    params: tuple = ()

    def __post_init__(self):
        if self.form not in OPERATOR_FORMS:
            raise ValueError(
                f"unknown form {self.form!r}; expected one of {OPERATOR_FORMS}"
            )
        need_vs = form_value_size(self.form, self.element.cell.dim)
        if self.element.value_size != need_vs:
            raise ValueError(
                f"{self.form} requires value_size {need_vs}, "
                f"got {self.element.value_size}"
            )
        if self.geometry.degree != 1 or self.geometry.cell.kind != self.element.cell.kind:
            raise ValueError("geometry element must be degree 1 on the same cell")

    @property
    def cell(self) -> ReferenceCell:
        return self.element.cell

    @property
    def coefficient_fields(self) -> int:
        """Number of vertex-valued coefficient fields the form reads."""
        return 2 if self.form == "elasticity_lame" else 0

    @property
    def has_state(self) -> bool:
        """Linearised form: reads the state u0 (a dof field with the layout
        of u, binding ``dat3``) at which the residual is linearised."""
        return self.form == "neohookean_tangent"


NEOHOOKEAN_DEFAULT = (1.0, 10.0)  # mu, lambda (BASELINE.json configs[4])


def operator_spec(form: str, cell, degree: int, params=None) -> OperatorSpec:
    """Convenience constructor (reference ``elements.py:289-296``)."""
    cell = reference_cell(cell)
    vs = form_value_size(form, cell.dim)
    elem = reference_element(cell, degree, vs)
    geo = reference_element(cell, 1, cell.dim)
    if params is None:
        params = NEOHOOKEAN_DEFAULT if form in ("neohookean", "neohookean_tangent") else ()
    return OperatorSpec(form, elem, geo, tuple(float(p) for p in params))


def integrand_degree(spec: OperatorSpec) -> int:
    """Quadrature-degree estimate: 2k on simplices, 2k + 2 on tensor cells
    (reference ``elements.py:299-306``)."""
    k = spec.element.degree
    est = 2 * k
    if not spec.cell.simplex:
        est += 2
    return est
