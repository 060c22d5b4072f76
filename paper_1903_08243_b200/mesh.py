"""Structured meshes and global Lagrange dof numbering.

Mirrors the reference ``fevec.mesh`` API (``/root/reference/pkg/src/fevec/
mesh.py``) with vectorised builders, so that the 10^7-cell meshes of the
BASELINE configs are generated in seconds:

* ``build_mesh(kind, nx, ny[, nz])``: unit square / unit cube.  2D output is
  identical to the reference (``mesh.py:29-61``: row-major vertices, squares
  split into ``(v00,v10,v01),(v10,v11,v01)``, quads in tensor order).  3D:
  hexahedra in tensor vertex order, or every cube split into the 6 Kuhn
  tetrahedra (path 0 -> e_s0 -> e_s0+e_s1 -> (1,1,1) for each permutation s,
  last two vertices swapped on odd permutations so that det J > 0).
* ``build_dof_map(mesh, element)``: in 2D the reference numbering
  (``mesh.py:71-115``: vertex dofs = vertex ids, then edge dofs in first-seen
  order with orientation flip, then cell interiors); in 3D every node is
  numbered by its position on the k-refined vertex lattice, vertex points
  first (dof id = vertex id), then the remaining lattice points in
  lexicographic order.  Conformity across faces is
  automatic.
* ``jitter_mesh``: seeded uniform perturbation of interior vertices by
  +-amplitude*h per coordinate (BASELINE configs).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from itertools import permutations

import numpy as np

from .elements import ReferenceElement, cell_edges, reference_cell

__all__ = ["Mesh", "DofMap", "build_mesh", "build_dof_map", "jitter_mesh",
           "kuhn_tets"]


@dataclass(frozen=True)
class Mesh:
    coords: np.ndarray     # [nvertices][dim], float64
    cell2vert: np.ndarray  # [ncells][nvert_per_cell], int32
    cell: object           # ReferenceCell
    grid: tuple = field(default=None, compare=False)  # (nx, ny[, nz]) if structured

    @property
    def ncells(self) -> int:
        return len(self.cell2vert)

    @property
    def nvertices(self) -> int:
        return len(self.coords)

    @property
    def dim(self) -> int:
        return self.coords.shape[1]


def _perm_parity(p) -> int:
    p = list(p)
    par = 0
    for i in range(len(p)):
        for j in range(i + 1, len(p)):
            if p[i] > p[j]:
                par ^= 1
    return par


def kuhn_tets() -> np.ndarray:
    """The 6 Kuhn tetrahedra of the unit cube as cube-corner bit masks
    [6][4] (bit0 = x, bit1 = y, bit2 = z), positively oriented."""
    tets = []
    for s in permutations(range(3)):
        path = [0, 1 << s[0], (1 << s[0]) | (1 << s[1]), 7]
        if _perm_parity(s):
            path[2], path[3] = path[3], path[2]
        tets.append(path)
    return np.array(tets, dtype=np.int64)


def build_mesh(kind: str, nx: int, ny: int, nz: int = None) -> Mesh:
    """Structured mesh of the unit square (2D cells) or unit cube (3D)."""
    cell = reference_cell(kind)
    if nx < 1 or ny < 1 or (cell.dim == 3 and (nz is None or nz < 1)):
        raise ValueError("mesh needs at least one cell per direction")
    if cell.dim == 2:
        xs = np.linspace(0.0, 1.0, nx + 1)
        ys = np.linspace(0.0, 1.0, ny + 1)
        X, Y = np.meshgrid(xs, ys, indexing="xy")   # row-major: x fastest
        coords = np.stack([X.ravel(), Y.ravel()], axis=1).astype(np.float64)
        j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
        i, j = i.ravel(), j.ravel()
        v00 = j * (nx + 1) + i
        v10, v01, v11 = v00 + 1, v00 + nx + 1, v00 + nx + 2
        if cell.kind == "triangle":
            c2v = np.empty((2 * nx * ny, 3), dtype=np.int64)
            c2v[0::2] = np.stack([v00, v10, v01], axis=1)
            c2v[1::2] = np.stack([v10, v11, v01], axis=1)
        else:
            c2v = np.stack([v00, v10, v01, v11], axis=1)
        grid = (nx, ny)
    else:
        xs = np.linspace(0.0, 1.0, nx + 1)
        ys = np.linspace(0.0, 1.0, ny + 1)
        zs = np.linspace(0.0, 1.0, nz + 1)
        Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
        coords = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1).astype(np.float64)
        l, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        base = (i + (nx + 1) * (j + (ny + 1) * l)).ravel()
        corner = np.array([(b & 1) + (nx + 1) * (((b >> 1) & 1) + (ny + 1) * ((b >> 2) & 1))
                           for b in range(8)], dtype=np.int64)
        if cell.kind == "hexahedron":
            c2v = base[:, None] + corner[None, :]
        else:
            kt = kuhn_tets()                       # [6][4] corner masks
            c2v = (base[:, None, None] + corner[kt][None, :, :]).reshape(-1, 4)
        grid = (nx, ny, nz)
    coords.setflags(write=False)
    c2v = np.ascontiguousarray(c2v, dtype=np.int32)
    c2v.setflags(write=False)
    return Mesh(coords, c2v, cell, grid)


def jitter_mesh(mesh: Mesh, rng, amplitude: float = 0.1) -> Mesh:
    """Perturb every interior vertex (no coordinate equal to 0 or 1) by
    uniform(-amplitude*h, amplitude*h) per coordinate, h = 1/n per
    direction.  Boundary vertices stay fixed."""
    if mesh.grid is None:
        raise ValueError("jitter needs a structured mesh")
    d = mesh.dim
    h = np.array([1.0 / n for n in mesh.grid[:d]])
    delta = rng.uniform(-1.0, 1.0, size=(mesh.nvertices, d)) * (amplitude * h)[None, :]
    x = np.array(mesh.coords)
    interior = np.all((x > 0.0) & (x < 1.0), axis=1)
    x[interior] += delta[interior]
    x.setflags(write=False)
    return Mesh(x, mesh.cell2vert, mesh.cell, mesh.grid)


@dataclass(frozen=True)
class DofMap:
    cell2dof: np.ndarray  # [ncells][ndof_scalar], int32
    ndofs_global: int     # scalar dof count (multiply by value_size for vectors)
    element: ReferenceElement


def _reference_numbering(mesh: Mesh, element: ReferenceElement) -> DofMap:
    """Vectorised restatement of the reference ``build_dof_map``
    (``mesh.py:71-115``); produces the identical numbering."""
    k = element.degree
    edges = cell_edges(mesh.cell)
    per_edge = k - 1
    nloc = element.ndof_scalar
    nv = mesh.cell.nvertices
    nc = mesh.ncells
    n_interior = nloc - nv - per_edge * len(edges)
    c2v = np.asarray(mesh.cell2vert, dtype=np.int64)
    cell2dof = np.empty((nc, nloc), dtype=np.int64)
    cell2dof[:, :nv] = c2v
    next_dof = mesh.nvertices
    if per_edge > 0:
        ea = np.array([a for a, _ in edges])
        eb = np.array([b for _, b in edges])
        ga, gb = c2v[:, ea], c2v[:, eb]                     # [nc][ne]
        lo, hi = np.minimum(ga, gb), np.maximum(ga, gb)
        keys = (lo * mesh.nvertices + hi).ravel()           # cell-major, edge-minor
        uniq, first, inv = np.unique(keys, return_index=True, return_inverse=True)
        order = np.argsort(first, kind="stable")            # first-seen order
        rank = np.empty(len(uniq), dtype=np.int64)
        rank[order] = np.arange(len(uniq))
        base = (next_dof + per_edge * rank[inv]).reshape(nc, len(edges))
        flip = (ga > gb)
        t = np.arange(per_edge)
        slot = np.where(flip[:, :, None], per_edge - 1 - t[None, None, :], t[None, None, :])
        cell2dof[:, nv:nv + per_edge * len(edges)] = (base[:, :, None] + slot).reshape(nc, -1)
        next_dof += per_edge * len(uniq)
    if n_interior > 0:
        pos = nv + per_edge * len(edges)
        cell2dof[:, pos:] = (next_dof + np.arange(nc)[:, None] * n_interior
                             + np.arange(n_interior)[None, :])
        next_dof += nc * n_interior
    out = np.ascontiguousarray(cell2dof, dtype=np.int32)
    out.setflags(write=False)
    return DofMap(out, int(next_dof), element)


def _lattice_numbering(mesh: Mesh, element: ReferenceElement) -> DofMap:
    """Position-on-lattice numbering for structured 3D meshes."""
    nx, ny, nz = mesh.grid
    k = element.degree
    Lx, Ly = k * nx + 1, k * ny + 1
    c2v = np.asarray(mesh.cell2vert, dtype=np.int64)
    # integer vertex coordinates of every cell vertex
    vi = c2v % (nx + 1)
    vj = (c2v // (nx + 1)) % (ny + 1)
    vl = c2v // ((nx + 1) * (ny + 1))
    V = np.stack([vi, vj, vl], axis=-1)                  # [nc][nv][3]
    # node offsets: k * xi as integer weights on the cell's vertices
    nodes = np.array([[int(x * k) for x in node] for node in element.nodes], dtype=np.int64)
    if mesh.cell.simplex:
        # P(node) = k*v0 + sum_a (k xi_a) (v_a - v0)
        P = k * V[:, None, 0, :] + np.einsum("ia,cad->cid", nodes, V[:, 1:, :] - V[:, None, 0, :])
    else:
        P = k * V[:, None, 0, :] + nodes[None, :, :]
    I, J, L = P[..., 0], P[..., 1], P[..., 2]
    lin = I + Lx * (J + Ly * L)
    # number of vertex lattice points strictly before (I,J,L) in lex order
    cdiv = lambda a: -(-a // k)
    before = (cdiv(L) * (ny + 1) * (nx + 1)
              + np.where(L % k == 0, cdiv(J) * (nx + 1), 0)
              + np.where((L % k == 0) & (J % k == 0), cdiv(I), 0))
    is_vertex = (I % k == 0) & (J % k == 0) & (L % k == 0)
    vid = I // k + (nx + 1) * (J // k + (ny + 1) * (L // k))
    nverts = (nx + 1) * (ny + 1) * (nz + 1)
    dof = np.where(is_vertex, vid, nverts + lin - before)
    ndofs = Lx * Ly * (k * nz + 1)
    out = np.ascontiguousarray(dof, dtype=np.int32)
    out.setflags(write=False)
    return DofMap(out, int(ndofs), element)


def build_dof_map(mesh: Mesh, element: ReferenceElement) -> DofMap:
    """Global numbering for an equispaced Lagrange space on the mesh."""
    if element.cell.kind != mesh.cell.kind:
        raise ValueError("element and mesh cell kinds differ")
    if mesh.dim == 2:
        return _reference_numbering(mesh, element)
    if mesh.grid is None:
        raise ValueError("3D dof numbering needs a structured (lattice) mesh")
    return _lattice_numbering(mesh, element)
