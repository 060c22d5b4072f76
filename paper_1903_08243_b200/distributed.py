"""Element partition across GPUs with shared-dof halo sums.

The reference is single-process; the paper ran one MPI
process per core over a partitioned mesh.  Here: one process
per GPU (torchrun), the structured mesh is cut into z-slabs of whole cube
layers, every rank assembles y_local = sum over ITS cells P_e^T A_e(P_e u)
with the sm_100a kernels, and the only exchange is the sum of the partial
results on the node planes two neighbouring slabs share:

    rank r:  y[top plane]    += y_{r+1}[bottom plane]
             y[bottom plane] += y_{r-1}[top plane]

done with NCCL point-to-point send/recv (torch.distributed batch P2P, one
group per apply).  Both neighbours end with the fully summed interface
values, so the distributed y restricted to each slab equals the
single-domain y (partition independence, reference test_reference.py:72-89).

Slab-local numbering: nodes of the k-refined lattice, vertex points first
(dof id = vertex id, as the reference numbers them, mesh.py:95 -- the
kernels then read no separate vertex map), then the other lattice points,
both lexicographic (x fastest, z slowest).  An interface plane is therefore
two contiguous blocks (its vertex points at the start/end of the vertex
section, its other points at the start/end of the rest): no gather lists.
Inputs are drawn per lattice plane from SeedSequence((seed, stream, plane)),
so a plane shared by two ranks gets identical coordinates and coefficients
on both.

Scaling modes: STRONG (``slab_split``, what bench.py runs): the config's one
fixed mesh is cut into world slabs of nz/world layers -- the BASELINE C5
partition (128 cube layers -> 128/N per GPU), applied to every structured
config (3D: z-slabs; 2D: rows of squares).  WEAK (``slab_range``): every rank
owns nz layers of an nz*world-layer mesh.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .configs import Config
from .elements import operator_spec, quadrature_rule
from .mesh import DofMap, Mesh, kuhn_tets

__all__ = ["Slab", "build_slab", "DistributedOperator", "slab_range", "slab_split", "global_dof_index", "exchange_loopback", "vertex_first_ids"]


@dataclass
class Slab:
    config: Config
    spec: object
    rule: object
    mesh: Mesh
    dofmap: DofMap
    u: np.ndarray
    mu: np.ndarray
    lam: np.ndarray
    z0: int            # first cube layer (global)
    z1: int            # one past the last cube layer
    nz_global: int
    plane: int         # nodes per lattice plane (Lx * Ly)
    state: np.ndarray = None   # u0 of a linearised form (C6), per-plane seeded like u
    nvert: int = 0             # vertices of the slab (= vertex dofs, numbered first)
    nvp: int = 0               # vertices per layer plane
    global_index: np.ndarray = None   # single-domain scalar dof id of every slab dof
    boundary_first: bool = False      # cell order: first layer, last layer, interior layers

    def interface_ranges(self, side: str):
        """Scalar-dof ranges [a, b) of the interface node plane at the bottom
        (``"below"``) or top (``"above"``) of the slab: its vertex points
        (a block of the vertex section) and its other lattice points (a
        block of the rest), both in lexicographic order on either side of
        the interface."""
        n = self.dofmap.ndofs_global
        rest = self.plane - self.nvp          # non-vertex points of a vertex plane
        if side == "below":
            return [(0, self.nvp), (self.nvert, self.nvert + rest)]
        return [(self.nvert - self.nvp, self.nvert), (n - rest, n)]

    def coef(self):
        if self.mu is not None:
            return (self.mu, self.lam)
        if self.state is not None:
            return (self.state, None)
        return None

    @property
    def ndofs(self) -> int:
        return self.spec.element.value_size * self.dofmap.ndofs_global

    @property
    def has_below(self) -> bool:
        return self.z0 > 0

    @property
    def has_above(self) -> bool:
        return self.z1 < self.nz_global


def _plane_rng(seed, stream, plane):
    return np.random.default_rng(np.random.SeedSequence([seed, stream, plane]))


def vertex_first_ids(P, ncells_per_axis, k):
    """Dof id of lattice points P[..., d] on the k-refined lattice of an
    n_0 x ... x n_{d-1} structured mesh: vertex points (all coordinates
    multiples of k) first with id = vertex id, then the other points in
    lexicographic order (x fastest) -- mesh.py _lattice_numbering, 2D or 3D."""
    d = len(ncells_per_axis)
    nv1 = [n + 1 for n in ncells_per_axis]
    Lk = [k * n + 1 for n in ncells_per_axis]
    cdiv = lambda a: -(-a // k)
    lin = np.zeros(P.shape[:-1], dtype=np.int64)
    vid = np.zeros(P.shape[:-1], dtype=np.int64)
    before = np.zeros(P.shape[:-1], dtype=np.int64)
    is_vertex = np.ones(P.shape[:-1], dtype=bool)
    stride_l, stride_v = 1, 1
    for a in range(d):
        lin += P[..., a] * stride_l
        vid += (P[..., a] // k) * stride_v
        stride_l *= Lk[a]
        stride_v *= nv1[a]
    # vertex points strictly before P in lexicographic order (slowest axis first)
    on_vertex_rows = np.ones(P.shape[:-1], dtype=bool)
    for a in range(d - 1, -1, -1):
        below = int(np.prod(nv1[:a])) if a > 0 else 1
        before += np.where(on_vertex_rows, cdiv(P[..., a]) * below, 0)
        on_vertex_rows &= P[..., a] % k == 0
        is_vertex &= P[..., a] % k == 0
    nverts = int(np.prod(nv1))
    return np.where(is_vertex, vid, nverts + lin - before)


def vertex_first_table(L, k):
    """``vertex_first_ids`` for every point of a lattice with L[a] points per
    axis (x fastest), indexed by the lexicographic id: vertex points ranked
    among vertex points, the others after them ranked among the others."""
    flags = [np.arange(n) % k == 0 for n in L]
    isv = flags[-1]
    for f in flags[-2::-1]:
        isv = (isv[:, None] & f[None, :]).ravel()
    cv = np.cumsum(isv, dtype=np.int64)
    nv = int(cv[-1])
    lin = np.arange(isv.size, dtype=np.int64)
    return np.where(isv, cv - 1, nv + lin - cv)


def build_slab(cfg: Config, seed: int, z0: int, z1: int, nz_global: int, boundary_first: bool = False) -> Slab:
    """Cell layers [z0, z1) along the slowest axis (z in 3D, y in 2D) of the
    global structured mesh of a config (nx x ny x nz_global cubes, or nx x
    nz_global squares), with slab-local lattice numbering.  2D cells follow
    the reference split (mesh.py:52-57): squares into (v00,v10,v01),
    (v10,v11,v01), quads in tensor order.  ``boundary_first``: the cells of
    the LAST layer follow those of the first (cell order only; the dof
    numbering is unchanged), so the two boundary layers -- the only cells that
    touch an interface plane -- are ONE contiguous cell range and
    DistributedOperator applies them with one launch."""
    d = len(cfg.n)
    if d not in (2, 3):
        raise ValueError("slab partition needs a structured 2D or 3D config")
    nx = cfg.n[0]
    ny = cfg.n[1] if d == 3 else 1          # 2D: a single "row" of x per layer
    nzl = z1 - z0
    spec = operator_spec(cfg.form, cfg.cell, cfg.degree)
    rule = quadrature_rule(cfg.cell, cfg.qdegree)
    k = spec.element.degree
    vs = spec.element.value_size
    hz = 1.0 / nz_global
    xs = np.linspace(0.0, 1.0, nx + 1)
    if d == 3:
        ys = np.linspace(0.0, 1.0, ny + 1)
        Y, X = np.meshgrid(ys, xs, indexing="ij")
        h = np.array([1.0 / nx, 1.0 / ny, hz])
        nvp = (ny + 1) * (nx + 1)                   # vertices per layer plane
        inner = np.zeros((ny + 1, nx + 1), bool)
        inner[1:-1, 1:-1] = True
        inner = inner.ravel()
        base_plane = np.stack([X.ravel(), Y.ravel()], axis=1)
    else:
        h = np.array([1.0 / nx, hz])
        nvp = nx + 1
        inner = np.zeros(nx + 1, bool)
        inner[1:-1] = True
        base_plane = xs[:, None]
    coords = np.empty((nzl + 1, nvp, d))
    for lz in range(nzl + 1):
        gz = z0 + lz
        coords[lz, :, :d - 1] = base_plane
        coords[lz, :, d - 1] = gz * hz
        if cfg.jitter and 0 < gz < nz_global:
            delta = _plane_rng(seed, 0, gz).uniform(-1.0, 1.0, size=(nvp, d)) * (0.1 * h)
            coords[lz][inner] += delta[inner]
    coords = coords.reshape(-1, d)
    # cells: layers slowest; 6 Kuhn tets / one hex per cube, 2 tris / one quad per square
    boundary_first = bool(boundary_first) and nzl >= 3
    layers = np.arange(nzl)
    if boundary_first:
        layers = np.concatenate([[0, nzl - 1], np.arange(1, nzl - 1)])
    if d == 3:
        l, j, i = np.meshgrid(layers, np.arange(ny), np.arange(nx), indexing="ij")
        base = (i + (nx + 1) * (j + (ny + 1) * l)).ravel()
        corner = np.array([(b & 1) + (nx + 1) * (((b >> 1) & 1) + (ny + 1) * ((b >> 2) & 1))
                           for b in range(8)], dtype=np.int64)
        cells_bits = kuhn_tets() if cfg.cell == "tetrahedron" else np.arange(8)[None, :]
    else:
        l, i = np.meshgrid(layers, np.arange(nx), indexing="ij")
        base = (i + (nx + 1) * l).ravel()
        corner = np.array([(b & 1) + (nx + 1) * ((b >> 1) & 1) for b in range(4)], dtype=np.int64)
        cells_bits = (np.array([[0, 1, 2], [1, 3, 2]]) if cfg.cell == "triangle"
                      else np.arange(4)[None, :])
    c2v = (base[:, None, None] + corner[cells_bits][None, :, :]).reshape(-1, cells_bits.shape[1])
    grid = (nx, ny, nzl) if d == 3 else (nx, nzl)
    mesh = Mesh(coords, np.ascontiguousarray(c2v, np.int32), spec.cell, grid)
    # slab-local numbering: lattice points, VERTEX POINTS FIRST (dof id =
    # vertex id, so map0[:, :nv] is the vertex map -- reference mesh.py:95,
    # no separate vertex-map traffic), then the other lattice points, both
    # lexicographic (x fastest, layer axis slowest)
    nper = (nx, ny, nzl) if d == 3 else (nx, nzl)
    L = [k * n + 1 for n in nper]
    strides = np.cumprod([1] + L[:-1])                       # lexicographic lattice strides
    nodes = np.array([[int(round(x * k)) for x in node] for node in spec.element.nodes], dtype=np.int64)
    # lattice offsets of every local node for each cell type of a cube/square
    # (a cell = cube origin + type), then broadcast over the cubes
    cbits = np.array([[(b >> a) & 1 for a in range(d)] for b in range(2 ** d)], dtype=np.int64)
    Vt = cbits[cells_bits]                                   # [types][nv][d]
    if spec.cell.simplex:
        off = k * Vt[:, None, 0, :] + np.einsum("ia,tad->tid", nodes, Vt[:, 1:, :] - Vt[:, None, 0, :])
    else:
        off = k * Vt[:, None, 0, :] + nodes[None, :, :]
    off_lin = off @ strides                                  # [types][nd]
    origin = np.stack([i.ravel(), (j.ravel() if d == 3 else l.ravel())] + ([l.ravel()] if d == 3 else []),
                      axis=1).astype(np.int64)               # cube origins, cell order
    lin = ((k * origin) @ strides)[:, None, None] + off_lin[None, :, :]
    lin = lin.reshape(-1, nodes.shape[0])                    # [ncells][nd] lexicographic lattice ids
    table = vertex_first_table(L, k)
    dof = table[lin]
    plane = int(np.prod(L[:-1]))
    nlat = plane * L[-1]
    dm = DofMap(np.ascontiguousarray(dof, np.int32), nlat, spec.element)
    lat = np.empty(nlat, dtype=np.int64)                     # lexicographic id of each dof
    lat[table] = np.arange(nlat, dtype=np.int64)
    # single-domain (world = 1) id of every slab dof: the same numbering on
    # the whole mesh; a slab's lattice points are the global ones shifted by
    # k z0 layers
    gtable = vertex_first_table(L[:-1] + [k * nz_global + 1], k)
    global_index = gtable[lat + k * z0 * plane]
    # coefficients per lattice plane (seeded per global plane, so a plane two
    # slabs share gets identical values on both)
    nmax = max(cfg.n[:-1] + (nz_global,))
    ulat = np.empty((L[-1], plane * vs))
    for q in range(L[-1]):
        ulat[q] = _plane_rng(seed, 1, k * z0 + q).uniform(-1.0, 1.0, plane * vs)
    u = ulat.reshape(nlat, vs)[lat].ravel()
    if cfg.u_scale == "h":
        u *= 0.01 / nmax
    mu = lam = None
    if spec.coefficient_fields:
        mu = np.concatenate([_plane_rng(seed, 2, z0 + lz).uniform(0.5, 2.0, nvp) for lz in range(nzl + 1)])
        lam = np.concatenate([_plane_rng(seed, 3, z0 + lz).uniform(0.5, 2.0, nvp) for lz in range(nzl + 1)])
    state = None
    if spec.has_state:
        slat = np.concatenate([_plane_rng(seed, 4, k * z0 + q).uniform(-1.0, 1.0, plane * vs)
                               for q in range(L[-1])])
        state = slat.reshape(nlat, vs)[lat].ravel() * (0.01 / nmax)
    nvert = (nzl + 1) * nvp
    return Slab(cfg, spec, rule, mesh, dm, u, mu, lam, z0, z1, nz_global, plane, state,
                nvert, nvp, global_index, boundary_first)


class DistributedOperator:
    """y = A u on this rank's slab, interface planes summed with the
    neighbouring ranks; ``torch.distributed`` must be initialised (NCCL for
    CUDA tensors, gloo for CPU tensors).

    ``local_apply(u, y)`` computes the slab-local action (overwrite).  With
    ``range_apply(u, y, start, end, overwrite)`` (the plan's fe_apply on a
    cell range) the exchange OVERLAPS the interior: cells are ordered cube
    layer by cube layer (z slowest), so the boundary layers -- the only cells
    touching an interface plane -- are two contiguous ranges.  They are
    applied first, the interface planes go out on NCCL (its stream waits for
    them, not for the interior), the interior layers run on the compute
    stream meanwhile, and the received partial sums are added after both."""

    def __init__(self, slab: Slab, local_apply, rank: int, world: int, range_apply=None):
        self.slab = slab
        self.local_apply = local_apply
        self.range_apply = range_apply
        self.rank = rank
        self.world = world
        vs = slab.spec.element.value_size
        self.ranges = {side: [(vs * a, vs * b) for a, b in slab.interface_ranges(side)]
                       for side in ("below", "above")}
        self.n_if = sum(b - a for a, b in self.ranges["below"])
        nzl = slab.mesh.grid[-1]
        self.layer_cells = slab.mesh.ncells // nzl
        self.nlayers = nzl
        self._bufs = None
        self._idx = {}

    def _sides(self):
        return [sd for sd, has in (("below", self.slab.has_below), ("above", self.slab.has_above)) if has]

    def _buffers(self, y):
        """(recv, send): one contiguous buffer each, a segment of n_if entries
        per interface this slab has (below first)."""
        import torch
        if self._bufs is None or self._bufs[0].device != y.device:
            n = self.n_if * max(1, len(self._sides()))
            self._bufs = tuple(torch.empty(n, dtype=y.dtype, device=y.device) for _ in range(2))
        return self._bufs

    def _index(self, y):
        """Entries of y on this slab's interface planes (the contiguous blocks
        of every plane concatenated, below first), as one index tensor on y's
        device: the pack and the unpack-add of ALL planes are one kernel each."""
        import torch
        if y.device not in self._idx:
            blocks = [torch.arange(a, b, device=y.device) for sd in self._sides() for a, b in self.ranges[sd]]
            self._idx[y.device] = torch.cat(blocks) if blocks else torch.empty(0, dtype=torch.long, device=y.device)
        return self._idx[y.device]

    def _pack(self, y):
        import torch
        recv, send = self._buffers(y)
        return torch.index_select(y, 0, self._index(y), out=send)

    def _unpack_add(self, y):
        recv, send = self._buffers(y)
        y.index_add_(0, self._index(y), recv)

    def _start_exchange(self, y):
        import torch.distributed as dist
        recv, send = self._buffers(y)
        sides = self._sides()
        if not sides:
            return []
        self._pack(y)
        ops = []
        for k, sd in enumerate(sides):
            peer = self.rank - 1 if sd == "below" else self.rank + 1
            seg = slice(k * self.n_if, (k + 1) * self.n_if)
            ops.append(dist.P2POp(dist.isend, send[seg], peer))
            ops.append(dist.P2POp(dist.irecv, recv[seg], peer))
        return dist.batch_isend_irecv(ops)

    def _finish_exchange(self, y, works):
        for w in works:
            w.wait()
        if works:
            self._unpack_add(y)

    def exchange(self, y):
        """Sum the interface planes with the neighbours (in place)."""
        self._finish_exchange(y, self._start_exchange(y))

    def apply(self, u, y):
        nc, lc = self.slab.mesh.ncells, self.layer_cells
        if self.range_apply is None or self.world == 1 or self.nlayers < 3:
            self.local_apply(u, y)
            self.exchange(y)
            return y
        # boundary layers first (the only cells touching an interface plane)
        if getattr(self.slab, "boundary_first", False):
            self.range_apply(u, y, 0, 2 * lc, True)     # zero-fills y, then both boundary layers (one launch)
            works = self._start_exchange(y)             # NCCL waits for the boundary cells
            self.range_apply(u, y, 2 * lc, nc, False)   # interior overlaps the exchange
            self._finish_exchange(y, works)
            return y
        self.range_apply(u, y, 0, lc, True)           # zero-fills y, then layer 0
        self.range_apply(u, y, nc - lc, nc, False)
        works = self._start_exchange(y)                 # NCCL waits for the boundary cells
        self.range_apply(u, y, lc, nc - lc, False)      # interior overlaps the exchange
        self._finish_exchange(y, works)
        return y


def exchange_loopback(ys, slabs):
    """In-process equivalent of DistributedOperator.exchange for a list of
    consecutive slabs' y vectors (one process driving several slabs, e.g. on
    one GPU): both neighbours of every interface end with the sum."""
    for (lo, slo), (hi, shi) in zip(zip(ys[:-1], slabs[:-1]), zip(ys[1:], slabs[1:])):
        vs = slo.spec.element.value_size
        for (a0, a1), (b0, b1) in zip(slo.interface_ranges("above"), shi.interface_ranges("below")):
            s = lo[vs * a0:vs * a1] + hi[vs * b0:vs * b1]
            lo[vs * a0:vs * a1] = s
            hi[vs * b0:vs * b1] = s


def slab_range(rank: int, world: int, nz_per_rank: int):
    """Weak scaling: rank r owns cell layers [r nz, (r+1) nz)."""
    return rank * nz_per_rank, (rank + 1) * nz_per_rank, world * nz_per_rank


def slab_split(rank: int, world: int, nz_global: int):
    """Strong scaling: the nz_global cell layers of ONE fixed mesh split into
    world contiguous slabs as evenly as possible (BASELINE C5: 128 layers ->
    128/N per GPU)."""
    if world > nz_global:
        raise ValueError(f"cannot split {nz_global} layers over {world} ranks")
    return rank * nz_global // world, (rank + 1) * nz_global // world, nz_global


def global_dof_index(slab: "Slab"):
    """Entries of the single-domain (world = 1) vector that this slab's
    vector holds, in slab order (value size included): y_slab = y_glob[idx]
    after the halo sums (partition independence)."""
    vs = slab.spec.element.value_size
    g = slab.global_index
    return (vs * g[:, None] + np.arange(vs)[None, :]).ravel()
