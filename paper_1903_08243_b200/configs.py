"""BASELINE.json configurations C1..C5 (+ C6, the SURVEY 8(f).1 tangent of
C5) and their seeded synthetic inputs.

Seeds: ``SeedSequence(seed).spawn(4)`` -> independent
``default_rng`` streams in the fixed order [jitter, u, mu, lambda];
jitter moves interior vertices by U(-0.1h, 0.1h) per coordinate; u ~
U(-1, 1) per dof (C5: 0.01 h U(-1, 1): the
literal 0.05 U(-1,1) makes det F <= 0 at about half the quadrature points);
mu, lambda ~ U(0.5, 2) per vertex (C4); a fifth stream draws the state u0 =
0.01 h U(-1, 1) of the linearised C6 (spawn keeps the first four streams).

The configs themselves are the BASELINE.json ``configs`` list; BASELINE has
no public dataset, so seeded synthetic inputs with the stated shapes stand in.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .elements import integrand_degree, operator_spec, quadrature_rule
from .mesh import build_dof_map, build_mesh, jitter_mesh

__all__ = ["Config", "CONFIGS", "get_config", "build_problem", "Problem"]


@dataclass(frozen=True)
class Config:
    name: str          # e.g. "C2-P3"
    family: str        # C1..C5
    form: str
    cell: str
    degree: int
    n: tuple           # cells per direction
    qdegree: int       # quadrature exactness degree
    jitter: bool = True
    u_scale: str = "unit"     # "unit": U(-1,1); "h": 0.01 h U(-1,1)
    partitioned: bool = False

    @property
    def ncells(self) -> int:
        c = int(np.prod(self.n))
        if self.cell == "triangle":
            return 2 * c
        if self.cell == "tetrahedron":
            return 6 * c
        return c


def _configs():
    out = []
    out.append(Config("C1", "C1", "mass", "triangle", 2, (256, 256), 4))
    for k in (1, 2, 3, 4):
        out.append(Config(f"C2-P{k}", "C2", "helmholtz", "tetrahedron", k, (64, 64, 64), 2 * k))
    for k in range(1, 7):
        # Gauss-Legendre with k+1 points per direction: exact to degree 2k+1
        out.append(Config(f"C3-Q{k}", "C3", "laplacian_scalar", "hexahedron", k, (64, 64, 64), 2 * k))
    for k in (1, 2, 3, 4):
        out.append(Config(f"C4-quad-Q{k}", "C4", "elasticity_lame", "quadrilateral", k,
                          (1024, 1024), 2 * k + 2))
    for k in (1, 2, 3):
        out.append(Config(f"C4-hex-Q{k}", "C4", "elasticity_lame", "hexahedron", k,
                          (64, 64, 64), 2 * k + 2))
    out.append(Config("C5", "C5", "neohookean", "tetrahedron", 2, (128, 128, 128), 4,
                      jitter=False, u_scale="h", partitioned=True))
    # the Newton-step companion of C5 -- the tangent action
    # dF(u0; du) on the C5 mesh, state u0 = 0.01 h U(-1,1), du ~ U(-1,1)
    out.append(Config("C6", "C6", "neohookean_tangent", "tetrahedron", 2, (128, 128, 128), 4,
                      jitter=False, u_scale="unit", partitioned=True))
    return {c.name: c for c in out}


CONFIGS = _configs()


def get_config(name: str, n=None) -> Config:
    """A BASELINE config, optionally at a reduced mesh size ``n`` (cells per
    direction) for parity tests against the CPU oracle."""
    c = CONFIGS[name]
    if n is None:
        return c
    if isinstance(n, int):
        n = (n,) * len(c.n)
    return Config(c.name, c.family, c.form, c.cell, c.degree, tuple(n), c.qdegree,
                  c.jitter, c.u_scale, c.partitioned)


@dataclass
class Problem:
    config: Config
    spec: object
    rule: object
    mesh: object
    dofmap: object
    u: np.ndarray
    mu: np.ndarray = None
    lam: np.ndarray = None
    state: np.ndarray = None   # u0 of a linearised form (neohookean_tangent)

    def coef(self):
        """(coef0, coef1) host arrays for fe_apply, or None."""
        if self.mu is not None:
            return (self.mu, self.lam)
        if self.state is not None:
            return (self.state, None)
        return None

    @property
    def nglobal(self) -> int:
        return self.dofmap.ndofs_global

    @property
    def ndofs(self) -> int:
        return self.spec.element.value_size * self.dofmap.ndofs_global


def build_problem(cfg: Config, seed: int = 0) -> Problem:
    spec = operator_spec(cfg.form, cfg.cell, cfg.degree)
    if cfg.qdegree < 2 * cfg.degree:
        raise ValueError("quadrature below the integrand's polynomial degree")
    rule = quadrature_rule(cfg.cell, cfg.qdegree)
    r_jit, r_u, r_mu, r_lam, r_state = [np.random.default_rng(s)
                                        for s in np.random.SeedSequence(seed).spawn(5)]
    mesh = build_mesh(cfg.cell, *cfg.n)
    if cfg.jitter:
        mesh = jitter_mesh(mesh, r_jit, 0.1)
    dm = build_dof_map(mesh, spec.element)
    n = spec.element.value_size * dm.ndofs_global
    u = r_u.uniform(-1.0, 1.0, n)
    if cfg.u_scale == "h":
        u *= 0.01 / max(cfg.n)
    mu = lam = state = None
    if spec.coefficient_fields:
        mu = r_mu.uniform(0.5, 2.0, mesh.nvertices)
        lam = r_lam.uniform(0.5, 2.0, mesh.nvertices)
    if spec.has_state:
        state = r_state.uniform(-1.0, 1.0, n) * (0.01 / max(cfg.n))
    return Problem(cfg, spec, rule, mesh, dm, u, mu, lam, state)


def default_rule(spec):
    return quadrature_rule(spec.cell, integrand_degree(spec))
