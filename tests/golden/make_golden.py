"""Generate golden vectors from the REAL reference implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference ``fevec`` package read-only from
``/root/reference/pkg/src`` and writes ``tests/golden/reference_2d.npz`` and
``tests/golden/c1_full.npz``.  The GPU box never runs this script; the
fixtures travel with the repo.

Inputs are built with the reference's own ``build_mesh`` and
``build_dof_map`` (``mesh.py:29-115``), jittered with the seeded protocol the
B200 package uses (SeedSequence(seed).spawn(4) -> [jitter, u, mu, lambda];
interior vertices moved by U(-0.1h, 0.1h) per coordinate), and the outputs
are ``fevec.reference.assemble_reference`` (``reference.py:18-83``) with the
reference's ``quadrature_rule(cell, integrand_degree(spec))``.
"""

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def jitter(coords, n, rng, amp=0.1):
    h = 1.0 / n
    x = np.array(coords, dtype=float)
    delta = rng.uniform(-1.0, 1.0, size=x.shape) * (amp * h)
    interior = np.all((x > 0.0) & (x < 1.0), axis=1)
    x[interior] += delta[interior]
    return x


def streams(seed):
    return [np.random.default_rng(s) for s in np.random.SeedSequence(seed).spawn(4)]


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    sys.path.insert(0, REF)
    from fevec.elements import integrand_degree, operator_spec, quadrature_rule
    from fevec.mesh import Mesh, build_dof_map, build_mesh
    from fevec.reference import assemble_reference

    out = {}
    names = []
    nx, ny = 4, 3
    for form in ("mass", "helmholtz", "laplacian", "elasticity"):
        for cell in ("tri", "quad"):
            for degree in (1, 2, 3, 4):
                seed = 100 * degree + len(names)
                rj, ru, _, _ = streams(seed)
                spec = operator_spec(form, cell, degree)
                rule = quadrature_rule(cell, integrand_degree(spec))
                m0 = build_mesh(cell, nx, ny)
                # jitter uses h = 1/nx for x and 1/ny for y as in the package
                x = np.array(m0.coords)
                delta = rj.uniform(-1.0, 1.0, size=x.shape) * (0.1 * np.array([1 / nx, 1 / ny]))
                interior = np.all((x > 0.0) & (x < 1.0), axis=1)
                x[interior] += delta[interior]
                mesh = Mesh(x, m0.cell2vert, m0.cell)
                dm = build_dof_map(mesh, spec.element)
                u = ru.uniform(-1.0, 1.0, spec.element.value_size * dm.ndofs_global)
                y = assemble_reference(spec, mesh, dm, rule, u)
                key = f"{form}_{cell}_{degree}"
                names.append(key)
                out[key + "/seed"] = np.array(seed)
                out[key + "/coords"] = x
                out[key + "/cell2vert"] = np.asarray(m0.cell2vert, np.int32)
                out[key + "/cell2dof"] = np.asarray(dm.cell2dof, np.int32)
                out[key + "/u"] = u
                out[key + "/y"] = y
                out[key + "/qpoints"] = np.asarray(rule.points)
                out[key + "/qweights"] = np.asarray(rule.weights)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "reference_2d.npz"), **out)

    # C1 at full size: mass P2 triangles, 256x256 squares, jittered, seed 0
    spec = operator_spec("mass", "tri", 2)
    rule = quadrature_rule("tri", integrand_degree(spec))
    m0 = build_mesh("tri", 256, 256)
    rj, ru, _, _ = streams(0)
    x = jitter(m0.coords, 256, rj)
    mesh = Mesh(x, m0.cell2vert, m0.cell)
    dm = build_dof_map(mesh, spec.element)
    u = ru.uniform(-1.0, 1.0, dm.ndofs_global)
    y = assemble_reference(spec, mesh, dm, rule, u)
    np.savez_compressed(
        os.path.join(HERE, "c1_full.npz"),
        y=y,
        input_digest=np.array(digest(x, np.asarray(dm.cell2dof, np.int32), u)),
        ndofs=np.array(dm.ndofs_global),
    )
    print(f"wrote {len(names)} 2D cases and the C1 full-size vector")


if __name__ == "__main__":
    main()
