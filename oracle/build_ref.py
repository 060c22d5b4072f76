"""Build the REAL reference's CPU kernels into oracle/_ref/ (recipe).

The reference ships no C sources; its CPU implementation of the hot path is
the C it generates at run time (fevec.codegen.emit, codegen.py:345-447) and
compiles with ``cc {BENCH_FLAGS} -shared -fPIC`` (jit.py:27,90-111).  This
script imports fevec read-only from /root/reference/pkg/src, emits the
wrap_<form> source for the reference-supported configs the benchmark compares
against, and compiles it with the reference's own BENCH_FLAGS into
oracle/_ref/ (git-ignored; travels to the GPU box with the repo snapshot,
where /root/reference does not exist).  Nothing is copied into the tree.

  C1            mass, triangles, P2       (the reference runs it natively)
  C4-quad proxy elasticity, quads, Q1..Q4 (reference form eps(u):grad v =
                                           BASELINE elasticity with mu = 1/2,
                                           lambda = 0)

Each kernel is emitted for the scalar target and for vector-ext at width 8
(AVX-512).  oracle/_ref/manifest.json lists them.
"""

import json
import os
import subprocess
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")
CASES = [("mass", "tri", 2)] + [("elasticity", "quad", k) for k in (1, 2, 3, 4)]


def main():
    if not os.path.isdir(REF):
        print("reference not present; oracle/_ref left as is")
        return
    sys.path.insert(0, REF)
    from fevec.bench import emit_for
    from fevec.codegen import Target
    from fevec.elements import integrand_degree, operator_spec, quadrature_rule
    from fevec.jit import BENCH_FLAGS

    os.makedirs(OUT, exist_ok=True)
    manifest = []
    for form, cell, k in CASES:
        spec = operator_spec(form, cell, k)
        rule = quadrature_rule(cell, integrand_degree(spec))
        for target in (Target("scalar"), Target("vector-ext", 8)):
            unit = emit_for(spec, target, rule)
            stem = f"{form}_{cell}_p{k}_{target.kind}_w{target.width}"
            src = os.path.join(OUT, stem + ".c")
            so = os.path.join(OUT, stem + ".so")
            with open(src, "w") as f:
                f.write(unit.source)
            flags = [fl if fl != "-march=native" else "-march=x86-64-v4" for fl in BENCH_FLAGS]
            subprocess.run(["cc", *flags, "-shared", "-fPIC", "-o", so, src, "-lm"], check=True)
            manifest.append({"form": form, "cell": cell, "degree": k, "target": target.kind,
                             "width": target.width, "entry": unit.entry, "so": stem + ".so",
                             "args": [a[0] for a in unit.args], "flags": flags})
    with open(os.path.join(OUT, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print(f"built {len(manifest)} reference kernels into {OUT}")


if __name__ == "__main__":
    main()
