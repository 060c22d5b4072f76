#!/usr/bin/env python
"""SASS instruction histograms of the hot kernels (cuobjdump -sass on the
built library), one block per kernel: FP64 math (DFMA/DMUL/DADD/DMMA),
memory (LDG/LDS/STS/REDG/LDGSTS), control (BAR/SHFL/BRA) -- the evidence
that the kernels are what DESIGN.md says (DMMA on the modal kernel, REDG
scatters, no library calls).

    python tools/sass_hist.py [--lib paper_1903_08243_b200/libfeb200.so] [--out FILE]
"""

import argparse
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# mangled-name fragments of the kernels the BASELINE configs select
HOT = ["affine_et_kernel", "macro_split_kernel", "affine_split_kernel", "dmma_modal_kernel",
       "macro_pipe_kernel", "hexq1_lap_kernel", "hexq2_lap_kernel", "plane1_kernel", "plane_kernel", "tensor_kernel", "quad_const_kernel",
       "pair_kernel", "quad_vtx_kernel", "k_zero_pdl"]
CLASSES = ["DMMA", "DFMA", "DMUL", "DADD", "MUFU", "LDG", "LDGSTS", "LDS", "STS", "REDG", "ATOMG",
           "LDC", "LDCU", "R2UR", "SHFL", "BAR", "BRA", "ACQBULK", "PREEXIT", "IMAD", "IADD3", "LOP3", "ISETP", "MOV"]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
        return out.splitlines()
    except OSError:
        return names


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_1903_08243_b200", "libfeb200.so"))
    ap.add_argument("--out", default=None)
    ap.add_argument("--all", action="store_true", help="every kernel, not only the hot families")
    args = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", args.lib], capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if cur and m:
            op = m.group(1)
            funcs[cur][op] += 1
            funcs[cur]["_total"] += 1
            if op == "DMMA":
                funcs[cur]["DMMA" + (m.group(2) or "")] += 0
    names = list(funcs)
    pretty = demangle(names)
    lines = [f"# cuobjdump -sass {os.path.relpath(args.lib, ROOT)}: static instruction counts per kernel",
             "# columns: " + " ".join(CLASSES) + " total"]
    for raw, nice in zip(names, pretty):
        if not args.all and not any(h in raw for h in HOT):
            continue
        c = funcs[raw]
        lines.append(f"== {nice[:200]}")
        lines.append("   " + " ".join(f"{k}={c.get(k, 0)}" for k in CLASSES) + f" total={c['_total']}")
    text = "\n".join(lines) + "\n"
    if args.out:
        with open(args.out, "w") as f:
            f.write(text)
    print(text, end="")


if __name__ == "__main__":
    main()
