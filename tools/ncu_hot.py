#!/usr/bin/env python
"""Top SASS lines of an ncu --set full report by warp-stall samples (the
source page with --import-source / -lineinfo): where each kernel's warps
wait, instruction by instruction.

    python tools/ncu_hot.py report.ncu-rep [--top 25]
"""

import csv
import io
import subprocess
import sys


def main(path, top):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if not rows:
        print("(no source page)")
        return
    while rows and "Address" not in rows[0]:
        rows = rows[1:]                      # "Kernel Name" preamble rows
    if not rows:
        print("(no source rows)")
        return
    hdr = rows[0]
    samp = [i for i, h in enumerate(hdr) if "Sampling" in h and "All" in h]
    src = [i for i, h in enumerate(hdr) if h.lower() in ("source", "sass")]
    if not samp or not src:
        print("columns:", hdr)
        return
    si, ci = samp[0], src[0]
    body = []
    for r in rows[1:]:
        try:
            body.append((float(r[si] or 0), r[ci].strip()))
        except (ValueError, IndexError):
            continue
    total = sum(v for v, _ in body) or 1.0
    ops = {}
    for v, s in body:
        op = s.split()[0] if s else "?"
        if op.startswith("@"):
            op = s.split()[1] if len(s.split()) > 1 else op
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0.0) + v
    print(f"# {path}: {int(total)} stall samples; by opcode: " +
          ", ".join(f"{k} {100 * v / total:.1f}%" for k, v in sorted(ops.items(), key=lambda t: -t[1])[:12]))
    for v, s in sorted(body, reverse=True)[:top]:
        print(f"{100 * v / total:6.2f}%  {s}")


if __name__ == "__main__":
    top = 25
    args = sys.argv[1:]
    if "--top" in args:
        top = int(args[args.index("--top") + 1])
        args = [a for a in args if a not in ("--top", str(top))]
    for p in args:
        main(p, top)
