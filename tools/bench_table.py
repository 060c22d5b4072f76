#!/usr/bin/env python
"""Side-by-side per-operator table of bench.py JSON lines (A/B runs).

    python tools/bench_table.py gpurun_out/a.log gpurun_out/b.log [--md]
"""

import json
import sys


def load(path):
    for line in reversed(open(path).read().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    raise SystemExit(f"{path}: no JSON line")


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    md = "--md" in sys.argv
    runs = [load(p) for p in args]
    ops = list(runs[0]["ms_per_operator_median"])
    head = ["operator", "kernel"] + [f"ms[{i}]" for i in range(len(runs))] + [f"frac[{i}]" for i in range(len(runs))]
    rows = []
    for op in ops:
        r = [op, runs[0]["kernel_per_operator"].get(op, "")]
        r += [f"{d['ms_per_operator_median'].get(op, float('nan')):.4f}" for d in runs]
        r += [f"{d['roofline_frac_per_operator'].get(op, float('nan')):.3f}" for d in runs]
        rows.append(r)
    rows.append(["step", ""] + [f"{d['ms_per_step']:.3f}" for d in runs] +
                [f"{d.get('step_roofline_frac', float('nan')):.3f}" for d in runs])
    rows.append(["value GFLOP/s", ""] + [f"{d['value']:.0f}" for d in runs] + ["" for _ in runs])
    if md:
        print("| " + " | ".join(head) + " |")
        print("|" + "---|" * len(head))
        for r in rows:
            print("| " + " | ".join(r) + " |")
    else:
        w = [max(len(str(x)) for x in col) for col in zip(head, *rows)]
        for r in [head] + rows:
            print("  ".join(str(x).ljust(n) for x, n in zip(r, w)))


if __name__ == "__main__":
    main()
