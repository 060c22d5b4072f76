#!/usr/bin/env python
"""Render tools/sweep.sh output (JSON lines) as a markdown table with the
frozen-flop roofline of every BASELINE config.

    python tools/render_sweep.py profiles/r01/sweep_v4.jsonl
"""

import json
import sys

ROOF = {  # F per cell (frozen), bound
}


def main(path):
    rows = [json.loads(l) for l in open(path) if l.strip().startswith("{")]
    print("| config | kernel | cells | time (µs, best of 20, L2 flushed) | GFLOP/s (frozen F) | roofline fraction |")
    print("|---|---|---|---|---|---|")
    for r in rows:
        if r.get("error"):
            print(f"| {r['config']} | error | | | | |")
            continue
        print(f"| {r['config']} | {r['kernel']} | {r['ncells']:,} | {r['best_ms'] * 1e3:.1f} | "
              f"{r['gflops']:.0f} | {r['roofline_frac']:.3f} |")


if __name__ == "__main__":
    main(sys.argv[1])
