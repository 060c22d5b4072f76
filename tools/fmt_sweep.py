#!/usr/bin/env python
"""Compact view of sweep JSON lines (stdin or files): config kernel us frac."""
import json
import sys

src = [open(f) for f in sys.argv[1:]] or [sys.stdin]
for f in src:
    for line in f:
        line = line.strip()
        if line.startswith("{"):
            try:
                d = json.loads(line)
            except ValueError:
                print(line[:120])
                continue
            if "best_ms" in d:
                extra = ""
                if "best_ms_with_zero_fill" in d:
                    extra = f"   (with zero-fill {d['best_ms_with_zero_fill'] * 1000:8.1f} us {d['roofline_frac_with_zero_fill']:.3f})"
                print(f"{d['config']:12s} {d['kernel']:28s} {d['best_ms'] * 1000:9.1f} us  {d['roofline_frac']:.3f}{extra}")
            else:
                print(line[:160])
        elif line:
            print(line)
