#!/usr/bin/env python
"""Pinned host <-> device copy bandwidth (the e2e path's floor): H2D, D2H,
and both directions at once, 136 MB buffers (C2-P4's u)."""
import json

import torch


def main():
    n = 17_000_000
    h1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d1 = torch.empty(n, dtype=torch.float64, device="cuda")
    d2 = torch.empty(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}

    def timed(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(reps):
            e0.record()
            fn()
            torch.cuda.synchronize()
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        return best

    b = n * 8
    out["h2d_GBs"] = b / timed(lambda: d1.copy_(h1, non_blocking=True)) / 1e9
    out["d2h_GBs"] = b / timed(lambda: h1.copy_(d1, non_blocking=True)) / 1e9

    def both():
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    out["duplex_GBs_total"] = 2 * b / timed(both) / 1e9
    print(json.dumps({k: round(v, 1) for k, v in out.items()}))


if __name__ == "__main__":
    main()
