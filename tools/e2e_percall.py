#!/usr/bin/env python
"""Per-operator host-entry (fe_wrap_host) call time against bare copies of
the same pinned buffers: H2D of u alone, D2H of y alone, both concurrently.
One synchronous call at a time (the e2e step's FE_E2E_THREADS=1 case),
bench.py's own problems.  Explains the e2e number operator by operator."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import bench
import paper_1903_08243_b200 as fe


def best(fn, reps=4, setup=None):
    b = 1e9
    for _ in range(reps + 1):
        if setup:
            setup()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        b = min(b, time.perf_counter() - t0)
    return 1e3 * b


def main():
    names = sys.argv[1:] or bench.BASELINE_OPS
    dev = torch.device("cuda")
    tot = {}
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for name in names:
        op = bench.build_ops([name], 0, dev, 0, 1)[0]
        prob = op["prob"]
        u = torch.empty(op["ndofs"], dtype=torch.float64, pin_memory=True)
        u.numpy()[:] = prob.u
        y = torch.zeros(op["ndofs"], dtype=torch.float64, pin_memory=True)
        def pinned(a):
            if a is None:
                return None
            t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
            t[...] = a
            return t
        b = fe.make_bindings(prob.mesh, prob.dofmap, u.numpy(), y.numpy(), pinned(prob.mu), pinned(prob.lam),
                             state=pinned(getattr(prob, "state", None)))
        op["h"](0, op["C"], b)
        du, dy = torch.empty_like(op["u"]), torch.zeros_like(op["u"])

        def up():
            with torch.cuda.stream(s1):
                du.copy_(u, non_blocking=True)

        def down():
            with torch.cuda.stream(s2):
                y.copy_(dy, non_blocking=True)

        r = {"op": name, "mb": round(8e-6 * op["ndofs"], 1),
             "call_ms": best(lambda: op["h"](0, op["C"], b), setup=lambda: y.zero_()),
             "h2d_ms": best(up), "d2h_ms": best(down), "duplex_ms": best(lambda: (up(), down()))}
        r["call_over_duplex"] = round(r["call_ms"] / r["duplex_ms"], 2)
        for k in ("call_ms", "h2d_ms", "d2h_ms", "duplex_ms"):
            tot[k] = tot.get(k, 0.0) + r[k]
            r[k] = round(r[k], 3)
        print(json.dumps(r), flush=True)
        del op, du, dy, u, y, b
        torch.cuda.empty_cache()
    print(json.dumps({"total": {k: round(v, 2) for k, v in tot.items()}}))


if __name__ == "__main__":
    main()
