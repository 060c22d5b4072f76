#!/usr/bin/env python
"""Host-entry (fe_wrap_host) time per C2 operator against its PCIe floor:
wall time of one synchronous call with dat0 zero and with dat0 nonzero,
next to the duplex copy of u up and y down alone (the same pinned buffers,
two streams).  Explains bench.py's e2e number."""
import json
import time

import numpy as np
import torch

import paper_1903_08243_b200 as fe
from paper_1903_08243_b200 import configs as C


def wall(fn, reps=10, setup=None):
    best = 1e9
    for _ in range(reps + 1):
        if setup:
            setup()
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    rows = []
    for name in ["C2-P1", "C2-P2", "C2-P3", "C2-P4"]:
        prob = C.build_problem(C.get_config(name), seed=0)
        h = fe.compile_and_load(fe.emit_for(prob.spec, fe.Target(), prob.rule))
        u = torch.empty(prob.ndofs, dtype=torch.float64, pin_memory=True).numpy()
        u[:] = prob.u
        y = torch.zeros(prob.ndofs, dtype=torch.float64, pin_memory=True).numpy()
        b = fe.make_bindings(prob.mesh, prob.dofmap, u, y)

        def call():
            h(0, prob.mesh.ncells, b)

        t_zero = wall(call, setup=lambda: y.__setitem__(slice(None), 0.0))
        t_nonzero = wall(call, setup=lambda: y.__setitem__(slice(None), 1.0))
        t_fill = 0.0
        du = torch.empty(prob.ndofs, dtype=torch.float64, device="cuda")
        dy = torch.empty(prob.ndofs, dtype=torch.float64, device="cuda")
        tu, ty = torch.from_numpy(u), torch.from_numpy(y)
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

        def duplex():
            with torch.cuda.stream(s1):
                du.copy_(tu, non_blocking=True)
            with torch.cuda.stream(s2):
                ty.copy_(dy, non_blocking=True)
            torch.cuda.synchronize()

        t_duplex = wall(duplex)
        rows.append({"op": name, "ndofs": prob.ndofs, "mb": 8e-6 * prob.ndofs,
                     "call_zero_ms": 1e3 * (t_zero - t_fill), "call_nonzero_ms": 1e3 * (t_nonzero - t_fill),
                     "duplex_copy_ms": 1e3 * t_duplex})
        print(json.dumps(rows[-1]), flush=True)
    tot = {k: sum(r[k] for r in rows) for k in ["call_zero_ms", "call_nonzero_ms", "duplex_copy_ms"]}
    print(json.dumps({"total": tot}))


if __name__ == "__main__":
    main()
