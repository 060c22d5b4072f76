#!/usr/bin/env python
"""Apply one BASELINE config's operator a few times (a short command for ncu).

    python tools/profile_apply.py --config C2-P4 [--n 64] [--reps 3] [--time]
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2-P4")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--time", action="store_true", help="CUDA-event timing with L2 flush")
    ap.add_argument("--generic", action="store_true")
    args = ap.parse_args()
    import torch
    import paper_1903_08243_b200 as fe
    from paper_1903_08243_b200 import configs as C
    from paper_1903_08243_b200.harness import roofline_time, time_device

    prob = C.build_problem(C.get_config(args.config, args.n), 0)
    h = fe.compile_and_load(fe.emit_for(prob.spec, fe.Target(generic=args.generic), prob.rule))
    dev = torch.device("cuda")
    m, dm = prob.mesh, prob.dofmap
    h.bind(torch.as_tensor(np.array(m.coords).ravel(), device=dev),
           torch.as_tensor(np.array(dm.cell2dof, np.int32).ravel(), device=dev),
           torch.as_tensor(np.array(m.cell2vert, np.int32).ravel(), device=dev),
           nglobal=dm.ndofs_global)
    u = torch.as_tensor(prob.u, device=dev)
    y = torch.zeros_like(u)
    coef = None
    if prob.coef() is not None:
        coef = tuple(None if c is None else torch.as_tensor(c, device=dev) for c in prob.coef())
    fn = lambda: h.apply(u, y, coef=coef, overwrite=True)
    if args.time:
        # the reference's protocol (bench.py:196-200): accumulate into an
        # output zeroed outside the timer; the overwrite path (zero-fill
        # inside the timed call) is reported next to it
        ts = time_device(lambda: h.apply(u, y, coef=coef), trials=max(args.reps, 10), warmup=3,
                         setup=lambda: y.zero_())
        tw = time_device(fn, trials=max(args.reps, 10), warmup=3)
        F = fe.flops_per_cell(prob.spec, prob.rule) * m.ncells
        troof = roofline_time(prob.spec, m, dm, prob.rule)
        troof_s = roofline_time(prob.spec, m, dm, prob.rule, menu="survey")
        print(json.dumps({"config": args.config, "kernel": h.info["kernel"], "ncells": m.ncells,
                          "best_ms": min(ts) * 1e3, "median_ms": float(np.median(ts)) * 1e3,
                          "gflops": F / min(ts) / 1e9, "roofline_frac": troof / min(ts),
                          "best_ms_with_zero_fill": min(tw) * 1e3,
                          "roofline_frac_with_zero_fill": troof / min(tw),
                          "roofline_frac_survey_F": troof_s / min(ts)}))
    else:
        for _ in range(args.reps):
            fn()
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
