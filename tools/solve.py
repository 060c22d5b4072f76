#!/usr/bin/env python
"""Matrix-free CG on one B200: solve A x = b, b = A u*, with
the sm_100a operator and an optional Jacobi preconditioner from
fe_diagonal; reports iterations, time per iteration (CUDA events) and the
error against u*.

    python tools/solve.py --config C2-P2 [--no-jacobi] [--rtol 1e-10]
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
    ap.add_argument("--config", default="C2-P2")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--rtol", type=float, default=1e-10)
    ap.add_argument("--maxiter", type=int, default=5000)
    ap.add_argument("--no-jacobi", action="store_true")
    args = ap.parse_args()
    import torch
    import paper_1903_08243_b200 as fe
    from paper_1903_08243_b200 import configs as C
    from paper_1903_08243_b200.solver import cg, jacobi

    prob = C.build_problem(C.get_config(args.config, args.n), 0)
    dev = torch.device("cuda")
    h = fe.compile_and_load(fe.emit_for(prob.spec, fe.Target(), prob.rule))
    h.bind(torch.tensor(np.asarray(prob.mesh.coords).ravel(), device=dev),
           torch.tensor(np.asarray(prob.dofmap.cell2dof, np.int32).ravel(), device=dev),
           torch.tensor(np.asarray(prob.mesh.cell2vert, np.int32).ravel(), device=dev),
           nglobal=prob.dofmap.ndofs_global)
    coef = None
    if prob.coef() is not None:
        coef = tuple(None if c is None else torch.tensor(c, device=dev) for c in prob.coef())
    A = lambda u, y: h.apply(u, y, coef=coef, overwrite=True)
    u = torch.tensor(prob.u, device=dev)
    b = torch.empty_like(u)
    A(u, b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    M = None if args.no_jacobi else jacobi(h.diagonal(coef=coef))
    e1.record()
    torch.cuda.synchronize()
    t_diag = e0.elapsed_time(e1) / 1e3
    e0.record()
    x, info = cg(A, b, rtol=args.rtol, maxiter=args.maxiter, precond=M, check_every=10)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    print(json.dumps({"config": args.config, "kernel": h.info["kernel"], "ndofs": prob.ndofs,
                      "jacobi": M is not None, "iterations": info.iterations,
                      "converged": info.converged, "final_rel_residual": info.residuals[-1],
                      "max_err_vs_manufactured": float((x - u).abs().max()),
                      "solve_s": round(t, 4), "ms_per_iteration": round(t / max(info.iterations, 1) * 1e3, 4),
                      "diagonal_setup_s": round(t_diag, 4)}))


if __name__ == "__main__":
    main()
