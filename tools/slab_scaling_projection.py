#!/usr/bin/env python
"""Strong-scaling PROJECTION for the partitioned configs from one GPU.

Not a multi-GPU measurement (the box has one GPU): for N = 1, 2, 4, 8 the
slab a middle rank would own (nz/N cell layers of the config's fixed mesh,
two interfaces: the worst case) is built and the rank-local part of
DistributedOperator.apply is timed on this GPU with the bench's protocol
(cold L2, CUDA events, median): boundary layers first (overwrite + layer 0,
last layer), the pack of both interface planes (one kernel), the interior
layers, the unpack-add of the received planes (one kernel).  The NCCL send/recv itself is replaced by
nothing: its cost (message bytes below, ~2 us at NVLink peer bandwidth plus
~10 us of latency) is hidden behind the interior layers, which the table
shows next to it.  Projected efficiency = T_1 / (N T_N): what wave
quantisation, the three launches per apply and the pack/unpack cost, i.e. an
upper bound for the real run.

    python tools/slab_scaling_projection.py [C5 C2-P4 ...]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    import paper_1903_08243_b200 as fe
    from paper_1903_08243_b200.distributed import DistributedOperator
    from paper_1903_08243_b200.harness import time_device

    names = sys.argv[1:] or ["C5", "C2-P4", "C3-Q6", "C4-hex-Q3"]
    dev = torch.device("cuda")
    for name in names:
        t1 = None
        for world in (1, 2, 4, 8):
            rank = world // 2
            prob = bench.build_problem_for_rank(name, 0, rank, world)
            h = fe.compile_and_load(fe.emit_for(prob.spec, fe.Target(), prob.rule))
            m, dm = prob.mesh, prob.dofmap
            h.bind(torch.tensor(np.asarray(m.coords).ravel(), device=dev),
                   torch.tensor(np.asarray(dm.cell2dof, np.int32).ravel(), device=dev),
                   torch.tensor(np.asarray(m.cell2vert, np.int32).ravel(), device=dev),
                   nglobal=dm.ndofs_global)
            u = torch.tensor(prob.u, device=dev)
            y = torch.zeros_like(u)
            coef = None
            if prob.coef() is not None:
                coef = tuple(None if c is None else torch.tensor(c, device=dev) for c in prob.coef())
            rng = lambda uu, yy, a, b, ow: h.apply(uu, yy, a, b, coef=coef, overwrite=ow)
            op = DistributedOperator(prob, lambda uu, yy: h.apply(uu, yy, coef=coef, overwrite=True),
                                     rank, world, range_apply=rng)
            nc, lc = m.ncells, op.layer_cells

            def local_part():
                if world == 1:
                    h.apply(u, y, coef=coef, overwrite=True)
                    return
                if prob.boundary_first:
                    rng(u, y, 0, 2 * lc, True)
                    op._pack(y)
                    rng(u, y, 2 * lc, nc, False)
                else:
                    rng(u, y, 0, lc, True)
                    rng(u, y, nc - lc, nc, False)
                    op._pack(y)
                    rng(u, y, lc, nc - lc, False)
                op._unpack_add(y)

            def interior():
                if prob.boundary_first:
                    rng(u, y, 2 * lc, nc, False)
                else:
                    rng(u, y, lc, nc - lc, False)

            t = float(np.median(time_device(local_part, trials=10, warmup=3)))
            ti = float(np.median(time_device(interior, trials=10, warmup=3))) if world > 1 else t
            if world == 1:
                t1 = t
            row = {"config": name, "n_gpus": world, "slab_layers": int(m.grid[-1]), "cells": int(nc),
                   "ms_rank_local": round(t * 1e3, 4), "ms_interior_only": round(ti * 1e3, 4),
                   "interface_bytes_per_direction": int(op.n_if * 8) if world > 1 else 0,
                   "projected_efficiency": round(t1 / (world * t), 3)}
            print(json.dumps(row), flush=True)
            del h, u, y, op, prob
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
