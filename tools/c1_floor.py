#!/usr/bin/env python
"""Latency floor of C1 (mass P2, 131k triangles, 8.4 MB compulsory) under the
same timing protocol as the sweep (L2 flushed, GPU spin, CUDA events):

* launch:   a fill of y (263k doubles): one launch + 2 MB of writes;
* stream:   a coalesced read of every compulsory byte (map, coordinates, u),
            summed into one value -- the HBM-bound ideal without indirection;
* gather:   y_c = sum_i u[map[i][c]] -- the dependent map -> u round trip
            with no arithmetic and no scatter (torch gather + sum);
* C1:       the operator (element_tensor kernel), accumulate protocol;
* C1 warm:  the operator back to back with the L2 NOT flushed (inputs
            L2-resident, as inside a solver loop);
* C1 graph: 100 applies captured in one CUDA graph, time per apply
            (launch overhead amortised, L2-resident: the throughput of the
            operator inside a captured solver iteration).

    python tools/c1_floor.py
"""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1903_08243_b200 as fe
    from paper_1903_08243_b200 import configs as C
    from paper_1903_08243_b200.harness import time_device

    prob = C.build_problem(C.get_config("C1"), 0)
    dev = torch.device("cuda")
    m, dm = prob.mesh, prob.dofmap
    h = fe.compile_and_load(fe.emit_for(prob.spec, fe.Target(), prob.rule))
    coords = torch.tensor(np.asarray(m.coords).ravel(), device=dev)
    mp = torch.tensor(np.asarray(dm.cell2dof, np.int32).ravel(), device=dev)
    h.bind(coords, mp, torch.tensor(np.asarray(m.cell2vert, np.int32).ravel(), device=dev),
           nglobal=dm.ndofs_global)
    u = torch.tensor(prob.u, device=dev)
    y = torch.zeros_like(u)
    soa = mp.view(-1, 6).t().contiguous().long()      # [6][nc], the kernel's SoA layout
    out = torch.empty(m.ncells, dtype=torch.float64, device=dev)
    rows = {}

    def best(fn, **kw):
        return min(time_device(fn, trials=30, warmup=3, **kw)) * 1e6

    rows["launch_fill_us"] = best(lambda: y.fill_(0.0))
    flat = [mp, coords, u]
    rows["stream_read_us"] = best(lambda: [t.sum() for t in flat])
    rows["stream_read_launches"] = len(flat)
    rows["gather_map_u_us"] = best(lambda: torch.sum(u[soa], dim=0, out=out))
    rows["c1_us"] = best(lambda: h.apply(u, y), setup=lambda: y.zero_())
    rows["c1_warm_us"] = best(lambda: h.apply(u, y), flush=False)
    try:
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            h.apply(u, y)                      # warm-up on the capture stream
            with torch.cuda.graph(g, stream=side):
                for _ in range(100):
                    h.apply(u, y)
        torch.cuda.current_stream().wait_stream(side)
        rows["c1_graph_us_per_apply"] = best(lambda: g.replay(), flush=False) / 100
    except Exception as e:  # capture unsupported: report why
        rows["c1_graph_error"] = str(e)[:120]
    rows["compulsory_MB"] = 8.41
    rows["hbm_time_us"] = 8.41e6 / 6547.8e9 * 1e6
    print(json.dumps({k: round(v, 2) if isinstance(v, float) else v for k, v in rows.items()}))


if __name__ == "__main__":
    main()
