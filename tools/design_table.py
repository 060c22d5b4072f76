#!/usr/bin/env python
"""Render DESIGN.md's per-operator results table from a bench.py JSON line
(the driver's protocol: median over steps, zero-fill inside the timed
call, cold clean L2), so DESIGN's fractions are exactly what the bench
printed.

    python tools/design_table.py profiles/r02/bench_final.log
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

LIMITER = {
    "C1": "latency: one wave of 131k cells, map -> coordinates/u dependent round trips; 8 MB problem (L2-resident)",
    "C2-P1": "gather latency (4 dependent loads per macro-cell) + 2.1M REDs; FP64 pipe ~40%",
    "C2-P2": "FP64 pipe + 15.7M REDs",
    "C2-P3": "DMMA pipe 66%, gather latency (long scoreboard), 81% of DMMA flops useful",
    "C2-P4": "DMMA pipe 76% (math-pipe throttle), 92% of DMMA flops useful",
    "C3-Q1": "thread per cell, dependent gather latency",
    "C3-Q2": "plane_t: 255 registers, 8 warps/SM",
    "C3-Q3": "plane: FP64 pipe 61%, 224 registers",
    "C3-Q4": "plane: registers (P^2 dof + output planes per thread)",
    "C3-Q5": "team kernel (36-thread teams, CTA barriers): FP64 pipe 45%, smem + barrier stalls",
    "C3-Q6": "team kernel (49-thread teams): FP64 pipe 57%",
    "C4-quad-Q1": "FP64",
    "C4-quad-Q2": "FP64",
    "C4-quad-Q3": "pair: FP64 pipe 52%, 255 registers, 8 warps/SM",
    "C4-quad-Q4": "pair: 255 registers, 12% occupancy",
    "C4-hex-Q1": "FP64",
    "C4-hex-Q2": "team kernel: FP64 pipe ~56%, smem round trips, 128 registers + spill",
    "C4-hex-Q3": "team kernel: 255 registers, 25-thread teams (1 per warp), smem store conflicts",
    "C5": "FP64 pipe 70%, 238 registers -> 8 warps/SM (dependent-FMA 'wait' stalls)",
}


def main(path):
    import paper_1903_08243_b200 as fe
    from paper_1903_08243_b200 import configs as C
    d = None
    for line in open(path).read().splitlines():
        if line.startswith("{"):
            d = json.loads(line)
    ms, fr = d["ms_per_operator_median"], d["roofline_frac_per_operator"]
    fe_exec = d.get("roofline_frac_vs_executed_flops", {})
    print("| config | kernel | cells | F/cell (SURVEY F) | median ms | GFLOP/s | fraction | limiter |")
    print("|---|---|---|---|---|---|---|---|")
    for name in d["config"]["operators"]:
        cfg = C.get_config(name)
        spec = fe.operator_spec(cfg.form, cfg.cell, cfg.degree)
        rule = fe.quadrature_rule(cfg.cell, cfg.qdegree)
        F = fe.flops_per_cell(spec, rule)
        Fs = fe.flops_per_cell(spec, rule, menu="survey")
        Fx = fe.flops_per_cell(spec, rule, menu="executed")
        ftxt = f"{F:,}" + (f" ({Fs:,})" if Fs != F else "") + (f"; executes {Fx:,}" if Fx < F else "")
        frac = f"**{fr[name]:.3f}**" + (f" ({fe_exec[name]:.3f} vs executed)" if name in fe_exec else "")
        g = F * cfg.ncells / (ms[name] * 1e-3) / 1e9
        print(f"| {name} | {d['kernel_per_operator'][name]} | {cfg.ncells:,} | {ftxt} | {ms[name]:.4f} | "
              f"{g:,.0f} | {frac} | {LIMITER.get(name, '')} |")
    print(f"| **step** | | | | {d['ms_per_step']:.3f} | {d['value']:,.0f} | "
          f"**{d['step_roofline_frac']:.3f}** | whole step, sum of T_roof / time |")


if __name__ == "__main__":
    main(sys.argv[1])
