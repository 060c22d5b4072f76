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
    "C1": "latency: one wave of 131k cells, map -> coordinates/u dependent round trips; 8 MB problem; a bare y-fill launch is 5 us of it; 3.9 us per apply inside a CUDA graph (profiles/r01/c1_floor.txt)",
    "C2-P1": "gather latency (long scoreboard 4.1 of 7.4 stall cycles/inst) + 2.1M REDs; FP64 pipe 51% while it runs; ~5 us of the 19.4 are launch + zero-fill; cp.async-pipelined variant slower (ab_macro_pipe.txt)",
    "C2-P2": "FP64 pipe + 15.7M REDs",
    "C2-P3": "DMMA pipe 61% + DFMA 13%, gather latency; 59 DMMA per 8 cells (92% useful) after the split-tuple packing",
    "C2-P4": "DMMA pipe 76% (math-pipe throttle), 92% of the DMMA flops useful",
    "C3-Q1": "thread per cell, FP64 pipe 59% while it runs; 21.1 us kernel + launch/zero-fill: dependent gather latency over 3.5 waves",
    "C3-Q2": "thread per cell (round 2): FP64 pipe 63%, 255 registers (268 B spill), gather exposed at kernel start",
    "C3-Q3": "plane kernel, 8-warp CTAs: FP64 pipe 61%, 206 registers",
    "C3-Q4": "plane kernel: FP64 pipe 57%, 244 registers (P^2 dof + output planes per thread)",
    "C3-Q5": "team kernel (36-thread teams, CTA barriers, register-prefetch gather), direct algorithm with even-odd 1D contractions (executes 58,788 flops)",
    "C3-Q6": "team kernel (49-thread teams), direct algorithm with even-odd 1D contractions (executes 97,644 flops); 128 registers with 112 B of spills, 135 R2UR",
    "C4-quad-Q1": "FP64",
    "C4-quad-Q2": "FP64",
    "C4-quad-Q3": "even-odd pair kernel (select-free): 255 registers, 2 warps/SMSP, gather exposed; executes 4,124 flops",
    "C4-quad-Q4": "even-odd pair kernel (select-free, 2,632 instructions; executes 6,364 flops): 255 registers, 2 warps/SMSP, gather exposed; the 42 us zero-fill of its 269 MB y is 9% of the apply",
    "C4-hex-Q1": "FP64",
    "C4-hex-Q2": "team kernel (16-thread teams, 9 / 12 of 16 lanes busy in the z / y stages): FP64 pipe 57%",
    "C4-hex-Q3": "team kernel (25-thread teams, one per warp: 78% of the lanes; 16 / 20 of 25 in the z / y stages), even-odd contractions: FP64 pipe 58%",
    "C5": "FP64 pipe 73%, 254 registers -> 8 warps/SM; executes fewer flops than the menu's F (0.53 of the roof counted on executed flops)",
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
