#!/usr/bin/env python
"""Benchmark of the matrix-free FE operator action on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2] [--seed S]

Workload (BASELINE.json configs[1], the first config the metric is quoted on
that is not the reference's own CPU case): Helmholtz action on P1..P4
tetrahedra, 64^3 cubes x 6 Kuhn tets (1,572,864 cells), interior vertices
jittered +-0.1h, u ~ U[-1,1] (seeded synthetic inputs; BASELINE has no
dataset).  One STEP applies the four operators P1, P2, P3, P4 once each
(y = A_k u_k, y zero-filled inside the step).  The L2 is flushed between
steps (outside the CUDA-event pairs).

value  = sum_k F_k C / sum of step times, in GFLOP/s with the FROZEN flop
         counts F_k of SURVEY.md Appendix B (metric "FP64 GFLOP/s ...");
e2e    = the same metric through the reference-facing host call
         (fe_wrap_host: pinned host u/y -> device, apply, y -> host);
roofline = the dominant kernel (P4) against the measured FP64 peak.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.094        # measured DMMA peak, profiles/r01_fp64_peaks.json
FP64_DFMA_TFLOPS = 34.162        # measured DFMA peak, same file


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "source": "fallback"}


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML)
# ---------------------------------------------------------------------------


class ClockSampler:
    REASONS = {
        0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting",
    }

    def __init__(self, index=0, period=0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------

WORKLOADS = {
    "C2": ["C2-P1", "C2-P2", "C2-P3", "C2-P4"],
    "C1": ["C1"],
    "C3": [f"C3-Q{k}" for k in range(1, 7)],
    "C4": [f"C4-quad-Q{k}" for k in range(1, 5)] + [f"C4-hex-Q{k}" for k in range(1, 4)],
    "C5": ["C5"],
}


def build_ops(names, seed, device):
    """Problems, plans and resident device buffers for every config."""
    import torch
    import paper_1903_08243_b200 as fe
    from paper_1903_08243_b200 import configs as C
    ops = []
    for name in names:
        prob = C.build_problem(C.get_config(name), seed)
        h = fe.compile_and_load(fe.emit_for(prob.spec, fe.Target(), prob.rule))
        m, dm = prob.mesh, prob.dofmap
        h.bind(torch.as_tensor(np.ascontiguousarray(m.coords).ravel(), device=device),
               torch.as_tensor(np.ascontiguousarray(dm.cell2dof, np.int32).ravel(), device=device),
               None, nglobal=dm.ndofs_global)
        u = torch.as_tensor(prob.u, device=device)
        y = torch.zeros_like(u)
        coef = None
        if prob.mu is not None:
            coef = (torch.as_tensor(prob.mu, device=device), torch.as_tensor(prob.lam, device=device))
        F = fe.flops_per_cell(prob.spec, prob.rule)
        B = fe.bytes_per_cell(prob.spec, m, dm)
        ops.append(dict(name=name, prob=prob, h=h, u=u, y=y, coef=coef, F=F, B=B,
                        C=m.ncells, ndofs=prob.ndofs))
    return ops


def parity_sample(ops, ncheck=3000):
    """rel-L2 of the GPU result against the CPU oracle on a cell sub-range
    of every operator (the full-size oracle is too slow for a bench run;
    full-size parity is covered by tests/)."""
    import torch
    from oracle import fe_oracle as fo
    worst = 0.0
    for op in ops:
        prob = op["prob"]
        end = min(ncheck, op["C"])
        yd = torch.zeros_like(op["u"])
        op["h"].apply(op["u"], yd, 0, end, coef=op["coef"])
        torch.cuda.synchronize()
        P = fo.Problem(prob.spec.form, prob.spec.cell.kind, prob.spec.element.degree,
                       prob.rule.exactness_degree, prob.spec.params)
        ref = fo.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u,
                          prob.mu, prob.lam, 0, end)
        worst = max(worst, fo.rel_l2(yd.cpu().numpy(), ref))
    return worst


def cpu_baseline(ops, budget_s=12.0):
    """The oracle port (numpy, 1 thread) on a bounded sample of every
    operator's cells; reported in the metric's unit (frozen flops)."""
    from oracle import fe_oracle as fo
    tot_flop, tot_t, desc = 0.0, 0.0, []
    per = budget_s / len(ops)
    for op in ops:
        prob = op["prob"]
        P = fo.Problem(prob.spec.form, prob.spec.cell.kind, prob.spec.element.degree,
                       prob.rule.exactness_degree, prob.spec.params)
        n = 256
        while True:
            t0 = time.perf_counter()
            fo.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u,
                        prob.mu, prob.lam, 0, n)
            dt = time.perf_counter() - t0
            if dt > per / 4 or n >= op["C"]:
                break
            n = min(op["C"], n * 4)
        tot_flop += op["F"] * n
        tot_t += dt
        desc.append(f"{op['name']}:{n} cells")
    return {"value": tot_flop / tot_t / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "port",
            "sample": "numpy oracle (oracle/fe_oracle.py) on the first cells of each operator: "
                      + ", ".join(desc)}


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1903_08243_b200.harness import L2Flusher

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    names = WORKLOADS[args.config]
    ops = build_ops(names, args.seed, dev)
    # element partition across ranks: contiguous cell blocks (weak: every rank
    # owns a full-size mesh's worth of cells of its own replica)
    parity = parity_sample(ops) if rank == 0 else None
    flush = L2Flusher(local)
    stream = torch.cuda.current_stream()

    def step(events=None):
        for i, op in enumerate(ops):
            if events is not None:
                events[i][0].record(stream)
            op["h"].apply(op["u"], op["y"], coef=op["coef"], overwrite=True)
            if events is not None:
                events[i][1].record(stream)

    for _ in range(args.warmup):
        flush()
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    per_op = np.zeros(len(ops))
    step_times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in ops]
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            step(ev)
            s1.record(stream)
            s1.synchronize()
            step_times.append(s0.elapsed_time(s1) * 1e-3)
            per_op += [e0.elapsed_time(e1) * 1e-3 for e0, e1 in ev]
    torch.cuda.synchronize()
    t_total = float(sum(step_times))
    if world > 1:
        t = torch.tensor([t_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_total = float(t.item())
        dist.barrier()
    flop_step = sum(op["F"] * op["C"] for op in ops)
    dofs_step = sum(op["ndofs"] for op in ops)
    value = world * flop_step * args.steps / t_total / 1e9

    # e2e through the reference-facing host entry (pinned host buffers)
    e2e = None
    if rank == 0:
        e2e = run_e2e(ops, args)
    if rank == 0:
        peaks = measured_peaks()
        dom = int(np.argmax([op["F"] * op["C"] for op in ops]))
        t_dom = per_op[dom] / args.steps
        achieved = ops[dom]["F"] * ops[dom]["C"] / t_dom / 1e12
        troof = [max(op["F"] * op["C"] / (FP64_PEAK_TFLOPS * 1e12),
                     op["B"] * op["C"] / (peaks["hbm_gbs"] * 1e9)) for op in ops]
        line = {
            "metric": "FP64 GFLOP/s per matrix-free operator action (frozen flop counts, SURVEY.md App. B)",
            "value": round(value, 3),
            "unit": "GFLOP/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(t_total / args.steps * 1e3, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded jittered structured mesh, u~U[-1,1])",
            "config": {
                "workload": f"{args.config}: " + ", ".join(op["name"] for op in ops)
                            + (" helmholtz Pk tet 64^3x6 jittered" if args.config == "C2" else ""),
                "cells_per_operator": [op["C"] for op in ops],
                "dofs_per_operator": [op["ndofs"] for op in ops],
                "seed": args.seed,
                "l2": "flushed (2x L2 write) between steps, outside the event pairs",
                "parallelism": f"replica x{world}" if world > 1 else "1 GPU",
            },
            "gdofs_per_s": round(world * dofs_step * args.steps / t_total / 1e9, 3),
            "roofline_frac_per_operator": {op["name"]: round(troof[i] / (per_op[i] / args.steps), 4)
                                           for i, op in enumerate(ops)},
            "ms_per_operator": {op["name"]: round(per_op[i] / args.steps * 1e3, 4)
                                for i, op in enumerate(ops)},
            "kernel_per_operator": {op["name"]: op["h"].info["kernel"] for op in ops},
            "step_roofline_frac": round(sum(troof) / (t_total / args.steps), 4),
            "parity_rel_l2_sample": parity,
            "roofline": {
                "bound": "fp64",
                "kernel": ops[dom]["name"] + ":" + ops[dom]["h"].info["kernel"],
                "achieved": round(achieved, 4),
                "peak": FP64_PEAK_TFLOPS,
                "peak_source": "measured FP64 DMMA peak on this pool's B200 (profiles/r01_fp64_peaks.json); "
                               "MEASURED_PEAKS.json has no FP64 entry",
                "unit": "TFLOP/s",
                "frac": round(achieved / FP64_PEAK_TFLOPS, 4),
                "traffic": None,
                "algorithmic_flop_per_launch": ops[dom]["F"] * ops[dom]["C"],
            },
            "e2e": e2e,
            "gpu_launches": len(ops) * args.steps,
            "clocks": clk.summary(),
        }
        line["cpu_baseline"] = cpu_baseline(ops) if world == 1 else None
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(ops, args):
    """Same metric through the public host API (GpuKernelHandle.__call__ with
    numpy bindings -> fe_wrap_host): every step uploads u and y from pinned
    host memory, applies, and downloads y."""
    import torch
    import paper_1903_08243_b200 as fe
    hb = []
    for op in ops:
        prob = op["prob"]
        u = torch.empty(op["ndofs"], dtype=torch.float64, pin_memory=True).numpy()
        u[:] = prob.u
        out = torch.zeros(op["ndofs"], dtype=torch.float64, pin_memory=True).numpy()
        b = fe.make_bindings(prob.mesh, prob.dofmap, u, out, prob.mu, prob.lam)
        op["h"].rebind()
        hb.append((op, b))
    steps = max(2, min(args.steps, 5))
    for op, b in hb:            # warm-up (binds the host mesh once)
        b["dat0"][:] = 0.0
        op["h"](0, op["C"], b)
    t = 0.0
    for _ in range(steps):
        for op, b in hb:
            b["dat0"][:] = 0.0
            t0 = time.perf_counter()
            op["h"](0, op["C"], b)
            t += time.perf_counter() - t0
    flop = sum(op["F"] * op["C"] for op in ops) * steps
    h2d = sum(2 * 8 * op["ndofs"] for op in ops)
    d2h = sum(8 * op["ndofs"] for op in ops)
    return {"value": round(flop / t / 1e9, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps,
            "path": "GpuKernelHandle(start,end,bindings) -> fe_wrap_host (pinned host buffers)"}


def run_reference(args):
    """--impl reference: the reference's CPU algorithm on the box's host cores.
    The reference has no code path for tetrahedra (elements.py:63-72), so the
    arm runs the oracle restatement of reference.py (oracle/fe_oracle.py) over
    a bounded sample of every operator, one process per host core."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from concurrent.futures import ProcessPoolExecutor
    from paper_1903_08243_b200 import configs as C
    import paper_1903_08243_b200 as fe
    cores = len(os.sched_getaffinity(0))
    names = WORKLOADS[args.config]
    sample_cells = 2048 * cores
    t_steps = []
    flops = 0.0
    jobs = []
    for name in names:
        prob = C.build_problem(C.get_config(name), args.seed)
        F = fe.flops_per_cell(prob.spec, prob.rule)
        jobs.append((name, prob, F))
    with ProcessPoolExecutor(max_workers=cores) as ex:
        for it in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            step_flop = 0.0
            for name, prob, F in jobs:
                n = min(sample_cells, prob.mesh.ncells)
                cuts = np.linspace(0, n, cores + 1).astype(int)
                futs = [ex.submit(_oracle_chunk, name, args.seed, int(a), int(b))
                        for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
                for f in futs:
                    f.result()
                step_flop += F * n
            dt = time.perf_counter() - t0
            if it >= args.warmup:
                t_steps.append(dt)
                flops += step_flop
    value = flops / sum(t_steps) / 1e9
    line = {
        "impl": "reference",
        "metric": "FP64 GFLOP/s per matrix-free operator action (frozen flop counts, SURVEY.md App. B)",
        "value": round(value, 4), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(np.mean(t_steps) * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded jittered structured mesh, u~U[-1,1])",
        "config": {"workload": f"{args.config}: " + ", ".join(names), "seed": args.seed,
                   "sample_cells_per_operator": sample_cells},
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": cores, "kind": "port",
                         "sample": f"first {sample_cells} cells of each operator, split over {cores} "
                                   "processes (numpy restatement of reference.py; the reference "
                                   "has no tetrahedral code path)"},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


_CACHE = {}


def _oracle_chunk(name, seed, a, b):
    from oracle import fe_oracle as fo
    from paper_1903_08243_b200 import configs as C
    if name not in _CACHE:
        prob = C.build_problem(C.get_config(name), seed)
        P = fo.Problem(prob.spec.form, prob.spec.cell.kind, prob.spec.element.degree,
                       prob.rule.exactness_degree, prob.spec.params)
        _CACHE[name] = (prob, P)
    prob, P = _CACHE[name]
    fo.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u,
                prob.mu, prob.lam, a, b)
    return b - a


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
