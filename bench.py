#!/usr/bin/env python
"""Benchmark of the matrix-free FE operator action on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2] [--seed S]

Workload (BASELINE.json configs[1] -- configs[0] is the reference's own CPU
case): the Helmholtz action on P1..P4 tetrahedra, 64^3 cubes x 6 Kuhn tets
(1,572,864 cells) per GPU, interior vertices jittered +-0.1h, u ~ U[-1,1]
(seeded synthetic inputs; BASELINE names no dataset).  One STEP applies the
four operators P1..P4 once each (y = A_k u_k, y zero-filled inside the
step).  Inputs (u, y, maps: 0.1-1 GB per operator) exceed the 126 MB L2 and
the L2 is additionally flushed between steps, outside the event pairs.

Multi-GPU (torchrun, one process per GPU): every rank owns a 64^3-cube
z-slab of a 64 x 64 x 64N global mesh (weak scaling) and the interface node
planes are summed with the neighbouring ranks over NCCL after every apply
(paper_1903_08243_b200/distributed.py).  Timing: CUDA events per step on
the launching stream, barrier + synchronize around the timed loop, max over
ranks.

value    = sum_k F_k C_k / time, GFLOP/s with the FROZEN per-cell flop counts
           of SURVEY.md Appendix B, over all ranks;
e2e      = the same metric through the public host API (GpuKernelHandle
           with numpy bindings -> fe_wrap_host: pinned host u/y uploaded,
           applied, y downloaded every step);
roofline = the dominant kernel (P4) against the measured FP64 peak.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.094   # measured FP64 DMMA peak on this pool (profiles/r01_fp64_peaks.json)
METRIC = "FP64 GFLOP/s per matrix-free operator action (minimum flop counts of the SURVEY.md App. B menu, round-1 entries included)"
WORKLOADS = {
    "C2": ["C2-P1", "C2-P2", "C2-P3", "C2-P4"],
    "C1": ["C1"],
    "C3": [f"C3-Q{k}" for k in range(1, 7)],
    "C4": [f"C4-quad-Q{k}" for k in range(1, 5)] + [f"C4-hex-Q{k}" for k in range(1, 4)],
    "C5": ["C5"],
    "C6": ["C6"],
}
WORKLOAD_TEXT = {
    "C2": "Helmholtz P1-P4 tetrahedra, 64^3 cubes x 6 tets per GPU, jittered",
    "C1": "mass P2 triangles, 256^2 x 2, jittered (reference's own config)",
    "C3": "scalar Laplacian Q1-Q6 hexahedra 64^3 per GPU, k+1 GL points",
    "C4": "Lame elasticity Q1-Q4 quads 1024^2, Q1-Q3 hexes 64^3 per GPU",
    "C5": "neo-Hookean residual P2 tetrahedra 128^3 x 6 per GPU",
    "C6": "neo-Hookean tangent action (SURVEY 8f.1) P2 tetrahedra 128^3 x 6 per GPU",
}


def ncu_traffic(label):
    """DRAM bytes per launch of a kernel from a committed ncu --set full
    capture (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            entry = json.load(f).get(label)
    except (OSError, ValueError):
        return None
    return None if entry is None else entry["dram_bytes_per_launch"]


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
            d["source"] = "MEASURED_PEAKS.json"
            return d
    except OSError:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """NVML SM clock + throttle reasons sampled during the timed region."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index=0, period=0.002):
        self.samples, self.reasons, self.max_mhz, self.period = [], set(), None, period
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def sample(self):
        """One reading (also called from the timed loop after every step, so
        short timed regions are covered even if the thread is starved)."""
        if not self.nv:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.reasons.update(n for b, n in self.REASONS.items() if r & b)
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self.sample()
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
# problems (per rank)
# ---------------------------------------------------------------------------


def build_problem_for_rank(name, seed, rank, world):
    """3D configs: this rank's z-slab of the weak-scaled global mesh;
    2D configs: the full problem (independent replica per rank)."""
    from paper_1903_08243_b200 import configs as C
    from paper_1903_08243_b200.distributed import build_slab, slab_range
    cfg = C.get_config(name)
    if len(cfg.n) == 3:
        z0, z1, nzg = slab_range(rank, world, cfg.n[2])
        return build_slab(cfg, seed, z0, z1, nzg), True
    return C.build_problem(cfg, seed), False


def build_ops(names, seed, device, rank, world):
    import torch
    import paper_1903_08243_b200 as fe
    from paper_1903_08243_b200.distributed import DistributedOperator
    ops = []
    for name in names:
        prob, slab = build_problem_for_rank(name, seed, rank, world)
        h = fe.compile_and_load(fe.emit_for(prob.spec, fe.Target(), prob.rule))
        m, dm = prob.mesh, prob.dofmap
        h.bind(torch.tensor(np.asarray(m.coords).ravel(), device=device),
               torch.tensor(np.asarray(dm.cell2dof, np.int32).ravel(), device=device),
               torch.tensor(np.asarray(m.cell2vert, np.int32).ravel(), device=device),
               nglobal=dm.ndofs_global)
        u = torch.tensor(prob.u, device=device)
        y = torch.zeros_like(u)
        coef = None
        if prob.coef() is not None:
            coef = tuple(None if c is None else torch.tensor(c, device=device) for c in prob.coef())
        op = dict(name=name, prob=prob, h=h, u=u, y=y, coef=coef, C=m.ncells, ndofs=prob.ndofs,
                  F=fe.flops_per_cell(prob.spec, prob.rule),
                  B=fe.bytes_per_cell(prob.spec, m, dm))
        local = (lambda h, coef: lambda uu, yy: h.apply(uu, yy, coef=coef, overwrite=True))(h, coef)
        rng = (lambda h, coef: lambda uu, yy, a, b, ow: h.apply(uu, yy, a, b, coef=coef,
                                                                 overwrite=ow))(h, coef)
        op["dist"] = (DistributedOperator(prob, local, rank, world, range_apply=rng)
                      if (slab and world > 1) else None)
        op["run"] = op["dist"].apply if op["dist"] else local
        ops.append(op)
    return ops


def oracle_problem(prob):
    from oracle import fe_oracle as fo
    return fo.Problem(prob.spec.form, prob.spec.cell.kind, prob.spec.element.degree,
                      prob.rule.exactness_degree, prob.spec.params)


def parity_sample(ops, ncheck=4096):
    """rel-L2 of the GPU action against the C oracle on the first cells of
    every operator (the full-size oracle is minutes; tests/ cover it)."""
    import torch
    from oracle import fe_oracle as fo
    from oracle import fe_oracle_c as foc
    worst = 0.0
    for op in ops:
        prob = op["prob"]
        end = min(ncheck, op["C"])
        yd = torch.zeros_like(op["u"])
        op["h"].apply(op["u"], yd, 0, end, coef=op["coef"])
        torch.cuda.synchronize()
        ref = _cpu_assemble(prob, end, 8)
        worst = max(worst, fo.rel_l2(yd.cpu().numpy(), ref))
    return worst


def _cpu_assemble(prob, end, threads):
    """C restatement of the reference loop (oracle/fe_oracle.c) over the
    first `end` cells; the numpy restatement for forms the C one lacks
    (neohookean_tangent)."""
    from oracle import fe_oracle as fo
    from oracle import fe_oracle_c as foc
    P = oracle_problem(prob)
    if prob.spec.form in foc.FORMS:
        return foc.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u,
                            prob.mu, prob.lam, 0, end, threads=threads)
    return fo.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u,
                       prob.mu, prob.lam, 0, end, state=getattr(prob, "state", None))


def cpu_measure(ops_or_probs, budget_s=20.0):
    """Reference CPU path on the host cores over a bounded sample of each
    operator: the reference's own generated C (oracle/_ref, vector-ext w8)
    where the reference supports the config, else the C restatement of its
    loop (oracle/fe_oracle.c); all host cores, time in the metric's unit."""
    from oracle import fe_oracle_c as foc
    from oracle import ref_c
    import paper_1903_08243_b200 as fe
    cores = len(os.sched_getaffinity(0))
    per = budget_s / len(ops_or_probs)
    flop = tsum = 0.0
    kinds, desc = set(), []
    for op in ops_or_probs:
        prob = op["prob"]
        F = op["F"]
        sp = prob.spec
        rcell = {"triangle": "tri", "quadrilateral": "quad"}.get(sp.cell.kind)
        use_ref = rcell is not None and ref_c.available(sp.form, rcell, sp.element.degree)
        P = oracle_problem(prob)
        n = 1024
        while True:
            end = min(n, op["C"])
            if use_ref:
                k = ref_c.RefKernel(sp.form, rcell, sp.element.degree)
                b = fe.make_bindings(prob.mesh, prob.dofmap, prob.u, np.zeros(prob.ndofs))
                t0 = time.perf_counter()
                k.run_threads(end, b, cores)
                dt = time.perf_counter() - t0
            else:
                t0 = time.perf_counter()
                _cpu_assemble(prob, end, cores)
                dt = time.perf_counter() - t0
            if dt > per / 3 or end >= op["C"]:
                break
            n *= 2
        flop += F * end
        tsum += dt
        kinds.add("reference" if use_ref else "port")
        desc.append(f"{op['name']}: first {end} cells")
    kind = "reference" if kinds == {"reference"} else "port"
    src = ("reference-generated vector-ext C (oracle/_ref, fevec BENCH_FLAGS)" if kind == "reference"
           else "C restatement of the reference cell loop (oracle/fe_oracle.c, -O3 -ffast-math, "
                "OpenMP over cell chunks); the reference has no code path for this config")
    return {"value": round(flop / tsum / 1e9, 4), "unit": "GFLOP/s", "cores": cores, "kind": kind,
            "sample": f"{src}; " + ", ".join(desc), "seconds": round(tsum, 3)}


def run_e2e(ops, steps):
    """Same metric through the public host API (numpy bindings ->
    GpuKernelHandle.__call__ -> fe_wrap_host): per step and operator, u is
    uploaded from pinned host memory, applied, y is downloaded (y's zero
    chunks are detected on the host and not uploaded)."""
    import torch
    import paper_1903_08243_b200 as fe
    hb = []
    for op in ops:
        prob = op["prob"]
        u = torch.empty(op["ndofs"], dtype=torch.float64, pin_memory=True).numpy()
        u[:] = prob.u
        out = torch.zeros(op["ndofs"], dtype=torch.float64, pin_memory=True).numpy()
        hb.append((op, fe.make_bindings(prob.mesh, prob.dofmap, u, out, prob.mu, prob.lam,
                                        state=getattr(prob, "state", None))))
    for op, b in hb:                 # warm-up: binds the host mesh once
        op["h"](0, op["C"], b)
    t = 0.0
    for _ in range(steps):
        for op, b in hb:
            b["dat0"][:] = 0.0
            t0 = time.perf_counter()
            op["h"](0, op["C"], b)
            t += time.perf_counter() - t0
    for op, _ in hb:                 # restore the device binding
        op["h"].rebind()
    flop = sum(op["F"] * op["C"] for op in ops) * steps
    return {"value": round(flop / t / 1e9, 3), "unit": "GFLOP/s",
            # dat0 is zero every step (y = A u): the host entry detects its
            # all-zero chunks while u uploads and does not upload them
            "h2d_bytes_per_step": sum(8 * op["ndofs"] for op in ops),
            "d2h_bytes_per_step": sum(8 * op["ndofs"] for op in ops), "steps": steps,
            "path": "GpuKernelHandle(start, end, numpy bindings) -> fe_wrap_host, pinned host buffers; "
                    "dat0 zeroed before each call (outside the timer), its zero chunks are scanned "
                    "on the host inside the timer and not uploaded"}


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1903_08243_b200.harness import L2Flusher, gpu_busy_wait

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        dist.barrier()   # collective first: the communicator exists before any P2P batch
    names = WORKLOADS[args.config]
    ops = build_ops(names, args.seed, dev, rank, world)
    parity = parity_sample(ops) if rank == 0 else None
    flush = L2Flusher(local)
    stream = torch.cuda.current_stream()
    # rebuild the device binding after parity_sample's partial apply
    for _ in range(args.warmup):
        flush()
        for op in ops:
            op["run"](op["u"], op["y"])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    per_op = np.zeros(len(ops))
    t_total = 0.0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in ops]
            gpu_busy_wait()              # host submission latency stays outside the events
            for (e0, e1), op in zip(ev, ops):
                e0.record(stream)
                op["run"](op["u"], op["y"])
                e1.record(stream)
            clk.sample()                 # while this step is executing on the GPU
            ev[-1][1].synchronize()
            ts = [e0.elapsed_time(e1) * 1e-3 for e0, e1 in ev]
            per_op += ts
            t_total += sum(ts)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if world > 1:
        t = torch.tensor([t_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_total = float(t.item())
    flop_step = sum(op["F"] * op["C"] for op in ops)
    dofs_step = sum(op["ndofs"] for op in ops)
    value = world * flop_step * args.steps / t_total / 1e9
    if rank == 0:
        peaks = measured_peaks()
        e2e = run_e2e(ops, max(3, min(args.steps, 20)))
        dom = int(np.argmax([op["F"] * op["C"] for op in ops]))
        t_dom = per_op[dom] / args.steps
        achieved = ops[dom]["F"] * ops[dom]["C"] / t_dom / 1e12
        troof = [max(op["F"] * op["C"] / (FP64_PEAK_TFLOPS * 1e12),
                     op["B"] * op["C"] / (peaks["hbm_gbs"] * 1e9)) for op in ops]
        line = {
            "metric": METRIC,
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
            "data": "synthetic: seeded jittered structured mesh, u ~ U[-1,1] (BASELINE names no dataset)",
            "config": {
                "workload": f"{args.config}: {WORKLOAD_TEXT[args.config]}",
                "operators": names,
                "cells_per_gpu": [op["C"] for op in ops],
                "dofs_per_gpu": [op["ndofs"] for op in ops],
                "seed": args.seed,
                "l2": "inputs larger than L2 and L2 flushed (2x L2 write) between steps, outside the events",
                "parallelism": (f"z-slab element partition over {world} GPUs, NCCL halo sums"
                                if world > 1 else "1 GPU"),
            },
            "gdofs_per_s": round(world * dofs_step * args.steps / t_total / 1e9, 3),
            "ms_per_operator": {op["name"]: round(per_op[i] / args.steps * 1e3, 4) for i, op in enumerate(ops)},
            "roofline_frac_per_operator": {op["name"]: round(troof[i] / (per_op[i] / args.steps), 4)
                                           for i, op in enumerate(ops)},
            "kernel_per_operator": {op["name"]: op["h"].info["kernel"] for op in ops},
            "step_roofline_frac": round(sum(troof) / (t_total / args.steps), 4),
            "parity_rel_l2_sample": parity,
            "roofline": {
                "bound": "fp64",
                "kernel": ops[dom]["name"] + ":" + ops[dom]["h"].info["kernel"],
                "achieved": round(achieved, 4),
                "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s",
                "frac": round(achieved / FP64_PEAK_TFLOPS, 4),
                "traffic": ncu_traffic(ops[dom]["name"] + ":" + ops[dom]["h"].info["kernel"]),
                "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum per launch, one "
                                  "ncu --set full capture (profiles/traffic.json)",
                "peak_source": "measured FP64 (DMMA) peak on this pool's B200s, profiles/r01_fp64_peaks.json "
                               "(MEASURED_PEAKS.json has no FP64 entry)",
                "algorithmic_flop_per_launch": ops[dom]["F"] * ops[dom]["C"],
            },
            "e2e": e2e,
            "gpu_launches": len(ops) * args.steps,
            "clocks": clk.summary(),
            "cpu_baseline": cpu_measure(ops) if world == 1 else None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args):
    """--impl reference: the reference's CPU implementation of the path on the
    box's host cores (all of them), on this arm's config/metric/unit; each
    step is a bounded sample of every operator."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import paper_1903_08243_b200 as fe
    names = WORKLOADS[args.config]
    ops = []
    for name in names:
        prob, _ = build_problem_for_rank(name, args.seed, 0, 1)
        ops.append(dict(name=name, prob=prob, C=prob.mesh.ncells, ndofs=prob.ndofs,
                        F=fe.flops_per_cell(prob.spec, prob.rule)))
    # the whole --steps K --warmup W run stays near two minutes of CPU work
    budget = max(0.4, 120.0 / max(1, args.steps + args.warmup))
    vals = []
    for it in range(args.warmup + args.steps):
        r = cpu_measure(ops, budget_s=budget)
        if it >= args.warmup:
            vals.append(r)
    value = float(np.mean([v["value"] for v in vals]))
    secs = float(np.mean([v["seconds"] for v in vals]))
    last = vals[-1]
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded jittered structured mesh, u ~ U[-1,1]",
        "config": {"workload": f"{args.config}: {WORKLOAD_TEXT[args.config]}", "operators": names,
                   "seed": args.seed},
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": last["cores"],
                         "kind": last["kind"], "sample": last["sample"]},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
