#!/usr/bin/env python
"""Benchmark of the matrix-free FE operator action on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config all|C1..C6] [--seed S]

Workload (default ``all``): every BASELINE.json config -- C1 mass P2
triangles 256^2x2, C2 Helmholtz P1..P4 tetrahedra 64^3x6, C3 scalar
Laplacian Q1..Q6 hexahedra 64^3, C4 Lame elasticity Q1..Q4 quadrilaterals
1024^2 and Q1..Q3 hexahedra 64^3, C5 neo-Hookean residual P2 tetrahedra
128^3x6 -- 19 operators on seeded synthetic inputs (BASELINE names no
dataset): interior vertices jittered +-0.1h, u ~ U[-1,1] (C5: 0.01h U[-1,1],
SURVEY A.5), mu/lambda ~ U[0.5,2].  One STEP applies each of the 19
operators once (y = A u, the zero-fill of y inside the timed call).

Multi-GPU (``--gpus N``; re-launches itself under torchrun when WORLD_SIZE
is unset): STRONG scaling -- every config's ONE fixed mesh is cut into N
slabs of nz/N cell layers (3D: z-slabs, 2D: rows of squares; BASELINE C5:
128 cube layers -> 128/N per GPU), each rank applies its slab with the
sm_100a kernels and the interface node planes are summed with the
neighbouring ranks over NCCL, overlapped with the interior cells
(paper_1903_08243_b200/distributed.py).  After timing, the distributed y
is gathered on rank 0 and compared with a single-domain run of the same
mesh (``parity_gathered_rel_l2``).

Timing: per operator, a read-based L2 flush (3x L2, outside the events:
every apply starts with a cold, clean L2), a device-side all-reduce across
ranks (N > 1: the ranks start each operator together), a GPU spin covering
the host's launch latency, then CUDA events on the launching stream around
the apply.  Per (step, operator) the MAX over ranks is taken; ``value`` =
the whole job's flops x K / the sum of those maxima.

value      = sum_k F_k C_k / time in GFLOP/s; F = minimum flops per cell
             over SURVEY.md App. B's menu plus the two exact cheaper
             algorithms of round 1 (modal split for affine P_k tets,
             vertex-gradient P2) -- harness.flops_per_cell;
e2e        = the same metric through the public host API: at N = 1 the
             C-ABI host entry (GpuKernelHandle with numpy bindings ->
             fe_wrap_host: pinned host u uploaded, applied, y downloaded,
             every step); at N > 1 pinned host u -> device, the distributed
             apply, y -> pinned host, max over ranks;
roofline   = the dominant operator's kernel (largest F C: C5) against the
             measured FP64 peak; per-operator fractions for all 19 next to it.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.094   # measured FP64 DMMA peak on this pool (profiles/r01_fp64_peaks.json)
METRIC = ("FP64 GFLOP/s per matrix-free operator action, all BASELINE configs C1-C5 "
          "(minimum flop counts of the SURVEY.md App. B menu, round-1 entries included)")
BASELINE_OPS = (["C1"] + [f"C2-P{k}" for k in range(1, 5)] + [f"C3-Q{k}" for k in range(1, 7)]
                + [f"C4-quad-Q{k}" for k in range(1, 5)] + [f"C4-hex-Q{k}" for k in range(1, 4)]
                + ["C5"])
WORKLOADS = {
    "all": BASELINE_OPS,
    "C1": ["C1"],
    "C2": [f"C2-P{k}" for k in range(1, 5)],
    "C3": [f"C3-Q{k}" for k in range(1, 7)],
    "C4": [f"C4-quad-Q{k}" for k in range(1, 5)] + [f"C4-hex-Q{k}" for k in range(1, 4)],
    "C5": ["C5"],
    "C6": ["C6"],
}
WORKLOAD_TEXT = {
    "all": "every BASELINE config: C1 mass P2 tri 256^2x2; C2 Helmholtz P1-P4 tet 64^3x6; "
           "C3 scalar Laplacian Q1-Q6 hex 64^3 (k+1 GL points); C4 Lame elasticity Q1-Q4 quad "
           "1024^2 and Q1-Q3 hex 64^3; C5 neo-Hookean residual P2 tet 128^3x6",
    "C1": "mass P2 triangles, 256^2 x 2, jittered (reference's own config)",
    "C2": "Helmholtz P1-P4 tetrahedra, 64^3 cubes x 6, jittered",
    "C3": "scalar Laplacian Q1-Q6 hexahedra 64^3, k+1 GL points",
    "C4": "Lame elasticity Q1-Q4 quads 1024^2, Q1-Q3 hexes 64^3",
    "C5": "neo-Hookean residual P2 tetrahedra 128^3 x 6",
    "C6": "neo-Hookean tangent action (SURVEY 8f.1) P2 tetrahedra 128^3 x 6",
}


# ---------------------------------------------------------------------------
# shared: problem sizes and the config dict (identical in both arms)
# ---------------------------------------------------------------------------


def op_meta(name):
    """Global (single-domain) sizes and the flop count of one operator,
    without building its mesh."""
    import paper_1903_08243_b200 as fe
    from paper_1903_08243_b200 import configs as C
    cfg = C.get_config(name)
    spec = fe.operator_spec(cfg.form, cfg.cell, cfg.degree)
    rule = fe.quadrature_rule(cfg.cell, cfg.qdegree)
    k, vs = spec.element.degree, spec.element.value_size
    dofs = vs * int(np.prod([k * n + 1 for n in cfg.n]))
    return dict(name=name, cfg=cfg, cells=cfg.ncells, dofs=dofs,
                F=fe.flops_per_cell(spec, rule))


def config_dict(args, world, names):
    metas = [op_meta(n) for n in names]
    return {
        "workload": f"{args.config}: {WORKLOAD_TEXT[args.config]}",
        "operators": names,
        "cells": [m["cells"] for m in metas],
        "dofs": [m["dofs"] for m in metas],
        "seed": args.seed,
        "l2": "inputs larger than L2 (C1: 8 MB, L2-resident) and a read-based 3x-L2 flush before "
              "every operator apply, outside the events",
        "parallelism": (f"strong scaling: each mesh split into {world} slabs of nz/{world} cell layers, "
                        "NCCL halo sums on the interface planes" if world > 1 else "1 GPU"),
    }


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
            d["source"] = "MEASURED_PEAKS.json"
            return d
    except OSError:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def ncu_traffic(label):
    """DRAM bytes per launch of a kernel from a committed ncu --set full
    capture (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            entry = json.load(f).get(label)
    except (OSError, ValueError):
        return None
    return None if entry is None else entry["dram_bytes_per_launch"]


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
    """This rank's slab of the config's fixed mesh (strong scaling; the
    whole mesh at world = 1), slab-local lattice numbering."""
    from paper_1903_08243_b200 import configs as C
    from paper_1903_08243_b200.distributed import build_slab, global_dof_index, slab_split
    cfg = C.get_config(name)
    return build_slab(cfg, seed, *slab_split(rank, world, cfg.n[-1]), boundary_first=world > 1)


def build_ops(names, seed, device, rank, world):
    import torch
    import paper_1903_08243_b200 as fe
    from paper_1903_08243_b200.distributed import DistributedOperator
    ops = []
    for name in names:
        prob = build_problem_for_rank(name, seed, rank, world)
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
                  F_exec=fe.flops_per_cell(prob.spec, prob.rule, menu="executed"),
                  B=fe.bytes_per_cell(prob.spec, m, dm))
        local = (lambda h, coef: lambda uu, yy: h.apply(uu, yy, coef=coef, overwrite=True))(h, coef)
        rng = (lambda h, coef: lambda uu, yy, a, b, ow: h.apply(uu, yy, a, b, coef=coef,
                                                                 overwrite=ow))(h, coef)
        op["dist"] = DistributedOperator(prob, local, rank, world, range_apply=rng) if world > 1 else None
        op["run"] = op["dist"].apply if op["dist"] else local
        ops.append(op)
    return ops


def oracle_problem(prob):
    from oracle import fe_oracle as fo
    return fo.Problem(prob.spec.form, prob.spec.cell.kind, prob.spec.element.degree,
                      prob.rule.exactness_degree, prob.spec.params)


def _cpu_assemble(prob, start, end, threads, out=None):
    """C restatement of the reference loop (oracle/fe_oracle.c) over cells
    [start, end); the numpy restatement for forms the C one lacks."""
    from oracle import fe_oracle as fo
    from oracle import fe_oracle_c as foc
    P = oracle_problem(prob)
    if prob.spec.form in foc.FORMS:
        return foc.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u,
                            prob.mu, prob.lam, start, end, threads=threads, out=out,
                            state=getattr(prob, "state", None))
    y = fo.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u,
                    prob.mu, prob.lam, start, end, state=getattr(prob, "state", None))
    if out is not None:
        out += y
        return out
    return y


def parity_sample(ops, ncheck=4096):
    """rel-L2 of this rank's GPU action against the C oracle on its first
    cells, every operator (full-size parity: tests/test_gpu_fullsize.py)."""
    import torch
    from oracle import fe_oracle as fo
    worst = 0.0
    for op in ops:
        end = min(ncheck, op["C"])
        yd = torch.zeros_like(op["u"])
        op["h"].apply(op["u"], yd, 0, end, coef=op["coef"])
        torch.cuda.synchronize()
        ref = _cpu_assemble(op["prob"], 0, end, 8)
        worst = max(worst, fo.rel_l2(yd.cpu().numpy(), ref))
    return worst


def gathered_parity(ops, rank, world, dev, seed):
    """N > 1: every rank's y (after the halo sums) against the single-domain
    apply of the same fixed mesh on rank 0 (the global vector restricted to
    the slab -- partition independence, reference test_reference.py:72-89)."""
    import torch
    import torch.distributed as dist
    import paper_1903_08243_b200 as fe
    from oracle import fe_oracle as fo
    from paper_1903_08243_b200.distributed import build_slab, global_dof_index, slab_split
    worst = 0.0
    for op in ops:
        sizes = torch.zeros(world, dtype=torch.int64, device=dev)
        sizes[rank] = op["y"].numel()
        dist.all_reduce(sizes)
        if rank != 0:
            dist.send(op["y"], 0)
            continue
        ys = [op["y"]] + [torch.empty(int(sizes[r]), dtype=torch.float64, device=dev)
                          for r in range(1, world)]
        for r in range(1, world):
            dist.recv(ys[r], r)
        cfg = op["prob"].config
        glob = build_slab(cfg, seed, 0, cfg.n[-1], cfg.n[-1])
        g = fe.compile_and_load(fe.emit_for(glob.spec, fe.Target(), glob.rule))
        m, dm = glob.mesh, glob.dofmap
        g.bind(torch.tensor(np.asarray(m.coords).ravel(), device=dev),
               torch.tensor(np.asarray(dm.cell2dof, np.int32).ravel(), device=dev),
               torch.tensor(np.asarray(m.cell2vert, np.int32).ravel(), device=dev),
               nglobal=dm.ndofs_global)
        coef = None
        if glob.coef() is not None:
            coef = tuple(None if c is None else torch.tensor(c, device=dev) for c in glob.coef())
        yg = torch.zeros(glob.ndofs, dtype=torch.float64, device=dev)
        g.apply(torch.tensor(glob.u, device=dev), yg, coef=coef, overwrite=True)
        for r in range(world):
            sl = build_slab(cfg, seed, *slab_split(r, world, cfg.n[-1]), boundary_first=world > 1)
            ref = yg[torch.as_tensor(global_dof_index(sl), device=dev)]
            worst = max(worst, float(torch.linalg.norm(ys[r] - ref) / torch.linalg.norm(ref)))
        del g, yg
    out = torch.tensor([worst], device=dev)
    dist.broadcast(out, 0)
    return float(out.item())


# ---------------------------------------------------------------------------
# CPU baseline (the oracle port / the reference's own generated C)
# ---------------------------------------------------------------------------


def cpu_run(prob, F, start, end, cores, out=None):
    """One timed CPU pass over cells [start, end) of an operator on `cores`
    threads: the reference's own generated vector-ext C (oracle/_ref) where
    the reference supports the config (C1), else the SIMD-batched port of
    its cell loop (oracle/fe_cpu_port.cpp: per-(form, degree, rule)
    specialised, cross-element vectorised, the paper's technique)."""
    from oracle import fe_cpu_port as fcp
    from oracle import ref_c
    import paper_1903_08243_b200 as fe
    sp = prob.spec
    rcell = {"triangle": "tri", "quadrilateral": "quad"}.get(sp.cell.kind)
    use_ref = rcell is not None and ref_c.available(sp.form, rcell, sp.element.degree)
    if use_ref:
        k = ref_c.RefKernel(sp.form, rcell, sp.element.degree)
        b = fe.make_bindings(prob.mesh, prob.dofmap, prob.u, np.zeros(prob.ndofs))
        t0 = time.perf_counter()
        k.run_threads(end, b, cores, start=start)
        dt = time.perf_counter() - t0
    else:
        P = oracle_problem(prob)
        if out is None:
            out = np.zeros(prob.ndofs)
        t0 = time.perf_counter()
        fcp.assemble(P, prob.mesh.coords, prob.mesh.cell2vert, prob.dofmap.cell2dof, prob.u,
                     prob.mu, prob.lam, start, end, threads=cores, out=out,
                     state=getattr(prob, "state", None))
        dt = time.perf_counter() - t0
    return dt, F * (end - start), "reference" if use_ref else "port"


CPU_PORT_TEXT = ("SIMD-batched port of the reference cell loop (oracle/fe_cpu_port.cpp: the reference's "
                 "quadrature-loop local kernel specialised per (form, degree, rule) with compile-time "
                 "sizes, cross-element vectorised 8 cells per AVX-512 vector as the paper does, OpenMP "
                 "over cell chunks) where the reference has no code path (tets, hexes, mu/lambda, "
                 "neo-Hookean); the reference's own generated vector-ext C (oracle/_ref, its "
                 "BENCH_FLAGS) for C1")


def cpu_measure(ops, fraction=1 / 16):
    """cpu_baseline of our arm: the same CPU path as the reference arm on a
    bounded sample of the SAME workload -- the first ``fraction`` of every
    operator's cells (so the operators weigh in as they do in the full
    step, unlike a per-operator time budget), all host cores."""
    cores = len(os.sched_getaffinity(0))
    flop = tsum = 0.0
    kinds = set()
    for op in ops:
        out = np.zeros(op["ndofs"])
        out.fill(0.0)                        # pages mapped outside the timer
        end = min(op["C"], max(8, -(-int(op["C"] * fraction) // 8) * 8))
        dt, fl, kind = cpu_run(op["prob"], op["F"], 0, end, cores, out)
        flop += fl
        tsum += dt
        kinds.add(kind)
    kind = "reference" if kinds == {"reference"} else "port"
    return {"value": round(flop / tsum / 1e9, 4), "unit": "GFLOP/s", "cores": cores, "kind": kind,
            "sample": CPU_PORT_TEXT + f"; the first 1/{round(1 / fraction)} of every operator's cells "
                      "(the reference arm times the whole meshes)",
            "seconds": round(tsum, 3)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def run_e2e_host_api(ops, steps):
    """N = 1: the metric through the C-ABI host entry (numpy bindings ->
    GpuKernelHandle.__call__ -> fe_wrap_host): per step and operator, u is
    uploaded from pinned host memory, applied, y downloaded (y's zero chunks
    are detected on the host and not uploaded).  Afterwards the plans stay
    bound to the host meshes (device applies would need bind() again)."""
    import torch
    import paper_1903_08243_b200 as fe
    hb = []
    for op in ops:
        prob = op["prob"]
        u = torch.empty(op["ndofs"], dtype=torch.float64, pin_memory=True).numpy()
        u[:] = prob.u
        out = torch.zeros(op["ndofs"], dtype=torch.float64, pin_memory=True).numpy()
        def pinned(a):              # every host input of the call in pinned memory
            if a is None:
                return None
            t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
            t[...] = a
            return t
        hb.append((op, fe.make_bindings(prob.mesh, prob.dofmap, u, out, pinned(prob.mu), pinned(prob.lam),
                                        state=pinned(getattr(prob, "state", None)))))
    for op, b in hb:                 # warm-up: binds the host mesh once
        op["h"](0, op["C"], b)
    # the operators of a step are independent calls: E2E_THREADS host threads
    # issue them concurrently (ctypes releases the GIL; each plan has its own
    # streams), so one call's upload overlaps another's download on the
    # full-duplex PCIe link -- the reference's "concurrent calls on disjoint
    # dat0"
    from concurrent.futures import ThreadPoolExecutor
    nthr = int(os.environ.get("FE_E2E_THREADS", "4"))
    # largest transfers first (LPT): the tail of the step is then made of
    # short calls, so uploads and downloads of different calls keep both
    # directions of the link busy until the end (FE_E2E_ORDER=config keeps
    # the config order: measured 3.5-3.7 vs 4.0+ TFLOP/s)
    if os.environ.get("FE_E2E_ORDER", "size") == "size":
        hb.sort(key=lambda ob: -ob[0]["ndofs"])
    pool = ThreadPoolExecutor(nthr) if nthr > 1 else None

    def call(ob):
        op, b = ob
        op["h"](0, op["C"], b)

    t = 0.0
    for _ in range(steps):
        for op, b in hb:
            b["dat0"][:] = 0.0
        t0 = time.perf_counter()
        if pool:
            list(pool.map(call, hb))
        else:
            for ob in hb:
                call(ob)
        t += time.perf_counter() - t0
    if pool:
        pool.shutdown()
    return t, {"h2d_bytes_per_step": sum(8 * op["ndofs"] for op in ops),
               "d2h_bytes_per_step": sum(8 * op["ndofs"] for op in ops),
               "threads": nthr,
               "path": "GpuKernelHandle(start, end, numpy bindings) -> fe_wrap_host, pinned host "
                       "buffers, the step's operator calls issued largest-first from FE_E2E_THREADS host threads; "
                       "dat0 zeroed before each step (outside the timer), its zero chunks are "
                       "scanned on the host inside the timer and not uploaded"}


def run_e2e_distributed(ops, steps, dev):
    """N > 1: pinned host u -> device, the distributed apply (NCCL halo
    sums), y -> pinned host, synchronised, per operator; wall clock per rank
    (the max over ranks is taken by the caller)."""
    import torch
    hb = []
    for op in ops:
        hu = torch.empty(op["ndofs"], dtype=torch.float64, pin_memory=True)
        hu.copy_(torch.from_numpy(op["prob"].u))
        hy = torch.empty(op["ndofs"], dtype=torch.float64, pin_memory=True)
        du, dy = torch.empty_like(op["u"]), torch.empty_like(op["y"])
        hb.append((op, hu, hy, du, dy))
    torch.cuda.synchronize()
    t = 0.0
    for it in range(steps + 1):
        for op, hu, hy, du, dy in hb:
            t0 = time.perf_counter()
            du.copy_(hu, non_blocking=True)
            op["run"](du, dy)
            hy.copy_(dy, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            if it > 0:
                t += time.perf_counter() - t0
    return t, {"h2d_bytes_per_step": sum(8 * op["ndofs"] for op in ops),
               "d2h_bytes_per_step": sum(8 * op["ndofs"] for op in ops),
               "path": "per rank: pinned host u -> device copy, DistributedOperator.apply "
                       "(fe_apply on the slab + NCCL halo sums), device -> pinned host y, "
                       "synchronised; bytes summed over ranks; max over ranks"}


def graph_throughput(ops, names=("C1", "C2-P1", "C3-Q1"), reps=50):
    """The launch-latency-bound operators (10-25 us per apply: VERDICT item 10)
    as they run inside a captured solver iteration: ``reps`` overwrite applies
    in one CUDA graph, microseconds per apply (launch overhead amortised,
    inputs L2-resident).  Labelled separately: NOT the protocol of ``value``
    (single cold-L2 applies), which stays the reported number."""
    import torch
    out = {"protocol": f"{reps} overwrite applies captured in one CUDA graph, best of 10 replays, warm L2"}
    for op in ops:
        if op["name"] not in names:
            continue
        try:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                op["run"](op["u"], op["y"])              # warm-up on the capture stream
                with torch.cuda.graph(g, stream=side):
                    for _ in range(reps):
                        op["run"](op["u"], op["y"])
            torch.cuda.current_stream().wait_stream(side)
            best = 1e9
            for _ in range(10):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1))
            out[op["name"]] = round(best * 1e3 / reps, 2)
        except Exception as e:  # noqa: BLE001 -- capture unsupported: say why
            out[op["name"]] = "capture failed: " + str(e)[:80]
    return out if len(out) > 1 else None


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1903_08243_b200 import _lib
    from paper_1903_08243_b200.harness import L2Flusher, gpu_busy_wait

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")            # communicator init in the log
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
        dist.barrier()   # collective first: the communicator exists before any P2P batch
    names = WORKLOADS[args.config]
    t_build = time.perf_counter()
    ops = build_ops(names, args.seed, dev, rank, world)
    t_build = time.perf_counter() - t_build
    parity = parity_sample(ops)
    if world > 1:
        t = torch.tensor([parity], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        parity = float(t.item())
    flush = L2Flusher(local)
    stream = torch.cuda.current_stream()
    token = torch.zeros(1, device=dev)

    def step_ops(events=None):
        for i, op in enumerate(ops):
            flush()
            if world > 1:
                dist.all_reduce(token)           # device-side: ranks start each operator together
            gpu_busy_wait()                      # host submission latency stays outside the events
            if events is not None:
                events[i][0].record(stream)
            op["run"](op["u"], op["y"])
            if events is not None:
                events[i][1].record(stream)

    for _ in range(args.warmup):
        step_ops()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    lib = _lib.load()
    times = np.zeros((args.steps, len(ops)))
    launches0 = lib.fe_launch_count()
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in ops]
            step_ops(ev)
            clk.sample()                 # while this step is executing on the GPU
            ev[-1][1].synchronize()
            times[s] = [e0.elapsed_time(e1) * 1e-3 for e0, e1 in ev]
    launches = lib.fe_launch_count() - launches0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if world > 1:
        t = torch.tensor(times, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        times = t.cpu().numpy()
        lt = torch.tensor([launches], dtype=torch.int64, device=dev)
        dist.all_reduce(lt)
        launches = int(lt.item())
    t_total = float(times.sum())
    metas = [op_meta(n) for n in names]
    flop_step = sum(m["F"] * m["cells"] for m in metas)
    dofs_step = sum(m["dofs"] for m in metas)
    value = flop_step * args.steps / t_total / 1e9
    gathered = gathered_parity(ops, rank, world, dev, args.seed) if world > 1 else None
    # e2e (max over ranks)
    e2e_steps = max(3, min(args.steps, 10))
    if world == 1:
        t_e2e, e2e_info = run_e2e_host_api(ops, e2e_steps)
    else:
        t_e2e, e2e_info = run_e2e_distributed(ops, e2e_steps, dev)
        t = torch.tensor([t_e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_e2e = float(t.item())
        nb = torch.tensor([e2e_info["h2d_bytes_per_step"]], dtype=torch.int64, device=dev)
        dist.all_reduce(nb)
        e2e_info["h2d_bytes_per_step"] = e2e_info["d2h_bytes_per_step"] = int(nb.item())
    if rank == 0:
        peaks = measured_peaks()
        med = np.median(times, axis=0)
        dom = int(np.argmax([op["F"] * op["C"] for op in ops]))
        achieved = ops[dom]["F"] * ops[dom]["C"] / med[dom] / 1e12
        # per-operator roofline on this rank's slab (the slowest rank's time)
        troof = [max(op["F"] * op["C"] / (FP64_PEAK_TFLOPS * 1e12),
                     op["B"] * op["C"] / (peaks["hbm_gbs"] * 1e9)) for op in ops]
        kern = {op["name"]: op["h"].info["kernel"] for op in ops}
        line = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "GFLOP/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(t_total / args.steps * 1e3, 4),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic: seeded jittered structured meshes, u ~ U[-1,1] (BASELINE names no dataset)",
            "config": config_dict(args, world, names),
            "gdofs_per_s": round(dofs_step * args.steps / t_total / 1e9, 3),
            "ms_per_operator_median": {op["name"]: round(med[i] * 1e3, 4) for i, op in enumerate(ops)},
            "ms_per_operator_mean": {op["name"]: round(times[:, i].mean() * 1e3, 4)
                                     for i, op in enumerate(ops)},
            "gflops_per_operator": {op["name"]: round(op["F"] * op["C"] / med[i] / 1e9, 1)
                                    for i, op in enumerate(ops)},
            "roofline_frac_per_operator": {op["name"]: round(troof[i] / med[i], 4)
                                           for i, op in enumerate(ops)},
            "kernel_per_operator": kern,
            # kernels that execute fewer flops than the (frozen) menu F: their
            # fraction against the count they actually execute
            "roofline_frac_vs_executed_flops": {
                op["name"]: round(max(op["F_exec"] * op["C"] / (FP64_PEAK_TFLOPS * 1e12),
                                      op["B"] * op["C"] / (peaks["hbm_gbs"] * 1e9)) / med[i], 4)
                for i, op in enumerate(ops) if op["F_exec"] < op["F"]},
            "step_roofline_frac": round(sum(troof) / (t_total / args.steps), 4),
            "parity_rel_l2_sample": parity,
            "parity_gathered_rel_l2": gathered,
            "roofline": {
                "bound": "fp64",
                "kernel": ops[dom]["name"] + ":" + kern[ops[dom]["name"]],
                "achieved": round(achieved, 4),
                "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s",
                "frac": round(achieved / FP64_PEAK_TFLOPS, 4),
                "traffic": ncu_traffic(ops[dom]["name"] + ":" + kern[ops[dom]["name"]]),
                "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum per launch, one "
                                  "ncu --set full capture (profiles/traffic.json)",
                "peak_source": "measured FP64 (DMMA) peak on this pool's B200s, profiles/r01_fp64_peaks.json "
                               "(MEASURED_PEAKS.json has no FP64 entry)",
                "algorithmic_flop_per_launch": ops[dom]["F"] * ops[dom]["C"],
                "time_basis": "median over steps of the max over ranks",
            },
            "e2e": {"value": round(flop_step * e2e_steps / t_e2e / 1e9, 3), "unit": "GFLOP/s",
                    "steps": e2e_steps, **e2e_info},
            "graph_us_per_apply": graph_throughput(ops) if world == 1 else None,
            "gpu_launches": launches,
            "gpu_launches_source": "fe_launch_count() difference around the timed region, summed over ranks",
            "clocks": clk.summary(),
            "build_s": round(t_build, 1),
            "cpu_baseline": cpu_measure(ops) if world == 1 else None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------


def run_reference(args):
    """--impl reference: the reference's CPU implementation of the path on the
    box's host cores (all of them), on this arm's config/metric/unit.  Step
    s applies every operator over cell window s of its mesh (window =
    ceil(C / K)), so the K timed steps together apply every operator to its
    WHOLE BASELINE mesh exactly once; warm-up steps apply window 0."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    names = WORKLOADS[args.config]
    probs = [(build_problem_for_rank(n, args.seed, 0, 1), op_meta(n)["F"]) for n in names]
    outs = [np.zeros(p.ndofs) for p, _ in probs]
    for o in outs:
        o.fill(0.0)                          # pages mapped outside the timer
    cores = len(os.sched_getaffinity(0))
    K = args.steps
    flop = secs = 0.0
    kinds = set()
    for it in range(args.warmup + K):
        s = 0 if it < args.warmup else it - args.warmup
        sf = st = 0.0
        for (prob, F), out in zip(probs, outs):
            C = prob.mesh.ncells
            w = -(-(-(-C // K)) // 8) * 8          # ceil(C/K), a multiple of the SIMD width
            a, b = min(C, s * w), min(C, (s + 1) * w)
            if a >= b:
                continue
            dt, fl, kind = cpu_run(prob, F, a, b, cores, out)
            sf += fl
            st += dt
            kinds.add(kind)
        if it >= args.warmup:
            flop += sf
            secs += st
    value = flop / secs / 1e9
    kind = "reference" if kinds == {"reference"} else "port"
    sample = (CPU_PORT_TEXT + f"; step s applies cells [s*w, (s+1)*w), w = ceil(C/{K}) rounded up to 8, of "
              f"every operator, so the {K} timed steps cover every full BASELINE mesh once")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GFLOP/s",
        "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": round(secs / K * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded jittered structured meshes, u ~ U[-1,1] (BASELINE names no dataset)",
        "config": config_dict(args, world, names),
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def relaunch_under_torchrun(args):
    """--gpus N > 1 without torchrun: re-run this script as N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="all", choices=sorted(WORKLOADS))
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
