"""Verification and measurement harness (mirror of the reference
``fevec.bench``, ``/root/reference/pkg/src/fevec/bench.py``).

Same names and meaning where the reference has them: ``make_bindings``
(``bench.py:94-101``), ``random_coefficients`` (``:104-107``),
``flops_per_cell``, ``bytes_per_cell``, ``arithmetic_intensity``,
``verify_target`` (``:152-164``, raises ``VerificationError``),
``run_configuration`` (``:167-224``), ``BenchmarkRecord``/``CSV_COLUMNS``/
``write_csv`` (``:38-42,227-231``) and ``roofline_rows`` (``:234-259``).

Differences, all deliberate:

* ``flops_per_cell`` is the algorithmic count of SURVEY.md Appendix B -- the
  minimum over its documented algorithm menu plus the two cheaper exact
  algorithms round 1 added (modal split for affine simplices, vertex-
  gradient P2; App. B allows lowering F, never raising it), FMA = 2 flops --
  not an interpreter tally of one implementation; ``menu="survey"`` gives
  SURVEY's frozen figures;
* ``bytes_per_cell`` is the compulsory-traffic model of SURVEY.md 8(d)
  (u read once, y written once, coordinates, one int32 node map whose vertex
  columns double as the vertex map, mu/lambda fields);
* ``verify_target`` takes the oracle as a callable (the product package
  never imports the oracle; tests and bench.py inject it);
* timing uses CUDA events on the launching stream with an L2 flush between
  applies; the default roofline peaks are the B200 figures measured on this
  pool (FP64 DMMA 37.09 TFLOP/s: profiles/r01_fp64_peaks.json; HBM
  6547.8 GB/s: MEASURED_PEAKS.json).
"""

from __future__ import annotations

import csv
import math
from dataclasses import dataclass

import numpy as np

from .elements import OperatorSpec, integrand_degree, quadrature_rule
from .mesh import DofMap, Mesh

__all__ = [
    "BenchmarkRecord", "CSV_COLUMNS", "VerificationError", "DEFAULT_PEAK_GFLOPS",
    "DEFAULT_BANDWIDTH_GBS", "make_bindings", "random_coefficients", "flops_per_cell",
    "bytes_per_cell", "arithmetic_intensity", "verify_target", "run_configuration",
    "write_csv", "roofline_rows", "rel_err", "rel_l2",
]

CSV_COLUMNS = (
    "operator", "cell", "degree", "target", "width", "ncells", "trials",
    "time_best_s", "time_mean_s", "flops_per_cell", "gflops", "ai",
    "speedup", "flags", "seed",
    # B200 extensions
    "gpus", "gdofs_per_s", "roofline_fraction", "parity_rel_l2", "cpu_cores", "cpu_time_s",
)

DEFAULT_PEAK_GFLOPS = 37094.0      # FP64 (DMMA) measured on this pool's B200s
DEFAULT_DFMA_GFLOPS = 34162.0      # FP64 DFMA measured
DEFAULT_BANDWIDTH_GBS = 6547.8     # MEASURED_PEAKS.json hbm_gbs


class VerificationError(Exception):
    pass


@dataclass(frozen=True)
class BenchmarkRecord:
    operator: str
    cell: str
    degree: int
    target: str
    width: int
    ncells: int
    trials: int
    time_best_s: float
    time_mean_s: float
    flops_per_cell: int
    gflops: float
    ai: float
    speedup: float
    flags: str
    seed: int
    gpus: int = 1
    gdofs_per_s: float = 0.0
    roofline_fraction: float = 0.0
    parity_rel_l2: float = float("nan")
    cpu_cores: int = 0
    cpu_time_s: float = float("nan")

    def row(self) -> list:
        return [getattr(self, c) for c in CSV_COLUMNS]


def make_bindings(mesh: Mesh, dofmap: DofMap, u, out, mu=None, lam=None, state=None) -> dict:
    """Binding names -> buffers (reference bench.py:94-101); dat3/dat4 carry
    the mu/lambda vertex fields of elasticity_lame, dat3 the state u0 of a
    linearised form (neohookean_tangent)."""
    b = {
        "dat0": out,
        "dat1": np.ascontiguousarray(mesh.coords, dtype=np.float64).ravel(),
        "dat2": np.ascontiguousarray(u, dtype=np.float64),
        "map0": np.ascontiguousarray(dofmap.cell2dof, dtype=np.int32).ravel(),
        "map1": np.ascontiguousarray(mesh.cell2vert, dtype=np.int32).ravel(),
    }
    if mu is not None:
        b["dat3"] = np.ascontiguousarray(mu, dtype=np.float64)
        b["dat4"] = np.ascontiguousarray(lam, dtype=np.float64)
    if state is not None:
        b["dat3"] = np.ascontiguousarray(state, dtype=np.float64)
    return b


def random_coefficients(spec: OperatorSpec, dofmap: DofMap, seed: int) -> np.ndarray:
    """u ~ U(-1, 1) (reference bench.py:104-107)."""
    rng = np.random.default_rng(seed)
    n = spec.element.value_size * dofmap.ndofs_global
    return rng.uniform(-1.0, 1.0, n)


# ---------------------------------------------------------------------------
# frozen flop model and compulsory bytes (8d)
# ---------------------------------------------------------------------------


def _interp_sumfact(d: int, p: int, q: int) -> int:
    colloc = sum(2 * q ** s * p ** (d - s + 1) for s in range(1, d + 1)) + 2 * d * q ** (d + 1)
    if d == 2:
        direct = 4 * q * p * p + 4 * q * q * p
    else:
        direct = 4 * q * p ** 3 + 6 * q * q * p * p + 6 * q ** 3 * p
    return min(colloc, direct)


def flops_per_cell(spec: OperatorSpec, rule=None, menu: str = "min") -> int:
    """Minimum flop count per cell over the algorithm menu of SURVEY.md
    Appendix B.  ``menu="min"`` (default) includes the cheaper exact
    algorithms added in round 1 (modal split for affine P_k tets,
    vertex-gradient P2 for the hyperelastic forms) -- SURVEY App. B allows
    lowering F that way, and it keeps every fraction <= 1;
    ``menu="survey"`` returns SURVEY's frozen values (reported next to it);
    ``menu="executed"`` the count of the algorithm the selected kernel runs
    where that is lower still (round 2: the physical-gradient C5/C6 kernel,
    the even-odd team kernel of C3-Q5/Q6)
    -- the headline keeps ``"min"`` frozen at its round-1 values, so a
    cheaper kernel shows as less time, and DESIGN.md reports both.
    For (form, cell) pairs outside the BASELINE configs it is the quadrature
    algorithm's count, noted as such in DESIGN.md."""
    best = menu != "survey"
    if rule is None:
        rule = quadrature_rule(spec.cell, integrand_degree(spec))
    form, cell = spec.form, spec.cell
    k = spec.element.degree
    nd = spec.element.ndof_scalar
    nq = rule.npoints
    d = cell.dim
    vs = spec.element.value_size
    if cell.simplex and form == "mass":
        return min(2 * nd * nd + nd + 8, 4 * nd * nq + 2 * nq + 8)
    if cell.kind == "tetrahedron" and form == "helmholtz":
        et = 14 * nd * nd + 13 * nd + 80
        quad = 16 * nd * nq + 20 * nq + 80
        split = 12 * nd * k ** 3 + 15 * k ** 3 + 2 * nd * nd + 2 * nd + 80
        # "modal split" (added to the menu in round 1, lowering F as SURVEY
        # App. B allows): the split algorithm on the m = dim P_{k-1} =
        # k(k+1)(k+2)/6 stiffness modes of elements.stiffness_modes instead
        # of the k^3 points -- 183 / 840 / 3,470 / 11,300 for k = 1..4
        # (the frozen SURVEY values were 183 / 1,380 / 5,940 / 17,685)
        m = k * (k + 1) * (k + 2) // 6
        modal = 12 * nd * m + 15 * m + 2 * nd * nd + 2 * nd + 80
        return min(et, quad, split, modal) if best else min(et, quad, split)
    if cell.kind == "hexahedron" and form == "laplacian_scalar":
        p, q = k + 1, rule.npoints_1d
        F = 2 * _interp_sumfact(3, p, q) + 148 * q ** 3 + 36
        if menu == "executed" and p == q and q >= 6:
            # round 2 team kernel at Q5/Q6 (kern_tensor.cuh, FE_TK_EO): the direct
            # algorithm with every 1D contraction in even-odd form -- per pencil a
            # split (2 floor(P/2) adds) shared by the B and D applications, per
            # application floor(Q/2) row pairs of (ceil(P/2) + floor(P/2)) FMAs + 2
            # adds and the middle row of an odd Q; the adjoint mirrors it
            hp, ne, hq, mq = p // 2, (p + 1) // 2, q // 2, q % 2
            appB = hq * ((ne + hp) * 2 + 2) + mq * ne * 2
            appD = hq * ((ne + hp) * 2 + 2) + mq * hp * 2
            sm = 2 * hp
            fwd = p * p * (sm + appB + appD) + q * p * (2 * sm + 2 * appB + appD) + q * q * (3 * sm + 2 * appB + appD)
            bwd = q * q * (2 * appB + appD + 3 * sm) + q * p * (2 * appB + appD + 2 * sm) + p * p * (appB + appD + sm)
            return min(F, fwd + bwd + 148 * q ** 3 + 36)
        return F
    if not cell.simplex and form == "elasticity_lame":
        p, q = k + 1, rule.npoints_1d
        P, g = (76, 8) if d == 2 else (254, 36)
        sf = 2 * d * _interp_sumfact(d, p, q) + P * q ** d + g
        dense = 4 * d * d * p ** d * q ** d + P * q ** d + g
        if menu == "executed" and d == 2 and k in (3, 4) and q == p + 1:
            # round 2 even-odd pair kernel (kern_pair.cuh pair_eo_kernel): counted
            # from its SASS (profiles/r02/sass_hist.txt), 2 DFMA + DMUL + DADD per
            # lane, two lanes per cell
            return min(sf, dense, {3: 2 * (2 * 726 + 271 + 339), 4: 2 * (2 * 1152 + 378 + 500)}[k])
        return min(sf, dense)
    # vertex-gradient P2 (round 1): grad_ref u is P1, so it is interpolated
    # from its 4 vertex values (9 x 4 FMA = 72 flops per point instead of 180)
    # after a 720-flop projection per field, and integrated through the 4
    # vertex moments (72 per point + 720 per cell)
    if cell.kind == "tetrahedron" and form == "neohookean" and k == 2:
        quad = nq * 543 + 52
        vtx = nq * (543 - 360 + 144) + 52 + 2 * 720
        if menu == "executed":
            # round 2 kernel (kern_quad.cuh, FE_VTX_PHYS): physical vertex
            # gradients H_v = G_v J^-1 (216) once per cell, per point
            # grad u = sum_v lambda_v H_v (72), F 3, cofactor + det 32, ln 1,
            # 1/J 1, P 37, weight 10, moments sum_v lambda_v P (72); per cell
            # geometry 52, G_v 720, S_v J^-T 216, projection 720
            return nq * (72 + 3 + 32 + 1 + 1 + 37 + 10 + 72) + 52 + 720 + 216 + 216 + 720
        return min(quad, vtx) if best else quad
    if cell.kind == "tetrahedron" and form == "neohookean_tangent" and k == 2:
        # per point: interpolate grad u0 and grad du (2 x 180), both to
        # physical (2 x 45), F 3, cofactor + det 32, 1/J 1, F^-1 9, ln J 1,
        # M = F^-1 dF 45, tr 2, M F^-1 45, dP 54, w|det| 10, dP J^-T 45,
        # integrate 180; per cell geometry 52
        quad = nq * 832 + 52
        vtx = nq * (832 - 540 + 216) + 52 + 3 * 720
        if menu == "executed":
            # round 2 kernel: per point the two physical gradients (2 x 72),
            # F 3, cofactor + det 32, 1/J 1, ln J 1, M = A dF 45, tr 2, M A 45,
            # dP 54, weight 10, moments 72; per cell geometry 52, 2 x (G_v 720
            # + H_v 216), S_v J^-T 216, projection 720
            return nq * (144 + 3 + 32 + 1 + 1 + 45 + 2 + 45 + 54 + 10 + 72) + 52 + 2 * 936 + 216 + 720
        return min(quad, vtx) if best else quad
    # generic quadrature algorithm: interpolation and integration of values
    # (2 nd per component) and reference gradients (2 nd d per component)
    per_q = 0
    if form in ("mass", "helmholtz"):
        per_q += 4 * nd * vs
    if form != "mass":
        per_q += 4 * nd * d * vs + 4 * d * d * vs + 20
    geo = 9 * d * d if not cell.simplex else 0
    return nq * (per_q + geo) + 8 * d * d


def bytes_per_cell(spec: OperatorSpec, mesh: Mesh, dofmap: DofMap) -> float:
    """Compulsory bytes per cell."""
    vs = spec.element.value_size
    n = dofmap.ndofs_global
    total = 8.0 * vs * n * 2 + 8.0 * mesh.dim * mesh.nvertices
    total += 4.0 * dofmap.cell2dof.size
    if spec.coefficient_fields:
        total += 8.0 * 2 * mesh.nvertices
    return total / mesh.ncells


def arithmetic_intensity(spec, mesh, dofmap, rule=None) -> float:
    return flops_per_cell(spec, rule) / bytes_per_cell(spec, mesh, dofmap)


def roofline_time(spec, mesh, dofmap, rule=None, peak_gflops=DEFAULT_PEAK_GFLOPS,
                  bandwidth_gbs=DEFAULT_BANDWIDTH_GBS, menu="min") -> float:
    """T_roof = max(F C / P_fp64, B / BW) in seconds."""
    F = flops_per_cell(spec, rule, menu) * mesh.ncells
    B = bytes_per_cell(spec, mesh, dofmap) * mesh.ncells
    return max(F / (peak_gflops * 1e9), B / (bandwidth_gbs * 1e9))


# ---------------------------------------------------------------------------
# verification
# ---------------------------------------------------------------------------


def rel_err(out, ref) -> float:
    """Reference metric (bench.py:147-149)."""
    out = np.asarray(out)
    return float(np.abs(out - ref).max()) / max(float(np.abs(ref).max()), 1.0)


def rel_l2(out, ref) -> float:
    """North-star metric: ||out - ref||_2 / ||ref||_2."""
    out = np.asarray(out)
    den = float(np.linalg.norm(ref))
    return float(np.linalg.norm(out - ref)) / (den if den > 0 else 1.0)


def verify_target(spec, target, mesh, dofmap, rule, handle, u, rtol, oracle,
                  mu=None, lam=None) -> float:
    """Run the kernel once (host path) against ``oracle(...)`` -> reference
    vector; raises VerificationError when rel-L2 exceeds rtol."""
    ref = oracle(spec, mesh, dofmap, rule, u, mu, lam)
    out = np.zeros_like(ref)
    handle(0, mesh.ncells, make_bindings(mesh, dofmap, u, out, mu, lam))
    err = rel_l2(out, ref)
    if not err <= rtol:
        raise VerificationError(
            f"{spec.form} {spec.cell.kind} p{spec.element.degree} {target.kind}: "
            f"relative L2 error {err:.3e} exceeds {rtol:.1e}")
    return err


# ---------------------------------------------------------------------------
# GPU timing
# ---------------------------------------------------------------------------


class L2Flusher:
    """Cold, clean L2 before a timed apply: READS a buffer of 3x the L2 size.
    Every line of the previous apply is evicted -- its dirty lines (y) are
    written back here, outside the timed region -- and what is left in the
    L2 is clean.  (A write-based flush leaves the L2 full of dirty lines whose
    write-back then lands inside the next timed apply: up to 126 MB of
    DRAM writes, ~20 us, charged to the operator.)"""

    def __init__(self, device=0):
        import torch
        l2 = torch.cuda.get_device_properties(device).L2_cache_size
        self.buf = torch.ones(max(3 * l2, 1 << 20) // 4, dtype=torch.int32, device=device)
        self.out = None

    def __call__(self):
        self.out = self.buf.sum()


def gpu_busy_wait(seconds=50e-6):
    """Queue a short spin kernel so the GPU is still busy while the host
    enqueues the next event pair and launches: the events then bracket GPU
    execution only, not host submission latency (~tens of us of Python and
    driver time, which would otherwise dominate small configs such as C1)."""
    import torch
    torch.cuda._sleep(int(seconds * 2.0e9))


def time_device(fn, trials=20, warmup=3, flush=True, stream=None, setup=None):
    """CUDA-event timing of ``fn()`` on ``stream`` with an optional L2 flush
    outside each event pair; ``setup()`` (e.g. zeroing the output, as the
    reference's bench.py:197-198 does outside its timer) runs before the
    flush, untimed.  Returns a list of seconds."""
    import torch
    stream = stream or torch.cuda.current_stream()
    fl = L2Flusher() if flush else None
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(trials):
        if setup:
            setup()
        if fl:
            fl()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        gpu_busy_wait()
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1) * 1e-3)
    return times


def run_configuration(spec, target, mesh, dofmap, trials=20, seed=0, rule=None, handle=None,
                      oracle=None, verify_rtol=1e-12, u=None, mu=None, lam=None,
                      skip_verify=False) -> BenchmarkRecord:
    """Create the plan, verify against the oracle (when given), then time
    ``trials`` applies over the whole mesh with CUDA events (reference
    bench.py:167-224: verification-gated best/mean timing)."""
    import torch
    from .jit import compile_and_load, emit_for
    if rule is None:
        rule = quadrature_rule(spec.cell, integrand_degree(spec))
    if handle is None:
        handle = compile_and_load(emit_for(spec, target, rule))
    if u is None:
        u = random_coefficients(spec, dofmap, seed)
    err = float("nan")
    if oracle is not None and not skip_verify:
        err = verify_target(spec, target, mesh, dofmap, rule, handle, u, verify_rtol, oracle, mu, lam)
    dev = torch.device("cuda")
    handle.bind(torch.as_tensor(np.ascontiguousarray(mesh.coords).ravel(), device=dev),
                torch.as_tensor(np.ascontiguousarray(dofmap.cell2dof, np.int32).ravel(), device=dev),
                torch.as_tensor(np.ascontiguousarray(mesh.cell2vert, np.int32).ravel(), device=dev),
                nglobal=dofmap.ndofs_global)
    ud = torch.as_tensor(u, device=dev)
    yd = torch.zeros_like(ud)
    coef = None
    if mu is not None:   # (mu, lambda) vertex fields, or (state u0, None) of a linearised form
        coef = tuple(None if c is None else torch.as_tensor(c, device=dev) for c in (mu, lam))
    times = time_device(lambda: handle.apply(ud, yd, coef=coef, overwrite=True), trials=trials)
    best, mean = min(times), sum(times) / len(times)
    fpc = flops_per_cell(spec, rule)
    bpc = bytes_per_cell(spec, mesh, dofmap)
    troof = roofline_time(spec, mesh, dofmap, rule)
    return BenchmarkRecord(
        operator=spec.form, cell=spec.cell.kind, degree=spec.element.degree,
        target=handle.info["kernel"], width=handle.info["block"], ncells=mesh.ncells,
        trials=trials, time_best_s=best, time_mean_s=mean, flops_per_cell=fpc,
        gflops=fpc * mesh.ncells / best / 1e9, ai=fpc / bpc, speedup=1.0, flags="sm_100a",
        seed=seed, gdofs_per_s=spec.element.value_size * dofmap.ndofs_global / best / 1e9,
        roofline_fraction=troof / best, parity_rel_l2=err)


def write_csv(records, fileobj) -> None:
    w = csv.writer(fileobj)
    w.writerow(CSV_COLUMNS)
    for r in records:
        w.writerow(r.row())


def roofline_rows(records, peak_gflops=DEFAULT_PEAK_GFLOPS, bandwidth_gbs=DEFAULT_BANDWIDTH_GBS):
    """Attainable performance per record and the ridge point (bench.py:234-259)."""
    ridge = peak_gflops / bandwidth_gbs
    rows = []
    for r in records:
        attainable = min(peak_gflops, r.ai * bandwidth_gbs)
        rows.append({
            "operator": r.operator, "cell": r.cell, "degree": r.degree, "target": r.target,
            "width": r.width, "ai": r.ai, "gflops": r.gflops,
            "attainable_gflops": attainable, "fraction_of_attainable": r.gflops / attainable,
            "memory_bound": r.ai < ridge,
        })
    return ridge, rows
