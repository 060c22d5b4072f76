"""Command line for the B200 path, mirroring the
reference's ``fevec`` CLI (``cli.py:60-130``, subcommands at ``:286-387``):

    python -m paper_1903_08243_b200 verify [--config C2-P3,...]   # specialised vs generic kernel
    python -m paper_1903_08243_b200 bench  [--config ...] [--trials 20] [--output bench.csv]
    python -m paper_1903_08243_b200 report bench.csv [--peak GFLOPS] [--bandwidth GBS]
    python -m paper_1903_08243_b200 info   [--config ...]

``verify`` is the reference's "every target equals the scalar target" check
(``cli.py:250-283``) on the GPU: the specialised sm_100a kernel of each
config against the generic reference-structured quadrature kernel
(``Target(generic=True)``) on the same seeded inputs -- the CPU oracle is
test infrastructure and is not imported here.  ``bench`` writes the
reference's CSV schema (``bench.py:38-42``) extended with gpus,
gdofs_per_s, roofline_fraction, parity_rel_l2, cpu_cores, cpu_time_s;
``report`` prints the roofline table (``cli.py:350-387``).  Configs are the
BASELINE ones (``configs.py``), optionally shrunk with ``--n``.
"""

from __future__ import annotations

import argparse
import csv
import sys

EXIT_OK, EXIT_FAIL, EXIT_USAGE = 0, 1, 2


def _csv_list(s: str):
    return [x for x in s.split(",") if x]


def _configs(args):
    from . import configs as C
    names = args.config or list(C.CONFIGS)
    for name in names:
        if name not in C.CONFIGS:
            raise SystemExit(f"unknown config {name!r}; expected one of {sorted(C.CONFIGS)}")
    return [C.get_config(name, args.n) for name in names]


def _device_problem(prob):
    import numpy as np
    import torch
    dev = torch.device("cuda")
    mesh = (torch.tensor(np.asarray(prob.mesh.coords).ravel(), device=dev),
            torch.tensor(np.asarray(prob.dofmap.cell2dof, np.int32).ravel(), device=dev),
            torch.tensor(np.asarray(prob.mesh.cell2vert, np.int32).ravel(), device=dev))
    coef = None
    if prob.coef() is not None:
        coef = tuple(None if c is None else torch.tensor(c, device=dev) for c in prob.coef())
    return mesh, torch.tensor(prob.u, device=dev), coef


def cmd_verify(args) -> int:
    import torch
    from . import configs as C
    from .harness import rel_l2
    from .jit import Target, compile_and_load, emit_for
    bad = 0
    for cfg in _configs(args):
        prob = C.build_problem(cfg, args.seed)
        mesh, u, coef = _device_problem(prob)
        outs = {}
        for generic in (False, True):
            try:
                h = compile_and_load(emit_for(prob.spec, Target(generic=generic), prob.rule))
            except Exception as e:  # no generic kernel for this rule
                outs[generic] = (None, str(e).split(":")[0])
                continue
            h.bind(*mesh, nglobal=prob.dofmap.ndofs_global)
            y = torch.zeros_like(u)
            h.apply(u, y, coef=coef, overwrite=True)
            outs[generic] = (y.cpu().numpy(), h.info["kernel"])
        (ys, ks), (yg, kg) = outs[False], outs[True]
        if yg is None:
            print(f"  {cfg.name}: {ks} (no generic kernel to compare: {kg})")
            continue
        err = rel_l2(ys, yg)
        ok = err <= args.rtol
        bad += not ok
        print(f"  {cfg.name}: {ks} vs {kg}: rel L2 {err:.2e} {'ok' if ok else 'FAIL'}")
    print(f"verify: {'all passed' if not bad else f'{bad} failed'}")
    return EXIT_OK if not bad else EXIT_FAIL


def cmd_bench(args) -> int:
    from . import configs as C
    from .harness import run_configuration, write_csv
    from .jit import Target
    records = []
    for cfg in _configs(args):
        prob = C.build_problem(cfg, args.seed)
        coef = prob.coef()
        rec = run_configuration(prob.spec, Target(), prob.mesh, prob.dofmap, trials=args.trials,
                                seed=args.seed, rule=prob.rule, u=prob.u,
                                mu=None if coef is None else coef[0],
                                lam=None if coef is None else coef[1])
        records.append(rec)
        print(f"  {cfg.name} {rec.target}: {rec.time_best_s * 1e6:.1f} us, {rec.gflops:.0f} GFLOP/s, "
              f"{rec.gdofs_per_s:.2f} GDoF/s, roofline {rec.roofline_fraction:.3f}")
    with open(args.output, "w", newline="") as f:
        write_csv(records, f)
    print(f"wrote {len(records)} records to {args.output}")
    return EXIT_OK


def cmd_report(args) -> int:
    from .harness import BenchmarkRecord, roofline_rows
    records = []
    for path in args.csv:
        with open(path, newline="") as f:
            for row in csv.DictReader(f):
                kw = {}
                for k, v in row.items():
                    f_ = BenchmarkRecord.__dataclass_fields__.get(k)
                    if f_ is None or v == "":
                        continue
                    t = f_.type if isinstance(f_.type, str) else f_.type.__name__
                    kw[k] = {"int": int, "float": float}.get(t, str)(v)
                records.append(BenchmarkRecord(**kw))
    if not records:
        print("report: no records", file=sys.stderr)
        return EXIT_USAGE
    ridge, rows = roofline_rows(records, args.peak, args.bandwidth)
    print(f"# peak {args.peak} GFLOP/s, bandwidth {args.bandwidth} GB/s, ridge point {ridge:.2f} flops/byte")
    header = ("operator", "cell", "degree", "target", "width", "ai", "gflops", "attainable_gflops",
              "fraction_of_attainable", "memory_bound")
    print(",".join(header))
    for r in rows:
        print(",".join(f"{r[k]:.4g}" if isinstance(r[k], float) else str(r[k]) for k in header))
    return EXIT_OK


def cmd_info(args) -> int:
    from . import configs as C
    from .harness import bytes_per_cell, flops_per_cell
    from .jit import Target, compile_and_load, emit_for
    for cfg in _configs(args):
        prob = C.build_problem(cfg, args.seed)
        h = compile_and_load(emit_for(prob.spec, Target(), prob.rule))
        print(f"  {cfg.name}: {cfg.form} {cfg.cell} k={cfg.degree} cells={prob.mesh.ncells:,} "
              f"dofs={prob.ndofs:,} kernel={h.info['kernel']} "
              f"F/cell={flops_per_cell(prob.spec, prob.rule):,} "
              f"B/cell={bytes_per_cell(prob.spec, prob.mesh, prob.dofmap):.1f}")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    from .harness import DEFAULT_BANDWIDTH_GBS, DEFAULT_PEAK_GFLOPS
    p = argparse.ArgumentParser(prog="python -m paper_1903_08243_b200",
                                description="B200 matrix-free FE operator action")
    sub = p.add_subparsers(dest="command")

    def common(sp):
        sp.add_argument("--config", type=_csv_list, default=None,
                        help="comma list of BASELINE configs (C1, C2-P1..C2-P4, C3-Q1.., C6); default all")
        sp.add_argument("--n", type=int, default=None, help="cells per direction (shrink the mesh)")
        sp.add_argument("--seed", type=int, default=0)

    v = sub.add_parser("verify", help="specialised kernel vs the generic quadrature kernel")
    common(v)
    v.add_argument("--rtol", type=float, default=1e-12)
    b = sub.add_parser("bench", help="time configurations and write a CSV")
    common(b)
    b.add_argument("--trials", type=int, default=20)
    b.add_argument("--output", default="bench.csv")
    r = sub.add_parser("report", help="roofline analysis of bench CSVs")
    r.add_argument("csv", nargs="+")
    r.add_argument("--peak", type=float, default=DEFAULT_PEAK_GFLOPS, help="FP64 GFLOP/s")
    r.add_argument("--bandwidth", type=float, default=DEFAULT_BANDWIDTH_GBS, help="HBM GB/s")
    i = sub.add_parser("info", help="selected kernel, flop and byte model per config")
    common(i)
    return p


def main(argv=None) -> int:
    parser = build_parser()
    args = parser.parse_args(list(sys.argv[1:] if argv is None else argv))
    if args.command is None:
        parser.print_help(sys.stderr)
        return EXIT_USAGE
    return {"verify": cmd_verify, "bench": cmd_bench, "report": cmd_report, "info": cmd_info}[args.command](args)
