"""CLI host logic: parser, CSV schema, report (no GPU)."""

import io

from paper_1903_08243_b200 import cli
from paper_1903_08243_b200.harness import CSV_COLUMNS, BenchmarkRecord, write_csv


def _rec(**kw):
    base = dict(operator="helmholtz", cell="tetrahedron", degree=4, target="dmma_modal", width=256,
                ncells=1572864, trials=20, time_best_s=6.9e-4, time_mean_s=7.0e-4,
                flops_per_cell=11300, gflops=25760.0, ai=35.6, speedup=1.0, flags="sm_100a", seed=0,
                gdofs_per_s=24.6, roofline_fraction=0.69, parity_rel_l2=1e-15)
    base.update(kw)
    return BenchmarkRecord(**base)


def test_csv_schema_extends_the_reference(tmp_path):
    ref_cols = ("operator", "cell", "degree", "target", "width", "ncells", "trials", "time_best_s",
                "time_mean_s", "flops_per_cell", "gflops", "ai", "speedup", "flags", "seed")
    assert CSV_COLUMNS[:len(ref_cols)] == ref_cols          # reference bench.py:38-42 first
    for c in ("gpus", "gdofs_per_s", "roofline_fraction", "parity_rel_l2", "cpu_cores", "cpu_time_s"):
        assert c in CSV_COLUMNS


def test_report_reads_bench_csv(tmp_path, capsys):
    path = tmp_path / "b.csv"
    with open(path, "w", newline="") as f:
        write_csv([_rec(), _rec(operator="mass", cell="triangle", degree=2, ai=1.3, gflops=1249.0)], f)
    assert cli.main(["report", str(path)]) == cli.EXIT_OK
    out = capsys.readouterr().out
    assert "ridge point" in out and "helmholtz,tetrahedron,4" in out
    lines = [l for l in out.splitlines() if l.startswith("mass")]
    assert lines and lines[0].endswith("True")                # C1 is memory bound


def test_parser_and_usage(capsys):
    assert cli.main([]) == cli.EXIT_USAGE
    a = cli.build_parser().parse_args(["bench", "--config", "C2-P3,C2-P4", "--trials", "5"])
    assert a.config == ["C2-P3", "C2-P4"] and a.trials == 5
