"""CLI subcommands on the B200."""

import csv

import pytest

from paper_1903_08243_b200 import cli

pytestmark = pytest.mark.gpu


def test_verify_specialised_against_generic_kernels(capsys):
    assert cli.main(["verify", "--config", "C1,C2-P2,C2-P4,C3-Q1,C4-hex-Q1,C5,C6", "--n", "3"]) == cli.EXIT_OK
    out = capsys.readouterr().out
    assert "all passed" in out and "dmma_modal vs quad" in out


def test_bench_writes_the_extended_csv(tmp_path, capsys):
    path = tmp_path / "b.csv"
    assert cli.main(["bench", "--config", "C2-P2,C6", "--n", "4", "--trials", "3",
                     "--output", str(path)]) == cli.EXIT_OK
    rows = list(csv.DictReader(open(path)))
    assert [r["operator"] for r in rows] == ["helmholtz", "neohookean_tangent"]
    assert all(float(r["roofline_fraction"]) > 0 and float(r["gdofs_per_s"]) > 0 for r in rows)
    assert cli.main(["report", str(path)]) == cli.EXIT_OK
