"""CLI (reference cli.py simulate/sweep): CPU-side behaviour."""

from pathlib import Path

from paper_2510_22221_b200 import cli

ROOT = Path(__file__).resolve().parents[1]


def test_dry_run_prints_derived_quantities(capsys):
    assert cli.main(["--dry-run", "simulate", str(ROOT / "configs/c1.cfg")]) == 0
    out = capsys.readouterr().out
    assert "steps = 300" in out and "cells = (64, 64, 64)" in out


def test_sweep_dry_run(capsys):
    assert cli.main(["--dry-run", "sweep", str(ROOT / "configs/c2.cfg")]) == 0
    assert "sweep of 7 runs" in capsys.readouterr().out


def test_usage_and_config_errors(tmp_path):
    assert cli.main(["nonsense"]) == cli.EXIT_USAGE
    bad = tmp_path / "bad.cfg"
    bad.write_text("[grid]\nnx = 4\n")
    assert cli.main(["simulate", str(bad)]) == cli.EXIT_USAGE
