"""CLI with the reference's subcommands and exit codes (cli.py:1-255)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2208_06194_b200 import cli


def test_dag_dot_matches_scheduler(tmp_path):
    out = tmp_path / "dag.dot"
    assert cli.main(["dag", "--p", "4", "--q", "3", "--out", str(out)]) == 0
    text = out.read_text()
    assert text.startswith("digraph")
    assert "DiagQR(0)" in text and "ApplyTrapReflector(0,1,1)" in text
    from paper_2208_06194_b200.scheduler import build_tiled_dag
    assert text.strip() == build_tiled_dag(4, 3).to_dot().strip()


def test_usage_errors_exit_2():
    assert cli.main(["dag", "--p", "1", "--q", "2"]) == 2  # p < q
    assert cli.main(["bench"]) == 2  # no family / config
    assert cli.main(["nosuchcommand"]) == 2
    assert cli.main(["bench", "--family", "laplace", "--n", "1000", "--b", "64"]) == 2  # n % b
    assert cli.main(["bench", "--config", "C1", "--algo", "mgs", "--exec", "taskgraph"]) == 2


def test_verify_reference_written_blr1(capsys):
    assert cli.main(["verify", "--in", os.path.join(GOLDEN, "blr1_mixed.bin")]) == 0
    info = json.loads(capsys.readouterr().out)
    assert info["m"] == 96 and info["n"] == 64 and info["b"] == 16 and info["max_rank"] == 4


def test_verify_compression_error_threshold(tmp_path, capsys):
    from paper_2208_06194_b200 import blr_to_dense, load_blr1
    path = os.path.join(GOLDEN, "blr1_mixed.bin")
    with open(path, "rb") as fh:
        d = blr_to_dense(load_blr1(fh))
    noisy = d + 1e-3 * np.linalg.norm(d) / np.sqrt(d.size) * np.random.default_rng(0).standard_normal(d.shape)
    np.save(tmp_path / "d.npy", noisy)
    assert cli.main(["verify", "--in", path, "--dense", str(tmp_path / "d.npy"), "--eps", "1e-1"]) == 0
    assert cli.main(["verify", "--in", path, "--dense", str(tmp_path / "d.npy"), "--eps", "1e-8"]) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["tiled-hh", "blocked-hh", "mgs"])
def test_bench_report_and_thresholds(tmp_path, algo):
    import __graft_entry__ as ge
    ge.build()
    out, csvp = tmp_path / "r.json", tmp_path / "r.csv"
    args = ["bench", "--family", "laplace", "--n", "2048", "--b", "256", "--eps", "1e-8", "--algo", algo,
            "--out", str(out), "--csv", str(csvp), "--dump-r", str(tmp_path / "r.blr1")]
    assert cli.main(args + ["--max-res", "1e-6", "--max-orth", "1e-6"]) == 0
    rep = json.loads(out.read_text())
    assert rep["algorithm"] == algo and rep["n"] == 2048 and rep["b"] == 256
    assert rep["res"] < 1e-6 and rep["orth"] < 1e-6 and rep["flops_total"] > 0
    assert rep["wall_ms"]["factorize"] > 0
    assert csvp.read_text().splitlines()[0].startswith("family,algo,exec")
    assert cli.main(["verify", "--in", str(tmp_path / "r.blr1")]) == 0
    # an impossible threshold is a numeric failure (exit 1)
    assert cli.main(args + ["--max-res", "1e-30"]) == 1


@pytest.mark.gpu
def test_gen_then_verify_roundtrip(tmp_path):
    import __graft_entry__ as ge
    ge.build()
    blr, dense = tmp_path / "a.blr1", tmp_path / "a.npy"
    assert cli.main(["gen", "--family", "expcov", "--n", "2048", "--b", "256", "--eps", "1e-8", "--out", str(blr),
                     "--dense-out", str(dense)]) == 0
    assert cli.main(["verify", "--in", str(blr), "--dense", str(dense), "--eps", "1e-7"]) == 0
