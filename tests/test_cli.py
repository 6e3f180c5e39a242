"""CLI on the B200 backend (paper_2508_00441_b200.cli), pinned to vectors the
reference CLI produced (tests/golden/gen_cli_golden.py): the SplitMix64 input
stream, the slices-table CSV, and `gemm` reports + C dumps (bitwise)."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2508_00441_b200 import cli

GOLD = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLD / "cli.json").read_text())
ARR = np.load(GOLD / "cli.npz")


def run(capsys, *argv):
    code = cli.main(list(argv))
    return code, capsys.readouterr().out


@pytest.mark.parametrize("i", range(len(META["gen"])))
def test_gen_matrix_matches_reference_stream(i):
    r, c, seed, lo, hi = META["gen"][i]
    x = cli.gen_matrix(r, c, seed, lo, hi)
    assert np.array_equal(x.view(np.uint64), ARR[f"gen{i}"])


def test_gen_matrix_properties():
    x = cli.gen_matrix(100, 100, 0, 1.0, 10.0)
    assert np.all(x > 1.0) and np.all(x < 10.0)
    with pytest.raises(ValueError):
        cli.gen_matrix(2, 2, 0, 5.0, 5.0)


def test_slices_table_matches_reference(capsys):
    code, out = run(capsys, "slices-table")
    assert code == 0 and out == META["slices_table"]


def test_make_inputs_modes():
    A, B = cli.make_inputs(4, 4, 4, 0, "identity")
    assert np.array_equal(A, np.eye(4))
    A, B = cli.make_inputs(3, 5, 4, 1, "powers2")
    assert np.all(np.log2(A) == np.round(np.log2(A))) and B.shape == (4, 5)
    with pytest.raises(SystemExit):
        cli.make_inputs(3, 4, 5, 0, "identity")


def test_version_and_bad_format_without_gpu(capsys):
    with pytest.raises(SystemExit):
        cli.main(["--version"])
    # unknown format: ValueError from get_format -> exit code 2 (reference behaviour), no GPU needed
    assert cli.main(["gemm", "--m", "4", "--n", "4", "--k", "8", "--type2", "fp4"]) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(META["gemm"])))
def test_gemm_report_and_dump_match_reference(cuda, capsys, tmp_path, i):
    case = META["gemm"][i]
    dump = tmp_path / "c.npy"
    code, out = run(capsys, *case["argv"], "--dump", str(dump))
    assert code == 0
    rep = json.loads(out)
    rep["stats"].pop("wall_s")
    rep.pop("wall_s_total")
    rep.pop("c_dump")
    assert rep == case["report"]
    assert np.array_equal(np.load(dump).view(np.uint64), ARR[f"c{i}"])


@pytest.mark.gpu
def test_accuracy_and_verify(cuda, capsys):
    code, out = run(capsys, "accuracy", "--m", "64", "--n", "48", "--k", "256", "--type2", "fp8e4m3")
    rep = json.loads(out)
    assert code == 0 and rep["err_oz"] <= rep["err_naive"] and rep["err_oz"] < 1e-13
    code, out = run(capsys, "verify", "--trials", "2000")
    rep = json.loads(out)
    assert code == 0 and rep["pass"] is True
    assert set(rep["suites"]) == {"fp64emu", "reconstruction", "errorfree"}
    assert all(s["checks"] > 0 and s["failures"] == 0 for s in rep["suites"].values())
    assert rep["suites"]["fp64emu"]["checks"] == 3 * 2000 + 1000  # reference schema: add, sub, mul + lt
