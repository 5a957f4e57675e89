"""Host-side parts of the device harness / CLI against
the reference's conventions (harness.py:87-131, 375-422; cli.py:27-170), and
the low-rank-update input row (lru_cov3d) against the reference's operator."""
import csv
import json

import pytest

from golden_util import h2_digest, load, problem
from paper_2509_11152_b200 import cli
from paper_2509_11152_b200.harness import (PROBLEMS, ExperimentConfig, write_outputs, write_sweep_outputs,
                                           write_thread_outputs)


def test_config_rows_and_overrides():
    c = ExperimentConfig.from_problem("cov2d", 16384)
    assert (c.m, c.p0, c.eta, c.eps, c.eps_lu, c.lru_rank) == (64, 8, 0.9, 1e-7, 1e-6, 0)
    c = ExperimentConfig.from_problem("lru_cov3d", 4096, eps_lu=None, seed=3)
    assert (c.m, c.eta, c.eps, c.eps_lu, c.lru_rank, c.seed) == (128, 0.9, 1e-8, 1e-7, 32, 3)
    assert set(PROBLEMS) == {"cov2d", "cov3d", "laplace2d", "helmholtz3d", "lru_cov3d"}
    with pytest.raises(ValueError):
        ExperimentConfig.from_problem("nope", 10)


def test_lru_operator_matches_reference():
    g = load("lru_cov3d_4096")
    _, _, _, h2, _ = problem("lru_cov3d_4096")
    assert h2_digest(h2) == str(g["h2_digest"])


def test_writers_layout(tmp_path):
    rep = {"version": "x", "n": 4, "e_b": 1e-12, "timings": {"factorization": 1.0},
           "phases": {"construction": 1.0, "partial_lu": 3.0},
           "levels": [{"level": 3, "time_s": 0.5, "csp": 9, "max_rank": 40}], "solution": [1, 2],
           "profile": {"kernels": {"gemm_schur": {"seconds": 1.0, "launches": 2, "gflop": 3.0, "gbytes": 4.0,
                                                  "bound": "tensor", "achieved": 3.0, "unit": "TFLOP/s",
                                                  "frac": 0.1}}}}
    write_outputs(rep, tmp_path)
    d = json.load(open(tmp_path / "report.json"))
    assert "solution" not in d and d["e_b"] == 1e-12
    rows = list(csv.reader(open(tmp_path / "levels.csv")))
    assert rows == [["level", "time_s", "csp", "max_rank"], ["3", "5.000000e-01", "9", "40"]]
    rows = list(csv.reader(open(tmp_path / "phases.csv")))
    assert rows[0] == ["phase", "time_s", "fraction"] and rows[2] == ["partial_lu", "3.000000e+00", "7.500000e-01"]
    assert list(csv.reader(open(tmp_path / "roofline.csv")))[1][0] == "gemm_schur"
    write_sweep_outputs({"rows": [{"n": 10, "factorization_s": 0.5}], "slopes": {"factorization_time": 1.01}},
                        tmp_path)
    assert list(csv.reader(open(tmp_path / "sweep.csv")))[1] == ["10", "5.000000e-01"]
    assert json.load(open(tmp_path / "slopes.json")) == {"factorization_time": 1.01}
    write_thread_outputs([{"threads": 1, "speedup": 1.0}], tmp_path)
    assert list(csv.reader(open(tmp_path / "threads.csv")))[0] == ["threads", "speedup"]


def test_cli_parses_reference_options():
    a = cli.parse(["sweep", "--problem", "helmholtz3d", "--n", "0", "--sizes", "1024,2048,4096", "--kappa", "0",
                   "--eps-lu", "1e-6", "--alpha-r", "0.01", "--refine-steps", "2", "--out", "o"])
    o = cli._overrides(a)
    assert a.command == "sweep" and o["kappa"] == 0.0 and o["eps_lu"] == 1e-6 and o["refine_steps"] == 2
    with pytest.raises(SystemExit):
        cli.parse(["run", "--problem", "nope", "--n", "4"])
