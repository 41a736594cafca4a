"""CLI contract (ref tests/test_cli.py, acceptance criteria 2 and 11).
Config errors are checked on CPU; runs need the GPU (marked)."""

import json

import pytest

from paper_2109_09056_b200 import cli


def test_unknown_config_key_exit_2(tmp_path, capsys):
    f = tmp_path / "c.json"
    f.write_text(json.dumps({"subcommannd": "md"}))
    assert cli.main(["md", "--config", str(f)]) == 2
    assert "unknown key: subcommannd" in capsys.readouterr().err


def test_bad_values_and_constraints_exit_2(tmp_path, capsys):
    f = tmp_path / "c.json"
    f.write_text(json.dumps({"steps": "many"}))
    assert cli.main(["md", "--config", str(f)]) == 2
    assert cli.main(["md", "--dt", "-0.1", "--output", "-"]) == 2
    assert cli.main(["md", "--cutoff", "99", "--output", "-"]) == 2
    assert cli.main(["md", "--ranks", "2,2", "--output", "-"]) == 2
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"steps": 5, "lattice_sells": 4}))
    assert cli.main(["md", "--config", str(bad)]) == 2
    assert "lattice_sells" in capsys.readouterr().err


def test_subcommand_mismatch_exit_2(tmp_path, capsys):
    f = tmp_path / "c.json"
    f.write_text(json.dumps({"subcommand": "pic"}))
    assert cli.main(["md", "--config", str(f)]) == 2
    capsys.readouterr()


def test_parse_precedence():
    cfg = cli.parse_config("md", None, {"steps": "7", "lattice_cells": None})
    assert cfg["steps"] == 7 and cfg["lattice_cells"] == 4


@pytest.mark.gpu
def test_seeded_runs_byte_identical_and_format(tmp_path):
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    args = ["md", "--steps", "5", "--lattice-cells", "3", "--density", "1.1", "--cutoff",
            "2.0", "--seed", "9"]
    assert cli.main(args + ["--output", str(a)]) == 0
    assert cli.main(args + ["--output", str(b)]) == 0
    assert a.read_bytes() == b.read_bytes()
    raw = a.read_bytes()
    assert b"\r" not in raw
    lines = raw.decode().splitlines()
    assert lines[0].startswith("# ") and "steps=5" in lines[0]
    assert lines[1] == "step,KE,PE,E_total,temperature"
    assert len(lines) == 2 + 6
    assert (tmp_path / "a.csv.phases.csv").read_bytes().splitlines()[1] == b"phase,seconds"


@pytest.mark.gpu
def test_layout_transparency(tmp_path):
    """Criterion 2 (md part): physics rows bitwise identical for V in {1,4,8,16,SoA}.
    V is the vector length of the AoSoA particle store the engine ingests its
    initial state through (MDDriver, pc_aosoa_field); the step loop then runs
    on SoA working arrays, so the rows must not depend on V."""
    n_md = 4 * 4 ** 3
    outs = []
    for v in (1, 4, 8, 16, n_md):
        p = tmp_path / f"md_{v}.csv"
        assert cli.main(["md", "--steps", "10", "--lattice-cells", "4", "--density", "1.1",
                         "--cutoff", "2.3", "--vector-length", str(v), "--output",
                         str(p)]) == 0
        outs.append(p.read_bytes().split(b"\n", 1)[1])
    assert all(o == outs[0] for o in outs)


@pytest.mark.gpu
def test_layout_bench_and_fabric(tmp_path):
    p = tmp_path / "lb.csv"
    assert cli.main(["layout-bench", "--steps", "3", "--lattice-cells", "4", "--density",
                     "1.1", "--cutoff", "2.3", "--vector-lengths", "1,16", "--output",
                     str(p)]) == 0
    lines = p.read_text().splitlines()
    assert lines[1] == "vector_length,phase,seconds,checksum"
    sums = {ln.split(",")[3] for ln in lines[2:]}
    assert len(sums) == 1
    # the V-dependent part: an AoSoA <-> SoA round trip of all fields per step
    rt = {ln.split(",")[0]: float(ln.split(",")[2]) for ln in lines[2:]
          if ln.split(",")[1] == "store_roundtrip"}
    assert set(rt) == {"1", "16"} and all(t > 0 for t in rt.values())
    q = tmp_path / "fab.csv"
    assert cli.main(["md", "--steps", "5", "--lattice-cells", "4", "--density", "1.1",
                     "--cutoff", "2.3", "--ranks", "2,2,2", "--output", str(q)]) == 0
    assert len(q.read_text().splitlines()) == 8


@pytest.mark.gpu
def test_ranks_byte_identical_deterministic(tmp_path):
    """Criterion 3 through the CLI (ref test_acceptance.py:79-92): in the default
    deterministic mode the physics rows are byte-identical for ranks 1x1x1 and
    2x2x2; --parallel (tile path) runs too."""
    outs = []
    for ranks in ("1,1,1", "2,2,2", "2,1,1"):
        p = tmp_path / f"r{ranks.replace(',', '')}.csv"
        assert cli.main(["md", "--steps", "12", "--lattice-cells", "6", "--rebuild-stride", "5",
                         "--skin", "0.3", "--ranks", ranks, "--output", str(p)]) == 0
        outs.append(p.read_bytes().split(b"\n", 1)[1])
    assert outs[0] == outs[1] == outs[2]
    q = tmp_path / "par.csv"
    assert cli.main(["md", "--steps", "12", "--lattice-cells", "6", "--parallel", "--output",
                     str(q)]) == 0
    assert len(q.read_text().splitlines()) == 2 + 13


def _golden_args():
    import importlib.util
    import os
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    spec = importlib.util.spec_from_file_location("make_cli_golden",
                                                  os.path.join(here, "make_cli_golden.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return here, mod.CASES


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["md_4", "md_6_ranks"])
def test_md_csv_matches_reference_cli(tmp_path, case):
    """f1 vs the reference CLI itself (tests/golden/make_cli_golden.py ran
    ``particula md`` unchanged, ref cli.py:173-206): the ``#`` echo line and
    the header byte for byte, every diagnostics value within 1e-8 relative
    (deterministic mode: FP64 LJ, id-ordered sums), the phases sidecar with
    the reference's six buckets."""
    import numpy as np
    here, cases = _golden_args()
    p = tmp_path / f"{case}.csv"
    assert cli.main(["md", *cases[case], "--output", str(p)]) == 0
    mine = p.read_text().splitlines()
    with open(f"{here}/cli_{case}.csv") as fh:
        ref = fh.read().splitlines()
    assert mine[0] == ref[0] and mine[1] == ref[1]
    assert len(mine) == len(ref)
    a = np.array([[float(t) for t in ln.split(",")] for ln in mine[2:]])
    b = np.array([[float(t) for t in ln.split(",")] for ln in ref[2:]])
    assert np.array_equal(a[:, 0], b[:, 0])
    assert np.max(np.abs(a[:, 1:] - b[:, 1:]) / np.abs(b[:, 1:])) < 1e-8
    side = (tmp_path / f"{case}.csv.phases.csv").read_text().splitlines()
    assert side[0] == ref[0] and side[1] == "phase,seconds"
    assert [ln.split(",")[0] for ln in side[2:]] == sorted(
        ["force", "halo", "integrate", "migrate", "neighbor", "sort"])
