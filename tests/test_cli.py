"""The CLI (paper_1810_09891_b200/cli.py) against the reference CLI's own
outputs (tests/golden/cli/, produced by make_cli_golden.py running nfftk.cli):
exit codes, error messages, CSV rows, result files.  Usage / I/O paths run on
the CPU; anything that builds a plan is a GPU test."""

import csv
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1810_09891_b200 import cli

DIR = os.path.join(GOLDEN, "cli")
G = json.load(open(os.path.join(DIR, "cli_golden.json")))


def argv_of(name, tmp):
    return [a.replace("{dir}", DIR).replace("{tmp}", str(tmp)) for a in G[name]["argv"]]


def run(name, tmp, capsys, extra=()):
    rc = cli.main(argv_of(name, tmp) + list(extra))
    return rc, capsys.readouterr()


# ---------------------------------------------------------------- CPU
@pytest.mark.parametrize("name", ["usage_no_fhat", "usage_dim_mismatch"])
def test_usage_errors_match_reference(name, tmp_path, capsys):
    rc, cap = run(name, tmp_path, capsys)
    assert rc == G[name]["rc"] == 2
    assert cap.err.strip().splitlines()[-1] == G[name]["stderr"]


def test_malformed_file_matches_reference(tmp_path, capsys):
    rc, cap = run("io_malformed", tmp_path, capsys)
    assert rc == G["io_malformed"]["rc"] == 2
    assert cap.err.strip().endswith("nodes_bad.txt:3: malformed number")
    assert G["io_malformed"]["stderr"].endswith("nodes_bad.txt:3: malformed number")


def test_file_format_errors(tmp_path):
    p = tmp_path / "v.txt"
    p.write_text("1 2 3\n")
    with pytest.raises(cli.CliError, match=r"v.txt:1: expected 're im' pair, got 3 fields"):
        cli.read_complex_vector(str(p))
    p.write_text("0.1\n")
    with pytest.raises(cli.CliError, match=r"v.txt:1: expected 2 coordinates, got 1"):
        cli.read_nodes(str(p), 2)
    p.write_text("\n\n")
    with pytest.raises(cli.CliError, match="no nodes found"):
        cli.read_nodes(str(p), 2)
    with pytest.raises(cli.CliError, match="cannot open"):
        cli.read_nodes(str(tmp_path / "missing.txt"), 2)


def test_vector_round_trip(tmp_path):
    v = np.array([1.0 / 3 - 2j, np.nextafter(0.5, 1) + 1e-300j, -0.0 + 0j])
    cli.write_complex_vector(str(tmp_path / "v.txt"), v)
    assert np.array_equal(cli.read_complex_vector(str(tmp_path / "v.txt")), v)


def test_generators_match_reference():
    """Values printed by the reference cli (gen_nodes seed 5, gen_fhat_test,
    _default_n_grid)."""
    x = cli.gen_nodes(2, 3, 5)
    assert np.allclose(x, [[0.30500292, 0.30794079], [0.01532556, -0.21419862],
                           [-0.4460693, -0.11663112]], atol=5e-9)
    assert np.allclose(cli.gen_fhat_test((4, 2)).real,
                       [0.30901699, 0.33333333, 0.41421356, 0.5, 0.5, 1.0, 0.41421356, 0.5], atol=5e-9)
    assert cli._default_n_grid(16) == [18, 22, 24, 28, 30, 34, 36, 40, 42, 46, 48, 52, 54, 58, 60, 64]
    with pytest.raises(cli.CliError):
        cli.gen_nodes(2, 0, 1)


# ---------------------------------------------------------------- GPU
def rows_of(path):
    with open(path) as fh:
        return list(csv.DictReader(fh))


def close(a, b, rtol=1e-6):
    a, b = float(a), float(b)
    return abs(a - b) <= rtol * abs(b) + 1e-15


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["verify_d1", "verify_d2", "verify_d3_gauss", "verify_fail_tol",
                                  "bench_m", "bench_n"])
def test_csv_rows_match_reference(name, tmp_path, capsys):
    out = tmp_path / "rows.csv"
    rc, _ = run(name, tmp_path, capsys, extra=["--out", str(out)])
    assert rc == G[name]["rc"]
    rows = rows_of(out)
    assert list(rows[0].keys()) == cli.CSV_FIELDS
    assert len(rows) == len(G[name]["rows"])
    for got, ref in zip(rows, G[name]["rows"]):
        for k in ("dim", "N", "n", "m"):
            assert got[k] == ref[k]
        assert close(got["e2"], ref["e2"]) and close(got["einf"], ref["einf"])
        assert float(got["trafo_ms"]) > 0 and float(got["precompute_ms"]) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("name,outfile", [("transform_d2", "out_trafo_d2.txt"),
                                          ("transform_d2_adjoint", "out_adjoint_d2.txt"),
                                          ("transform_d3", "out_trafo_d3.txt")])
def test_transform_files_match_reference(name, outfile, tmp_path, capsys):
    rc, _ = run(name, tmp_path, capsys)
    assert rc == 0
    got = cli.read_complex_vector(str(tmp_path / outfile))
    ref = cli.read_complex_vector(os.path.join(DIR, outfile))
    assert got.shape == ref.shape
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
