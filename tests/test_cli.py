"""CLI plumbing (CPU only): parser, grid and the reference CSV schema (bench.py:136-155)."""

from paper_2604_01356_b200 import cli


def test_csv_header_matches_reference_schema():
    assert cli.csv_header((1, 100, 1000)) == (
        "Ns,timesdcM1,timesccfM1,timesbM1,timesdcM100,timesccfM100,timesbM100,"
        "timesdcM1000,timesccfM1000,timesbM1000")


def test_n_grid_is_reference_geomspace():
    assert cli.n_grid(100, 10_000, 5) == [100, 316, 1000, 3162, 10000]


def test_write_csv_nan_for_missing(tmp_path):
    p = tmp_path / "x.csv"
    cli.write_csv(str(p), [100, 200], (1,), {(100, 1, "dac"): 1.5e-6})
    lines = p.read_text().splitlines()
    assert lines[1] == "100,1.500000e-06,nan,nan"
    assert p.read_text().endswith("\n")


def test_parser_subcommands():
    ap = cli._build_parser()
    a = ap.parse_args(["sample", "--sampler", "ccf", "--n", "5"])
    assert (a.command, a.sampler, a.n, a.weights_file) == ("sample", "ccf", 5, "-")
    a = ap.parse_args(["bench", "--quick"])
    assert a.quick and a.ratios == "1,100,1000"
