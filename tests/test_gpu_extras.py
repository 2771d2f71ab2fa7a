"""gather by index, device histogram and chi-square, CLI, on the GPU."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_gather_states_matches_numpy_take(drs):
    rng = np.random.default_rng(3)
    for K, d, div in [(1000, 40, 1), (257, 7, 1), (64, 40, 16), (5, 1, 3)]:
        states = rng.standard_normal((K, d))
        idx = rng.integers(0, K * div, size=5000)
        np.testing.assert_array_equal(drs.gather_states(states, idx, divisor=div), states[idx // div])
        out = drs.gather_states(torch.from_numpy(states).cuda(), torch.from_numpy(idx).cuda(), divisor=div)
        np.testing.assert_array_equal(out.cpu().numpy(), states[idx // div])
    with pytest.raises(IndexError):
        drs.gather_states(np.zeros((4, 2)), np.array([0, 4]))
    assert drs.gather_states(np.zeros((4, 2)), np.zeros(0, dtype=np.int64)).shape == (0, 2)


def test_resample_then_gather_pipeline(drs):
    """dac_sampler indices -> states of the chosen particles (EnGMF component = particle * N_Y + center)."""
    rng = np.random.default_rng(8)
    n, ny, d = 256, 64, 40
    w = np.exp(rng.standard_normal(n * ny))
    t = drs.build_weight_table(w)
    idx = drs.dac_sampler(t, n, drs.RngStream(5), device=True)
    x = torch.from_numpy(rng.standard_normal((n, d))).cuda()
    out = drs.gather_states(x, idx, divisor=ny)
    np.testing.assert_array_equal(out.cpu().numpy(), x.cpu().numpy()[idx.cpu().numpy() // ny])


def test_histogram_matches_bincount(drs):
    rng = np.random.default_rng(1)
    for m, n in [(16, 1_000_000), (1, 10), (100_000, 3_000_000)]:
        idx = np.sort(rng.integers(0, m, size=n)) if m > 1 else np.zeros(n, dtype=np.int64)
        np.testing.assert_array_equal(drs.histogram(idx, m), np.bincount(idx, minlength=m))
        rng.shuffle(idx)
        np.testing.assert_array_equal(drs.histogram(idx, m), np.bincount(idx, minlength=m))
    with pytest.raises(ValueError):
        drs.histogram(np.array([0, 5]), 5)


def test_chi_square_matches_reference_formula(drs):
    rng = np.random.default_rng(2)
    for m in (16, 1000, 300_000):
        w = rng.exponential(size=m)
        t = drs.build_weight_table(w)
        n = 1_000_000
        counts = rng.multinomial(n, t.weights().clip(0))
        expected = n * t.weights()
        ref = float(((counts.astype(np.float64) - expected) ** 2 / expected).sum())  # bench.py:221-225
        got = drs.chi_square_statistic(counts, t, n)
        assert abs(got - ref) <= 1e-12 * abs(ref)


def test_verify_statistics_passes(drs):
    reps = drs.verify_statistics(0)
    assert [r.sampler for r in reps] == ["dac", "ccf", "binary"]
    assert all(r.passed and r.dof == 15 for r in reps)


def test_cli_sample_matches_sampler(drs, tmp_path, capsys):
    from paper_2604_01356_b200.cli import main

    w = np.random.default_rng(4).exponential(size=300)
    f = tmp_path / "w.txt"
    f.write_text(" ".join(repr(float(v)) for v in w))
    for sampler in ("dac", "ccf", "binary"):
        assert main(["sample", str(f), "--sampler", sampler, "--n", "50", "--seed", "7"]) == 0
        got = [int(x) for x in capsys.readouterr().out.split()]
        fn = {"dac": drs.dac_sampler, "ccf": drs.ccf_sampler, "binary": drs.binary_sampler}[sampler]
        assert got == fn(drs.build_weight_table(w), 50, drs.RngStream(7)).tolist()
    assert main(["verify"]) == 0


def test_cli_bench_writes_reference_schema(drs, tmp_path):
    from paper_2604_01356_b200.cli import main

    out = tmp_path / "r.csv"
    assert main(["bench", "--n-min", "100", "--n-max", "1000", "--n-points", "2", "--ratios", "1,10",
                 "--trials", "2", "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == "Ns,timesdcM1,timesccfM1,timesbM1,timesdcM10,timesccfM10,timesbM10"
    assert len(lines) == 3 and all(float(v) > 0 for v in lines[1].split(",")[1:])


@pytest.mark.parametrize("M", [1, 2, 17, 8448, 8449, 300_001, 256 * 8448 + 5])
def test_log_table_bit_exact_vs_oracle(drs, orc, M):
    """max -> exp -> scan fused on the device == the oracle
    twin bit for bit (W and the index), across tile and group boundaries."""
    rng = np.random.default_rng(M)
    lw = np.log(1 / 256) + np.log(rng.dirichlet(np.ones(64), size=max(1, M // 64 + 1)).ravel()[:M]) \
        - 0.5 * rng.chisquare(6, size=M)
    t = drs.build_weight_table_from_log(lw)
    Wo, st = orc.build_table_log(lw)
    assert st == 0
    np.testing.assert_array_equal(t.cum, Wo)
    ns = orc.search_entries(M)
    ref_idx, _ = orc.index_l1_local(t.device_values.cpu().numpy(), orc.build_index(Wo))
    np.testing.assert_array_equal(t.device_index.cpu().numpy()[:ns], ref_idx[:ns])
    # the same table as build_weight_table of the device-exp weights
    np.testing.assert_array_equal(drs.build_weight_table(orc.exp(lw - lw.max())).cum, Wo)
    # and close to the reference pipeline np.exp + build_weight_table
    Wp, _ = orc.port_build_table(np.exp(lw - lw.max()))
    assert np.abs(t.cum - Wp).max() <= 1e-12


def test_log_table_errors(drs):
    with pytest.raises(ValueError, match="empty distribution"):
        drs.build_weight_table_from_log(np.zeros(0))
    with pytest.raises(ValueError, match="invalid weight"):
        drs.build_weight_table_from_log(np.array([0.0, np.nan, 1.0]))
    with pytest.raises(ValueError, match="invalid weight"):
        drs.build_weight_table_from_log(np.array([0.0, np.inf]))
    t = drs.build_weight_table_from_log(np.array([-np.inf, 0.0, -np.inf]))  # exp(-inf) = 0 weights
    np.testing.assert_array_equal(t.cum, [0.0, 1.0, 1.0])
