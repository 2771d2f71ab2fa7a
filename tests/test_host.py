"""Host-side logic that needs no GPU: stream keys, partitions, error mapping, bench inputs."""

import numpy as np
import pytest


def test_rngstream_key_and_accounting():
    from paper_2604_01356_b200.randkit import RngStream

    s = RngStream(2003)
    k = np.random.SeedSequence(2003).generate_state(2, np.uint64)
    assert s.key == (int(k[0]), int(k[1]))
    assert s._take(5) == 0 and s._take(3) == 5 and s.draws == 8 and s.position == 8
    c = s.substream(4).substream(2)
    k2 = np.random.SeedSequence(2003, spawn_key=(4, 2)).generate_state(2, np.uint64)
    assert c.key == (int(k2[0]), int(k2[1])) and c.draws == 0
    assert repr(c) == "RngStream(seed=2003, substream=(4, 2))"
    with pytest.raises(NotImplementedError):
        s.normals(3)


def test_shard_filters_partition():
    from paper_2604_01356_b200.batched import shard_filters

    for B in (1, 7, 4096):
        for world in (1, 2, 3, 8):
            cover = []
            for r in range(world):
                sl = shard_filters(B, r, world)
                cover.extend(range(B)[sl])
            assert cover == list(range(B))


def test_error_priority_matches_reference_order():
    from paper_2604_01356_b200.cdf import _raise_build_status, _raise_table_status

    with pytest.raises(ValueError, match="invalid weight"):
        _raise_build_status(0x1 | 0x2 | 0x4)
    with pytest.raises(ValueError, match="degenerate distribution"):
        _raise_build_status(0x2 | 0x4)
    with pytest.raises(ValueError, match="accumulation overflow"):
        _raise_build_status(0x4)
    _raise_build_status(0x20)  # repaired is informational
    with pytest.raises(ValueError, match="invalid weight"):
        _raise_table_status(0x40 | 0x80)
    with pytest.raises(ValueError, match="non-decreasing"):
        _raise_table_status(0x80 | 0x100)
    with pytest.raises(ValueError, match="end at exactly 1"):
        _raise_table_status(0x100)


def test_bench_weights_are_seeded():
    import bench

    a = bench.make_weights("c1")
    b = bench.make_weights("c1")
    np.testing.assert_array_equal(a, b)
    assert a.shape == (1 << 16,) and np.all(a > 0)
    np.testing.assert_array_equal(a, np.exp(np.random.default_rng(1001).standard_normal(1 << 16)))


def test_bench_c4_weights_shard_consistently():
    import bench

    full = bench.make_weights("c4", 0, 512)  # 8 filters of rank 0 of 512
    part = bench.make_weights("c4", 1, 512)
    assert full.shape == (8, 16384) and part.shape == (8, 16384)
    assert not np.array_equal(full, part)
    np.testing.assert_allclose(full.sum(axis=1) > 0, True)


def test_reference_arm_runs_on_cpu(capsys):
    import json
    import sys

    import bench

    argv = sys.argv
    sys.argv = ["bench.py", "--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0"]
    try:
        bench.main()
    finally:
        sys.argv = argv
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0
