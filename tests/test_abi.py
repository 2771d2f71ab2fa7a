"""The C-ABI library loads and exports every symbol include/drs.h declares (CPU only)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "drs.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dr_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_path():
    syms = declared_symbols()
    for s in ("dr_build_table", "dr_sorted_uniforms", "dr_match_binary", "dr_match_ccf", "dr_match_dac",
              "dr_check_sorted_open", "dr_resample_batched", "dr_shard_scan", "dr_shard_finalize"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2604_01356_b200 import _lib

    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_prototypes_cover_header():
    from paper_2604_01356_b200 import _lib

    assert set(declared_symbols()) == set(_lib._PROTOS)


def test_geometry_matches_oracle(orc):
    from paper_2604_01356_b200 import _lib

    lanes, warps, kt, ku, fan, grp = _lib.scan_geometry()
    assert (lanes, warps, kt, ku, fan, grp) == (32, 8, 33, 2, 16, 32)
    M = 123457
    assert _lib.load_library().dr_index_entries(M) == orc.lib().drs_ref_index_entries(M)


def test_no_gpu_means_loud_failure(monkeypatch):
    import torch

    from paper_2604_01356_b200 import _lib

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(RuntimeError, match="CUDA device"):
        _lib.lib()


def test_missing_library_is_loud(tmp_path):
    from paper_2604_01356_b200 import _lib

    with pytest.raises(RuntimeError, match="not built"):
        _lib.load_library(tmp_path / "libdrs.so")


def test_argument_errors_without_launch():
    from paper_2604_01356_b200 import _lib

    lib = _lib.load_library()
    assert lib.dr_build_table(None, 0, None, None, None, None, 0, None) == -1
    assert lib.dr_match_dac(None, None, 0, None, 0, None, 0, None) == -1
    assert lib.dr_strerror(-2) == b"workspace too small"
    assert lib.dr_workspace_bytes(1, 1 << 26, 0, 0) > lib.dr_workspace_bytes(1, 1 << 10, 0, 0)


def test_product_package_does_not_touch_oracle():
    pkg = ROOT / "paper_2604_01356_b200"
    for p in pkg.rglob("*.py"):
        src = p.read_text()
        assert "oracle" not in src.replace("oracle-backed", "").replace("linear_oracle", ""), p
