"""The C-ABI library loads and exports every symbol include/hetft.h declares
(no compute calls: this runs without a GPU)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "hetft.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_survey_boundary():
    syms = header_symbols()
    for s in ("hf_init", "hf_last_error", "hf_vote", "hf_copy", "hf_checkpoint", "hf_restore",
              "hf_inject_bitflip", "hf_inject_scale", "hf_scribble", "hf_gemm_tc", "hf_gemm_simt"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_1405_2912_b200 import _lib
    lib = _lib.load()
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_lib.EXPORTED) == set(header_symbols())


def test_result_struct_layout_matches_header():
    from paper_1405_2912_b200._lib import HfVoteResult
    assert ctypes.sizeof(HfVoteResult) == 8 * 8 + 8 + 8 + 4 * 4 + 8 + 8


def test_no_device_reports_cleanly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1405_2912_b200 import _lib
    lib = _lib.load()
    assert lib.hf_version() == 1
    assert lib.hf_device_count() == 0
    rc = lib.hf_init(0, 1)
    assert rc == _lib.HF_ENOINIT
    assert "no CUDA device" in _lib.last_error()
