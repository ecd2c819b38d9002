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


def test_struct_layouts_match_the_c_header(tmp_path):
    """Compile a probe against include/hetft.h with the host C compiler and
    compare sizeof/offsetof of hf_vote_result and hf_vote_item (and
    HF_VOTE_BATCH_MAX) with the ctypes mirrors in _lib."""
    import shutil
    import subprocess
    from pathlib import Path
    from paper_1405_2912_b200 import _lib
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    inc = Path(__file__).resolve().parents[1] / "include"
    src = tmp_path / "probe.c"
    fields_r = [f for f, _ in _lib.HfVoteResult._fields_]
    fields_i = [f for f, _ in _lib.HfVoteItem._fields_]
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "hetft.h"', "int main(void) {",
             'printf("R %zu\\n", sizeof(hf_vote_result));', 'printf("I %zu\\n", sizeof(hf_vote_item));',
             'printf("B %d\\n", HF_VOTE_BATCH_MAX);']
    lines += [f'printf("r.{f} %zu\\n", offsetof(hf_vote_result, {f}));' for f in fields_r]
    lines += [f'printf("i.{f} %zu\\n", offsetof(hf_vote_item, {f}));' for f in fields_i]
    lines += ["return 0; }"]
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "probe"
    subprocess.run([cc, "-I", str(inc), str(src), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                        check=True).stdout.splitlines())
    assert int(got["R"]) == ctypes.sizeof(_lib.HfVoteResult)
    assert int(got["I"]) == ctypes.sizeof(_lib.HfVoteItem)
    assert int(got["B"]) == _lib.HF_VOTE_BATCH_MAX
    for f in fields_r:
        assert int(got[f"r.{f}"]) == getattr(_lib.HfVoteResult, f).offset, f
    for f in fields_i:
        assert int(got[f"i.{f}"]) == getattr(_lib.HfVoteItem, f).offset, f
