"""NVTX ranges around the voted-task phases (tracing beside the
reference's ATT/VOTE/DONE lines).  Off unless HETFT_NVTX=1, so the product
path pays one attribute check; on, every task, replica round, vote and
settle shows up as a named range in nsys / ncu (`--nvtx --nvtx-include`).

    with nvtx.range("vote"):
        ...
"""

from __future__ import annotations

import contextlib
import os

ENABLED = os.environ.get("HETFT_NVTX", "0") not in ("", "0")

_push = _pop = None
if ENABLED:
    try:
        import torch
        _push, _pop = torch.cuda.nvtx.range_push, torch.cuda.nvtx.range_pop
    except Exception:  # noqa: BLE001 - no torch/CUDA: ranges become no-ops
        ENABLED = False


@contextlib.contextmanager
def _range(name: str):
    _push(name)
    try:
        yield
    finally:
        _pop()


_NULL = contextlib.nullcontext()


def range(name: str):  # noqa: A001 - mirrors torch.cuda.nvtx.range
    """A context manager: an NVTX range when enabled, else a shared no-op."""
    return _range(name) if ENABLED else _NULL
