"""Checksum oracle (numpy).  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates the position-sensitive 64-bit checksum of
paper_1405_2912_b200/csrc/copy.cu (new; no reference counterpart — the
reference keeps host copies and never verifies them, memory.py:176-189).
"""

from __future__ import annotations

import numpy as np

M32 = np.uint64(0xFFFFFFFF)


def checksum(data) -> int:
    raw = np.frombuffer(bytes(data) if not isinstance(data, np.ndarray) else data.tobytes(),
                        dtype=np.uint8)
    nbytes = raw.size
    if nbytes == 0:
        return 0
    pad = (-nbytes) % 4
    if pad:
        raw = np.concatenate([raw, np.zeros(pad, dtype=np.uint8)])
    w = raw.view("<u4").astype(np.uint64)
    j = np.arange(w.size, dtype=np.uint64)
    with np.errstate(over="ignore"):
        lo = (j * np.uint64(0x9E3779B9)) & M32
        hi = ((j >> np.uint64(32)) * np.uint64(0x7F4A7C15)) & M32
        x = w ^ lo ^ hi
        x = (x * np.uint64(0x85EBCA6B)) & M32
        x ^= x >> np.uint64(13)
        x = (x * np.uint64(0xC2B2AE35)) & M32
        x ^= x >> np.uint64(16)
        s = int(x.sum(dtype=np.uint64))
    return (s ^ ((nbytes * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF
