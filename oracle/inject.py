"""Fault-injection oracle.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""

from __future__ import annotations

import numpy as np


def corrupt_scale(view: np.ndarray, idx: int, rel: float) -> None:
    """In-place restatement of _corrupt_buffer's value rule,
    /root/reference/pkg/src/hetrt/devices.py:215-219: floats -> x*(1+rel)
    evaluated in binary64 then stored with round-to-nearest (rel if x == 0);
    integers XOR 0x01."""
    if view.dtype.kind == "f":
        x = float(view[idx])
        view[idx] = x * (1.0 + rel) if x != 0.0 else rel
    else:
        view[idx] = view[idx] ^ view.dtype.type(1)


def bitflip(view: np.ndarray, idx: int, bit: int) -> None:
    """In-place XOR of bit `bit` (0 = LSB) of element idx (new fault mode)."""
    raw = view.reshape(-1).view(np.uint8)
    w = view.dtype.itemsize
    raw[idx * w + bit // 8] ^= np.uint8(1 << (bit % 8))


def scribble(view: np.ndarray, data: bytes) -> None:
    """devices.py:241-246: the first min(8, nbytes) bytes are overwritten."""
    raw = view.reshape(-1).view(np.uint8)
    n = min(8, raw.size, len(data))
    raw[:n] = np.frombuffer(bytes(data[:n]), dtype=np.uint8)
