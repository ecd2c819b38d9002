"""Matmul oracle.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

No reference counterpart (the reference has no matmul workload; its bodies
are workloads.py:25-58).  The oracle accumulates in binary64 and rounds once
to float32; GPU variants are compared with it under the voter predicate.
"""

from __future__ import annotations

import numpy as np


def matmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    return (a.astype(np.float64) @ b.astype(np.float64)).astype(np.float32)


def make_inputs(n: int, seed: int):
    """U[1,2) operands — the reference's input distribution
    (workloads.py:70-72), drawn with PCG64 for speed at 2^24 elements."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(1.0, 2.0, size=(n, n)).astype(np.float32)
    b = rng.uniform(1.0, 2.0, size=(n, n)).astype(np.float32)
    return a, b
