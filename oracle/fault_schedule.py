"""Fault-schedule oracle.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates the per-attempt RNG draw order of the reference device model
(/root/reference/pkg/src/hetrt/devices.py:140-160 reset_rng/draw_fault and
:223-258 simulate_execution) on an MT19937
`random.Random(seed)` per unit, and applies the drawn fault to numpy views
the way the reference does.  The GPU path draws the same schedule on the host
and applies it with the hf_inject_* / hf_scribble kernels.
"""

from __future__ import annotations

import random
from typing import Optional, Sequence

import numpy as np

from . import inject


def draw_class(rng: random.Random, abort: float, api: float, hang: float, corrupt: float) -> Optional[str]:
    """devices.py:144-160: one uniform draw over cumulative edges."""
    r = rng.random()
    edge = abort
    if r < edge:
        return "abort"
    edge += api
    if r < edge:
        return "api_error"
    edge += hang
    if r < edge:
        return "hang"
    edge += corrupt
    if r < edge:
        return "corrupt"
    return None


def _int_view_len(nbytes: int, width: int) -> int:
    # executor._payload_view: INT areas of width 1/2/4/8 use a typed view,
    # other widths a uint8 view (executor.py:100-106)
    return nbytes // width if width in (1, 2, 4, 8) else nbytes


def apply_attempt(rng: random.Random, probs: Sequence[float], views: list, is_float: list,
                  rel: float = 0.01, element: Optional[int] = None, mode: str = "scale",
                  body=None) -> dict:
    """One attempt: draw (and apply to `views`, numpy arrays) in reference order.

    views are the write views in handle order (typed views for INT areas, as
    executor._payload_view builds them).  Returns the event record.
    """
    fault = draw_class(rng, *probs)
    ev = {"fault": fault, "scribble": [], "corrupt": None}
    if fault == "hang":
        return ev
    if fault in ("abort", "api_error"):
        for vi, v in enumerate(views):
            raw = v.view(np.uint8) if is_float[vi] else v
            n = min(8, raw.size)
            if n:
                vals = [rng.randrange(256) for _ in range(n)]
                raw[:n] = vals
                ev["scribble"].append((vi, vals))
        return ev
    if body is not None:
        body()
    if fault == "corrupt" and views:
        which = rng.randrange(len(views))
        v = views[which]
        n = v.size
        if n == 0:
            ev["corrupt"] = (which, -1, None)
            return ev
        idx = element if element is not None else rng.randrange(n)
        idx = min(idx, n - 1)
        if mode == "bitflip":
            bit = rng.randrange(8 * v.dtype.itemsize)
            inject.bitflip(v, idx, bit)
            ev["corrupt"] = (which, idx, bit)
        else:
            inject.corrupt_scale(v, idx, rel)
            ev["corrupt"] = (which, idx, rel)
    return ev
