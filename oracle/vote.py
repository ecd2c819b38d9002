"""K-replica vote oracle (numpy).  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Pair predicate: restates _compare_floats, /root/reference/pkg/src/hetrt/voting.py:68-81
(binary64: ok = (|a-b| <= δ·max(|a|,|b|)) & isfinite(|a-b|); ok |= a == b;
ok |= isnan(a) & isnan(b)) and the bitwise integer rule of voting.py:96-103.
Majority contract: SURVEY.md Appendix A (new; reduces to voting.py:106-123 at K = 2).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def _ordered(bits: np.ndarray, width: int) -> np.ndarray:
    """Sign-magnitude float bits -> ordered integers (as Python-int-safe object
    arithmetic avoided: int64 for f32, split handling for f64)."""
    if width == 4:
        i = bits.view(np.int32).astype(np.int64)
        return np.where(i >= 0, i, np.int64(-2147483648) - i)
    i = bits.view(np.int64)
    # INT64_MIN - i for negative i, computed with wraparound-free object math
    out = i.copy()
    neg = i < 0
    with np.errstate(over="ignore"):
        out[neg] = np.int64(-9223372036854775808) - i[neg]
    return out


def ulp_ok(a: np.ndarray, b: np.ndarray, ulp: int) -> np.ndarray:
    """Ordered-integer distance <= ulp, never across NaN (new rule)."""
    w = a.dtype.itemsize
    ua = a.view(np.uint32 if w == 4 else np.uint64)
    ub = b.view(np.uint32 if w == 4 else np.uint64)
    oa = _ordered(ua, w)
    ob = _ordered(ub, w)
    if w == 4:
        d = np.abs(oa - ob)
        ok = d <= ulp
    else:
        # |oa - ob| may exceed int64: compare in uint64 with the larger first
        hi = np.maximum(oa, ob).astype(np.uint64)
        lo = np.minimum(oa, ob).astype(np.uint64)
        with np.errstate(over="ignore"):
            d = hi - lo
        ok = d <= np.uint64(ulp)
    return ok & ~np.isnan(a) & ~np.isnan(b)


def pair_ok(a: np.ndarray, b: np.ndarray, delta: float, ulp=None) -> np.ndarray:
    """Element-wise agreement of two replicas (voting.py:68-81 / :96-103)."""
    if a.dtype.kind == "f":
        a64 = a.astype(np.float64)
        b64 = b.astype(np.float64)
        with np.errstate(invalid="ignore", over="ignore"):
            diff = np.abs(a64 - b64)
            ok = (diff <= delta * np.maximum(np.abs(a64), np.abs(b64))) & np.isfinite(diff)
            ok |= a64 == b64
            ok |= np.isnan(a64) & np.isnan(b64)
        if ulp is not None:
            ok |= ulp_ok(a, b, int(ulp))
        return ok
    return a == b


@dataclass
class OracleVote:
    verdict: str
    mismatch: list
    unresolved: int
    first_div: int
    winner: int
    voted: np.ndarray

    @property
    def faulty(self):
        return [r for r, m in enumerate(self.mismatch) if m > 0]


def vote(replicas, rel_tol=0.001, ulp_tol=None) -> OracleVote:
    """SURVEY.md Appendix A over numpy replicas of one dtype.

    replicas: K arrays (any shape; flattened).  rel_tol / ulp_tol: scalar or
    per-replica sequences; a pair uses the max of its two tolerances.
    """
    xs = [np.ascontiguousarray(r).reshape(-1) for r in replicas]
    K = len(xs)
    n = xs[0].size
    rel = [float(rel_tol)] * K if np.isscalar(rel_tol) else [float(x) for x in rel_tol]
    if ulp_tol is None:
        ulp = None
    else:
        ulp = [int(ulp_tol)] * K if np.isscalar(ulp_tol) else [int(x) for x in ulp_tol]
    agree = np.zeros((K, K, n), dtype=bool)
    for r in range(K):
        agree[r, r] = True
        for s in range(r + 1, K):
            u = None if ulp is None else max(ulp[r], ulp[s])
            ok = pair_ok(xs[r], xs[s], max(rel[r], rel[s]), u)
            agree[r, s] = ok
            agree[s, r] = ok
    counts = agree.sum(axis=1)                    # includes self
    majority = 2 * counts > K                     # 2*(agree_r + 1) > K
    has = majority.any(axis=0)
    v = np.where(has, np.argmax(majority, axis=0), 0)   # lowest majority replica
    idx = np.arange(n)
    voted = np.empty_like(xs[0])
    stacked = np.stack(xs)
    voted[:] = stacked[v, idx]
    mism = []
    bad_any = ~has
    for r in range(K):
        dis = ~has | ~agree[r, v, idx]
        mism.append(int(dis.sum()))
        bad_any = bad_any | dis
    bad = np.flatnonzero(bad_any)
    first = int(bad[0]) if bad.size else -1
    unres = int((~has).sum())
    winner = int(np.argmin(mism))                 # ties -> lowest index
    if unres > 0:
        verdict = "mismatch"
    elif any(m > 0 for m in mism):
        verdict = "corrected"
    else:
        verdict = "match"
    return OracleVote(verdict, mism, unres, first, winner, voted)


def vote_bytes(replicas, elem_width: int) -> OracleVote:
    """Integer areas of arbitrary width: elements agree iff all bytes agree."""
    xs = [np.frombuffer(np.ascontiguousarray(r).tobytes(), dtype=np.uint8).reshape(-1, elem_width)
          for r in replicas]
    K = len(xs)
    n = xs[0].shape[0]
    agree = np.zeros((K, K, n), dtype=bool)
    for r in range(K):
        agree[r, r] = True
        for s in range(r + 1, K):
            ok = np.all(xs[r] == xs[s], axis=1)
            agree[r, s] = ok
            agree[s, r] = ok
    counts = agree.sum(axis=1)
    majority = 2 * counts > K
    has = majority.any(axis=0)
    v = np.where(has, np.argmax(majority, axis=0), 0)
    idx = np.arange(n)
    voted = np.stack(xs)[v, idx].reshape(-1)
    mism = []
    bad_any = ~has
    for r in range(K):
        dis = ~has | ~agree[r, v, idx]
        mism.append(int(dis.sum()))
        bad_any |= dis
    bad = np.flatnonzero(bad_any)
    unres = int((~has).sum())
    verdict = "mismatch" if unres else ("corrected" if any(mism) else "match")
    return OracleVote(verdict, mism, unres, int(bad[0]) if bad.size else -1,
                      int(np.argmin(mism)), voted)


def reference_first_divergence(a: np.ndarray, b: np.ndarray, delta: float):
    """K = 2 restatement of compare_payloads' float branch (voting.py:84-95):
    the index of the first non-agreeing element or None."""
    bad = np.flatnonzero(~pair_ok(a, b, delta))
    return int(bad[0]) if bad.size else None
