"""Generate golden fixtures by running the REFERENCE implementation.

Run here (the reference is importable in this container, not on the GPU box):
    python tests/golden/make_golden.py
It imports hetrt from /root/reference/pkg/src and records, for seeded inputs,
what the reference itself returns:
  voter_golden.npz   — voting.compare verdicts + first divergence indices
                       (K = 2) on f32/f64/int payloads incl. NaN/inf/±0/
                       subnormal/boundary cases and the test_voter.py vectors
  inject_golden.json — simulate_execution outcomes: fault classes, corrupted
                       indices and the corrupted/scribbled payload bytes
The committed fixtures are what tests/ compare the oracle and the GPU with.
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True  # /root/reference is read-only

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from hetrt import (CorruptionSpec, FaultModel, ProcessingUnit, SpeedProfile,  # noqa: E402
                   ValueType, VoterConfig, compare, simulate_execution)

OUT = Path(__file__).resolve().parent


def _special_f32(rng, n):
    pool = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, -1e-45, 1.17549435e-38,
                     3.4028235e38, -3.4028235e38, 1.0, -1.0, 2.0 ** -149 * 3], dtype=np.float32)
    return pool[rng.integers(0, pool.size, n)]


def _boundary_pair(rng, n, delta, dtype):
    """b near a*(1±δ): walks a few ulps either side of the acceptance edge."""
    a = rng.uniform(-1e3, 1e3, n).astype(dtype)
    sign = rng.choice([-1.0, 1.0], n)
    target = a.astype(np.float64) * (1.0 + sign * delta)
    b = target.astype(dtype)
    steps = rng.integers(-6, 7, n)
    for i in range(n):
        for _ in range(abs(int(steps[i]))):
            b[i] = np.nextafter(b[i], dtype(np.inf) if steps[i] > 0 else dtype(-np.inf))
    return a, b


def voter_cases():
    rng = np.random.default_rng(20260117)
    cases = []  # (dtype_code, width, delta, a_bytes, b_bytes)

    def add(a, b, delta, vt="f32", width=None):
        a = np.asarray(a)
        b = np.asarray(b)
        cases.append((vt, width or a.dtype.itemsize, float(delta), a.tobytes(), b.tobytes()))

    f = np.float32
    # test_voter.py:35-70, :211-216 vectors
    add(f([1.0, 2.0]), f([1.0, 2.0]), 1e-3)
    add(f([1.0]), f([1.0005]), 1e-3)
    add(f([1.0]), f([1.002]), 1e-3)
    add(f([0.0]), f([-0.0]), 1e-3)
    add(f([np.nan]), f([np.nan]), 1e-3)
    add(f([np.nan]), f([1.0]), 1e-3)
    add(f([np.inf]), f([np.inf]), 1e-3)
    add(f([np.inf]), f([-np.inf]), 1e-3)
    add(f([1.0, np.nan, 3.0]), f([1.0, np.nan, 3.0]), 0.0)
    add(np.float64([1.0, 2.0]), np.float64([1.0, 2.0000001]), 1e-3, "f64")
    add(np.float64([1.0, 2.0]), np.float64([1.0, 2.0000001]), 1e-9, "f64")
    add(np.frombuffer(bytes([1, 2, 3, 4]), np.uint8), np.frombuffer(bytes([1, 2, 7, 4]), np.uint8),
        0.0, "int", 2)
    # random f32 with specials, various deltas
    for delta in (0.0, 1e-7, 1e-3, 0.5, 2.0):
        for n in (1, 3, 17, 1000, 4099):
            a = rng.uniform(-100, 100, n).astype(f)
            b = (a * (1 + rng.uniform(-3 * max(delta, 1e-7), 3 * max(delta, 1e-7), n))).astype(f)
            m = rng.random(n) < 0.1
            a[m] = _special_f32(rng, int(m.sum()))
            m2 = rng.random(n) < 0.1
            b[m2] = _special_f32(rng, int(m2.sum()))
            add(a, b, delta)
            add(a, a.copy(), delta)
    # exact-boundary sweeps
    for delta in (1e-3, 1e-5, 0.1, 1.0):
        for dt, code in ((np.float32, "f32"), (np.float64, "f64")):
            a, b = _boundary_pair(rng, 2000, delta, dt)
            add(a, b, delta, code)
            # single mismatching element at a random position among agreeing ones
            n = 3000
            a = rng.uniform(1, 2, n).astype(dt)
            b = a.copy()
            k = int(rng.integers(0, n))
            b[k] = dt(float(a[k]) * (1 + 3 * delta))
            add(a, b, delta, code)
    # subnormal-only and huge-magnitude sets
    a = (rng.integers(1, 2 ** 23, 3000).astype(np.uint32)).view(np.float32)
    b = (rng.integers(1, 2 ** 23, 3000).astype(np.uint32)).view(np.float32)
    add(a, b, 0.5)
    add(a, b, 1e-3)
    a = rng.uniform(1e37, 3e38, 3000).astype(f) * rng.choice([-1, 1], 3000).astype(f)
    b = rng.uniform(1e37, 3e38, 3000).astype(f) * rng.choice([-1, 1], 3000).astype(f)
    add(a, b, 1.5)
    add(a, b, 3.0)
    # f64 with specials
    for delta in (0.0, 1e-3, 1e-12):
        a = rng.uniform(-1e6, 1e6, 2000)
        b = a * (1 + rng.uniform(-2 * max(delta, 1e-13), 2 * max(delta, 1e-13), 2000))
        sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 1.7e308, -1.7e308])
        m = rng.random(2000) < 0.1
        a[m] = sp[rng.integers(0, sp.size, int(m.sum()))]
        m = rng.random(2000) < 0.1
        b[m] = sp[rng.integers(0, sp.size, int(m.sum()))]
        add(a, b, delta, "f64")
    # integer widths
    for width in (1, 2, 3, 4, 8, 12):
        for n in (1, 5, 1000):
            a = rng.integers(0, 256, n * width, dtype=np.uint8)
            b = a.copy()
            if n > 1:
                pos = rng.integers(0, n * width, max(1, n // 100))
                b[pos] ^= 0x10
            add(a, b, 0.0, "int", width)
            add(a, a.copy(), 0.0, "int", width)
    return cases


def build_voter_golden():
    cfg_cache = {}
    vts = {"f32": ValueType.FLOAT32, "f64": ValueType.FLOAT64, "int": ValueType.INT}
    cases = voter_cases()
    rows = []
    for vt, width, delta, a, b in cases:
        cfg = cfg_cache.setdefault(delta, VoterConfig(float_delta=delta))
        out = compare({"out": (a, vts[vt], width)}, {"out": (b, vts[vt], width)}, cfg)
        idx = -1 if out.first_divergence is None else int(out.first_divergence[1])
        rows.append((vt, width, delta, a, b, out.verdict, idx))
    # pack into an npz: concatenated payload blobs + offsets
    blob_a = b"".join(r[3] for r in rows)
    blob_b = b"".join(r[4] for r in rows)
    lens = np.array([len(r[3]) for r in rows], dtype=np.int64)
    np.savez_compressed(
        OUT / "voter_golden.npz",
        vt=np.array([r[0] for r in rows]),
        width=np.array([r[1] for r in rows], dtype=np.int64),
        delta=np.array([r[2] for r in rows], dtype=np.float64),
        lens=lens,
        blob_a=np.frombuffer(blob_a, dtype=np.uint8),
        blob_b=np.frombuffer(blob_b, dtype=np.uint8),
        verdict=np.array([r[5] for r in rows]),
        first_div=np.array([r[6] for r in rows], dtype=np.int64),
    )
    return len(rows)


def build_inject_golden():
    rows = []

    def unit(seed, **kw):
        spec = kw.pop("corruption", CorruptionSpec())
        return ProcessingUnit("u0", "cpu", "host", SpeedProfile(base_latency_ns=1000),
                              FaultModel(rng_seed=seed, corruption=spec, **kw))

    rng = np.random.default_rng(7)
    # corruption of float32/float64/int views, random and targeted elements
    for seed in range(12):
        for kind in ("f32", "f64", "u8", "u16", "u32", "u64"):
            n = int(rng.integers(1, 50))
            rel = float(rng.choice([0.01, 0.5, -0.3, 1e-4]))
            elem = None if seed % 3 else int(rng.integers(0, 2 * n))
            u = unit(seed, corrupt_prob=1.0,
                     corruption=CorruptionSpec(relative_magnitude=rel, element=elem))
            if kind in ("f32", "f64"):
                dt = np.float32 if kind == "f32" else np.float64
                bufs = [rng.uniform(-5, 5, n).astype(dt), rng.uniform(-5, 5, n + 3).astype(dt)]
                bufs[0][rng.integers(0, n)] = 0.0
                vt = ValueType.FLOAT32 if kind == "f32" else ValueType.FLOAT64
            else:
                dt = {"u8": np.uint8, "u16": np.uint16, "u32": np.uint32, "u64": np.uint64}[kind]
                bufs = [rng.integers(0, 200, n).astype(dt), rng.integers(0, 200, n + 3).astype(dt)]
                vt = ValueType.INT
            before = [b.tobytes().hex() for b in bufs]
            out = simulate_execution(u, "k", "cpu", n, write_views=[(b, vt) for b in bufs])
            rows.append({"kind": kind, "seed": seed, "rel": rel, "element": elem,
                         "probs": [0, 0, 0, 1.0], "before": before,
                         "after": [b.tobytes().hex() for b in bufs],
                         "fault": out.fault.value if out.fault else None,
                         "corrupted_index": out.corrupted_index})
    # scribbles on abort / api_error
    for seed in range(10):
        for kind in ("f32", "u32", "u8"):
            n = int(rng.integers(1, 20))
            dt = {"f32": np.float32, "u32": np.uint32, "u8": np.uint8}[kind]
            bufs = [np.zeros(n, dtype=dt), np.zeros(3, dtype=dt)]
            vt = ValueType.FLOAT32 if kind == "f32" else ValueType.INT
            u = unit(100 + seed, abort_prob=0.5, api_error_prob=0.5)
            before = [b.tobytes().hex() for b in bufs]
            out = simulate_execution(u, "k", "cpu", n, write_views=[(b, vt) for b in bufs])
            rows.append({"kind": kind, "seed": 100 + seed, "rel": 0.01, "element": None,
                         "probs": [0.5, 0.5, 0, 0], "before": before,
                         "after": [b.tobytes().hex() for b in bufs],
                         "fault": out.fault.value if out.fault else None,
                         "corrupted_index": out.corrupted_index})
    # long categorical sequences
    seqs = []
    for seed in (0, 1, 7, 42, 12345):
        probs = [0.1, 0.05, 0.05, 0.1]
        u = unit(seed, abort_prob=probs[0], api_error_prob=probs[1], hang_prob=probs[2],
                 corrupt_prob=probs[3])
        buf = np.ones(4, dtype=np.float32)
        seq = []
        for _ in range(400):
            out = simulate_execution(u, "k", "cpu", 4, write_views=[(buf, ValueType.FLOAT32)])
            seq.append(out.fault.value if out.fault else None)
        seqs.append({"seed": seed, "probs": probs, "faults": seq, "final": buf.tobytes().hex()})
    (OUT / "inject_golden.json").write_text(json.dumps({"attempts": rows, "sequences": seqs}))
    return len(rows), len(seqs)


if __name__ == "__main__":
    print("voter cases:", build_voter_golden())
    print("inject rows/seqs:", build_inject_golden())
