"""The oracle is pinned against fixtures produced by the reference itself
(tests/golden/make_golden.py) before it is trusted as a checker."""

import random

import numpy as np
import pytest

from golden_io import as_array, inject_golden, voter_cases
from oracle import fault_schedule, vote as ovote


CASES = voter_cases()


@pytest.mark.parametrize("case", CASES, ids=[f"{c['vt']}{c['width']}-{i}" for i, c in enumerate(CASES)])
def test_k2_oracle_matches_reference_compare(case):
    a = as_array(case["a"], case["vt"], case["width"])
    b = as_array(case["b"], case["vt"], case["width"])
    if case["vt"] == "int" and case["width"] not in (1, 2, 4, 8):
        res = ovote.vote_bytes([a, b], case["width"])
    elif case["vt"] == "int":
        res = ovote.vote([a, b], 0.0)
    else:
        res = ovote.vote([a, b], case["delta"])
    expect_match = case["verdict"] == "match"
    assert (res.verdict == "match") == expect_match
    assert res.first_div == case["first_div"]
    # K = 2: every disagreeing element is unresolved and counted on both sides
    assert res.mismatch[0] == res.mismatch[1] == res.unresolved


def test_golden_set_covers_both_verdicts():
    v = [c["verdict"] for c in CASES]
    assert v.count("match") > 10 and v.count("mismatch") > 10


_DT = {"f32": np.float32, "f64": np.float64, "u8": np.uint8, "u16": np.uint16,
       "u32": np.uint32, "u64": np.uint64}


@pytest.mark.parametrize("row", inject_golden()["attempts"])
def test_fault_schedule_oracle_replays_reference(row):
    dt = _DT[row["kind"]]
    views = [np.frombuffer(bytes.fromhex(h), dtype=dt).copy() for h in row["before"]]
    rng = random.Random(row["seed"])
    ev = fault_schedule.apply_attempt(rng, row["probs"], views,
                                      [row["kind"] in ("f32", "f64")] * len(views),
                                      rel=row["rel"], element=row["element"])
    assert ev["fault"] == row["fault"]
    if row["corrupted_index"] is not None:
        assert ev["corrupt"][1] == row["corrupted_index"]
    assert [v.tobytes().hex() for v in views] == row["after"]


@pytest.mark.parametrize("seq", inject_golden()["sequences"])
def test_fault_class_sequence_matches_reference(seq):
    rng = random.Random(seq["seed"])
    buf = np.ones(4, dtype=np.float32)
    got = []
    for _ in range(len(seq["faults"])):
        ev = fault_schedule.apply_attempt(rng, seq["probs"], [buf], [True])
        got.append(ev["fault"])
    assert got == seq["faults"]
    assert buf.tobytes().hex() == seq["final"]


def test_tmr_single_fault_corrected():
    rng = np.random.default_rng(1)
    x = rng.uniform(1, 2, 1000).astype(np.float32)
    bad = x.copy()
    bad[17] *= np.float32(1.5)
    res = ovote.vote([x, bad, x.copy()], 1e-3)
    assert res.verdict == "corrected"
    assert res.mismatch == [0, 1, 0]
    assert res.first_div == 17 and res.winner == 0
    assert np.array_equal(res.voted, x)


@pytest.mark.parametrize("row", inject_golden()["attempts"])
def test_simulate_execution_replays_reference(row):
    """The drop-in's simulate_execution (reference devices.py:223-259 API over
    host numpy views) reproduces the reference's recorded outcomes: fault
    class, corrupted element and the bytes of every write view."""
    import paper_1405_2912_b200 as hf
    dt = _DT[row["kind"]]
    vt = hf.ValueType.FLOAT32 if row["kind"] == "f32" else hf.ValueType.FLOAT64 if row["kind"] == "f64" \
        else hf.ValueType.INT
    views = [np.frombuffer(bytes.fromhex(h), dtype=dt).copy() for h in row["before"]]
    unit = {"id": "u", "kind": "cpu", "memory_space": "host", "seed": row["seed"],
            "corrupt_rel_magnitude": row["rel"], "corrupt_element": row["element"]}
    unit.update(dict(zip(("abort_prob", "api_error_prob", "hang_prob", "corrupt_prob"), row["probs"])))
    fleet = hf.load_fleet({"memory_spaces": [{"id": "host", "host": True}], "units": [unit]})
    out = hf.simulate_execution(fleet.units["u"], "k", "cpu", views[0].size, write_views=[(v, vt) for v in views])
    assert (out.fault.value if out.fault is not None else None) == row["fault"]
    if row["corrupted_index"] is not None:
        assert out.corrupted_index == row["corrupted_index"]
    assert [v.tobytes().hex() for v in views] == row["after"]
