"""Generate experiment-harness golden fixtures by running the REFERENCE.

Run here (the reference is importable in this container, not on the GPU box):
    python tests/golden/make_experiment_golden.py
For each spec below it runs hetrt.experiments.run_experiment strategy by
strategy (a strategy the reference cannot finish — e.g. HetDMR dead ends,
SURVEY.md §4.3 — is recorded as the exception name instead) and stores the
CSV rows plus the attempt/done trace.  The modelled fleets make every number
deterministic, so tests/test_experiments.py requires our harness to print
the same CSV rows and ATT/DONE trace lines byte for byte.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True  # /root/reference is read-only
sys.path.insert(0, "/root/reference/pkg/src")

from hetrt.experiments import CSV_HEADER, ExperimentSpec, run_experiment  # noqa: E402

OUT = Path(__file__).resolve().parent / "experiment_golden.json"

ALL = ["perfcp", "perfcp-fault-aware", "dmr", "hetdmr", "perfcp-avoidance", "perfcp-pinned"]

SPECS = [
    dict(workload="inc", fleet="default", strategies=ALL,
         sweep_var="gpu1.abort_prob", sweep_values=[0.0, 0.2, 0.5, 0.9], repetitions=6, seed=3, size=64),
    dict(workload="inc", fleet="default", strategies=ALL,
         sweep_var="gpu1.corrupt_prob", sweep_values=[0.1, 0.4, 0.8], repetitions=6, seed=4, size=48),
    dict(workload="inc", fleet="default", strategies=ALL,
         sweep_var="cpu0.api_error_prob", sweep_values=[0.0, 0.5], repetitions=5, seed=9, size=40),
    dict(workload="pathfinder-like", fleet="pathfinder", strategies=ALL,
         sweep_var="gpu1.corrupt_prob", sweep_values=[0.0, 0.3, 0.6], repetitions=6, seed=5, size=128),
    dict(workload="pathfinder-like", fleet="pathfinder", strategies=ALL,
         sweep_var="cpu0.hang_prob", sweep_values=[0.0, 0.25, 0.5], repetitions=6, seed=6, size=96),
    dict(workload="buggy-inc", fleet="default", strategies=ALL,
         sweep_var="size", sweep_values=[16, 64, 256], repetitions=4, seed=7),
    dict(workload="inc", fleet="default", strategies=ALL,
         sweep_var="gpu2.hang_prob", sweep_values=[0.0, 0.3, 0.7], repetitions=8, seed=11, size=32,
         timeout_factor=2.0, check_interval=3),
    dict(workload="inc", fleet="default", strategies=ALL,
         sweep_var="none", sweep_values=[0.0], repetitions=12, seed=12, size=20, attempt_limit=4),
]


def main() -> None:
    cases = []
    for spec in SPECS:
        for strategy in spec["strategies"]:
            s = dict(spec, strategies=[strategy])
            trace = "/tmp/_exp_golden_trace.txt"
            try:
                rows = run_experiment(ExperimentSpec(**s, trace=trace))
                csv = [r.csv_row() for r in rows]
                lines = Path(trace).read_text(encoding="utf-8").splitlines()
                err = None
            except Exception as exc:  # noqa: BLE001 - the reference's own failure is the fixture
                csv, lines, err = [], [], type(exc).__name__
            cases.append({"spec": s, "csv": csv, "trace": lines, "error": err,
                          "oracle_mismatches": [r.oracle_mismatches for r in rows] if err is None else []})
    OUT.write_text(json.dumps({"header": CSV_HEADER, "cases": cases}, indent=0), encoding="utf-8")
    ok = sum(c["error"] is None for c in cases)
    print(f"wrote {OUT} ({ok}/{len(cases)} strategy runs finished in the reference)")


if __name__ == "__main__":
    main()
