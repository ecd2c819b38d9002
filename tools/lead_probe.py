"""Which replica leads a HetTMR round (highest mean measured runtime -> the
LEAD_PRIORITY stream; with attach_kernel costs, as the matmul workload now
declares, the measured order is not consulted), and tasks/s, over a
bench-shaped device stream.
  HETFT_VOTE_STREAM=0|1 python tools/lead_probe.py [tasks]"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1405_2912_b200 import executor as ex  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
depth = sys.argv[sys.argv.index("--depth") + 1] if "--depth" in sys.argv else "1"
dmr = "--dmr" in sys.argv
sys.argv = [sys.argv[0], "--steps", str(steps), "--depth", depth]
args = bench.parse()
hf, rt, task = bench.build_runtime(0, 0.05, 1, kinds=bench.DMR_KINDS if dmr else bench.TMR_KINDS)
leads = []
orig = ex.Executor._expected_ns


def spy(self, t, sel):
    v = orig(self, t, sel)
    leads.append((sel.kernel, v))
    return v


ex.Executor._expected_ns = spy
tb = bench.TaskStreamBench(args, 0, 0, bench.DMR_KINDS if dmr else bench.TMR_KINDS,
                           hf.Strategy(hf.StrategyKind.HET_DMR if dmr else hf.StrategyKind.HET_TMR),
                           built=(hf, rt, task))
tb.warm()
leads.clear()
dt, _ = tb.timed(tb.device_stream, steps, True)
rounds = [leads[i:i + 3] for i in range(0, len(leads), 3)]
lead_k = {}
for r in rounds:
    k = max(r, key=lambda x: x[1])[0]
    lead_k[k] = lead_k.get(k, 0) + 1
print(json.dumps({"strategy": "dmr" if dmr else "tmr", "vote_stream": os.environ.get("HETFT_VOTE_STREAM", "1"), "tasks_per_s": steps / dt,
                  "ms_per_task": dt / steps * 1e3, "leads": lead_k,
                  "last_expected_ms": {k: v / 1e6 for k, v in rounds[-1]} if rounds else None}))
