"""A/B of the launch order of the two tensor-core replicas in a one-GPU
HetTMR round (which of TF32 / 3xBF16 gets the SIMT grid's last-wave holes
first), and of checkpoint copies on the copy engine vs the copy kernel.
Device-resident 4096^2 tasks through bench.TaskStreamBench, p = 0.05.

  python tools/tmr_order_ab.py [--steps 40]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
import paper_1405_2912_b200 as hf  # noqa: E402
from paper_1405_2912_b200 import executor as ex  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--variants", default="default,tc3-first")
ap.add_argument("--dmr", action="store_true", help="HetDMR (TC + SIMT) instead of HetTMR")
a = ap.parse_args()
args = argparse.Namespace(n=4096, fault_prob=0.05, seed=1, depth=1, warmup=3, trace_steps=False)

RANK = {"default": None, "tc3-first": {"mm_simt": 3, "mm_tc3x": 2, "mm_tc": 1},
        "tc-first": {"mm_simt": 3, "mm_tc": 2, "mm_tc3x": 1}}
orig = ex.Executor._expected_ns
for name in a.variants.split(",") * 2:
    r = RANK[name]
    ex.Executor._expected_ns = orig if r is None else (lambda self, task, sel, r=r: float(r[sel.kernel]))
    b = bench.TaskStreamBench(args, 0, 0, bench.DMR_KINDS if a.dmr else bench.TMR_KINDS,
                              hf.StrategyKind.HET_DMR if a.dmr else hf.StrategyKind.HET_TMR)
    b.warm()
    t, _ = b.timed(b.device_stream, a.steps, True)
    print(json.dumps({"variant": name, "tasks_per_s": a.steps / t, "ms_per_task": 1e3 * t / a.steps,
                      "votes": b.stats["votes"]}), flush=True)
    del b
