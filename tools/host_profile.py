"""cProfile of the host path of a voted-task stream (C5 shape: HetTMR 2048^2
on one GPU, device-resident inputs, TaskStream depth 1): the top functions by
own time, microseconds per task.

    python tools/host_profile.py [--tasks 1500] [--n 2048]
"""
import argparse
import cProfile
import pstats
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_1405_2912_b200 as hf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tasks", type=int, default=1500)
ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--top", type=int, default=45)
a = ap.parse_args()
args = argparse.Namespace(n=a.n, fault_prob=0.05, seed=1, depth=1, warmup=3, trace_steps=False)
b = bench.TaskStreamBench(args, 0, 0, bench.TMR_KINDS, hf.StrategyKind.HET_TMR)
b.warm()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
b.device_stream(a.tasks, False)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
rows = sorted(st.stats.items(), key=lambda kv: -kv[1][2])[:a.top]
print(f"{'own us/task':>12} {'cum us/task':>12} {'calls/task':>10}  function")
for (fn, line, name), (cc, nc, tt, ct, _) in rows:
    print(f"{1e6 * tt / a.tasks:12.1f} {1e6 * ct / a.tasks:12.1f} {nc / a.tasks:10.2f}  {Path(fn).name}:{line} {name}")
