"""GPU busy fraction of a C5-shaped task stream (HetTMR 2048^2, one GPU): the union of
kernel intervals in a torch.profiler trace over 300 tasks, per task, against the span."""
import sys, json, argparse, gzip
sys.path.insert(0, "/root/repo")
import torch, bench
import paper_1405_2912_b200 as hf
from torch.profiler import profile, ProfilerActivity
args = argparse.Namespace(n=2048, fault_prob=0.05, seed=1, depth=1, warmup=3, trace_steps=False)
b = bench.TaskStreamBench(args, 0, 0, bench.TMR_KINDS, hf.StrategyKind.HET_TMR)
b.warm()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    t, _ = b.timed(b.device_stream, 300, False)
prof.export_chrome_trace("/tmp/c5.json")
d = json.load(open("/tmp/c5.json"))
ev = sorted([e for e in d["traceEvents"] if e.get("ph") == "X" and e.get("cat") == "kernel"], key=lambda e: e["ts"])
# union of kernel intervals = GPU busy time
busy, cur_s, cur_e = 0.0, None, None
for e in ev:
    s, en = e["ts"], e["ts"] + e["dur"]
    if cur_e is None or s > cur_e:
        if cur_e is not None: busy += cur_e - cur_s
        cur_s, cur_e = s, en
    else:
        cur_e = max(cur_e, en)
busy += cur_e - cur_s
span = ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]
print(json.dumps({"tasks": 300, "wall_ms_per_task": t * 1e3 / 300, "gpu_busy_us_per_task": busy / 300,
                  "span_us_per_task": span / 300, "busy_frac": busy / span}))
