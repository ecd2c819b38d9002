"""Where the host time of a voted task goes (C5 shape: HetTMR 2048^2 task
stream on one GPU).  Wraps the runtime's main entry points with
perf_counter accumulators (inclusive times, ~0.3 us per wrapped call) and
prints microseconds per task for each, plus the wall rate.

    python tools/host_breakdown.py [--tasks 2000] [--n 2048] [--strategy hettmr]
"""
import argparse
import collections
import functools
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1405_2912_b200 as hf  # noqa: E402
from paper_1405_2912_b200 import backend as hb, executor as hx, kernels as hk, mapping as hm, memory as hmem  # noqa: E402
from paper_1405_2912_b200 import voting as hv, devices as hd, api as ha  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tasks", type=int, default=2000)
ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--strategy", default="hettmr")
args = ap.parse_args()

ACC = collections.defaultdict(float)
CNT = collections.Counter()


def wrap(owner, name, label=None):
    fn = getattr(owner, name)
    label = label or f"{getattr(owner, '__name__', owner)}.{name}"

    @functools.wraps(fn)
    def w(*a, **k):
        t = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            ACC[label] += time.perf_counter() - t
            CNT[label] += 1
    setattr(owner, name, w)


for owner, names in [
    (hx.Executor, ["begin_task", "finish_flight", "_launch_round", "_prepare", "_launch", "_finish", "_vote_start",
                   "_vote_finish", "_settle", "_resolve_round", "_emit_attempt_for", "_account_round"]),
    (hm.Mapper, ["select", "replace_replica", "timeout_for"]),
    (hmem.MemoryManager, ["request", "commit_success", "release", "_maybe_checkpoint", "register_buffer"]),
    (hb.CudaBackend, ["alloc", "unit_stream", "follow_all", "join", "timer_start", "timer_stop", "vote_start",
                      "checkpoint", "typed_view"]),
    (hk, ["gemm_tc", "gemm_simt", "vote_async", "checkpoint", "fill", "copy", "inject_bitflip"]),
    (hd, ["execute_attempt"]),
    (ha.TaskStream, ["submit", "_settle_oldest"]),
    (ha.Runtime, ["register_device_data", "release", "_bind"]),
]:
    for nm in names:
        if hasattr(owner, nm):
            wrap(owner, nm)
# modules imported by name elsewhere
hx.execute_attempt = hd.execute_attempt

n, nn = args.n, args.n * args.n
kinds = ("gpu-tc", "gpu-simt", "gpu-tc3") if args.strategy == "hettmr" else ("gpu-tc", "gpu-simt")
cfg = hf.gpu_fleet_config(devices=(0,), kinds=kinds)
cfg["memory_spaces"].append({"id": "gpu0ckpt", "device": 0})
for i, u in enumerate(cfg["units"]):
    u.update({"corrupt_prob": 0.05, "abort_prob": 0.01, "corrupt_mode": "bitflip", "seed": 17 + 101 * i})
rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(checkpoint_space="gpu0ckpt", serial_replicas=True,
                                                     attempt_limit=64))
task = hf.get_workload("matmul").attach(rt, kinds=kinds)
strat = hf.Strategy(hf.StrategyKind.HET_TMR if args.strategy == "hettmr" else hf.StrategyKind.HET_DMR)
rt.reserve("gpu0mem", nn * 4, 32)
A = (torch.rand(nn, device="cuda") + 1).view(torch.uint8)
B = (torch.rand(nn, device="cuda") + 1).view(torch.uint8)
C0 = torch.zeros(nn * 4, dtype=torch.uint8, device="cuda")


def run(k):
    q = []
    with rt.task_stream(depth=1) as ts:
        for _ in range(k):
            ar = tuple(rt.register_device_data(x, nn, hf.ValueType.FLOAT32, m, "gpu0mem")
                       for x, m in ((A, "r"), (B, "r"), (C0, "w")))
            q.append((ts.submit(task, dict(zip("ABC", ar), n=n), strat), ar))
            while q and q[0][0].success:
                for x in q.pop(0)[1]:
                    rt.release(x)
    for _, ar in q:
        for x in ar:
            rt.release(x)


run(20)
torch.cuda.synchronize()
ACC.clear()
CNT.clear()
t0 = time.perf_counter()
run(args.tasks)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
rows = sorted(((v / args.tasks * 1e6, k, CNT[k] / args.tasks) for k, v in ACC.items()), reverse=True)
print(json.dumps({"tasks_per_s": args.tasks / wall, "wall_us_per_task": wall / args.tasks * 1e6}))
for us, k, c in rows:
    print(f"{us:9.1f} us/task  {c:6.2f} calls/task  {k}")
