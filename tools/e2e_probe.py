"""Per-step wall times of bench.py's e2e loop (host buffers through the public
API), with the popped task's rounds, to find pipeline stalls.

  python tools/e2e_probe.py [--steps 60] [--p 0.05] [--nogc] [--depth 1]
"""
import argparse
import gc
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=60)
ap.add_argument("--p", type=float, default=0.05)
ap.add_argument("--depth", type=int, default=1)
ap.add_argument("--nogc", action="store_true")
ap.add_argument("--noreserve", action="store_true")
ap.add_argument("--lookahead", type=int, default=2)
ap.add_argument("--tmr", action="store_true", help="HetTMR (tc, simt, tc3) instead of bench.py's HetDMR")
ap.add_argument("--device", action="store_true", help="device-resident inputs (bench.py's `value` loop)")
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--kineto", default=None, help="write a torch.profiler chrome trace of the timed run here")
args = ap.parse_args()

if args.tmr:
    import paper_1405_2912_b200 as hf
    kinds = ("gpu-tc", "gpu-simt", "gpu-tc3")
    cfg = hf.gpu_fleet_config(devices=(0,), kinds=kinds)
    cfg["memory_spaces"].append({"id": "gpu0ckpt", "device": 0})
    for i, u in enumerate(cfg["units"]):
        u.update({"corrupt_prob": args.p, "corrupt_mode": "bitflip", "seed": 1_000_003 + i * 101 + 31})
    rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(checkpoint_space="gpu0ckpt", serial_replicas=True,
                                                         attempt_limit=64))
    task = hf.get_workload("matmul").attach(rt, kinds=kinds)
else:
    hf, rt, task = bench.build_runtime(0, args.p, 1, kinds=bench.DMR_KINDS)
n = args.n
nb = n * n * 4
space = "gpu0mem"
hA = (torch.rand(n * n) + 1).view(torch.uint8).pin_memory()
hB = (torch.rand(n * n) + 1).view(torch.uint8).pin_memory()
hC = torch.empty(nb, dtype=torch.uint8).pin_memory()
hZ = torch.zeros(nb, dtype=torch.uint8).pin_memory()
strat = hf.Strategy(hf.StrategyKind.HET_TMR if args.tmr else hf.StrategyKind.HET_DMR)
if not args.__dict__.get("noreserve"):
    rt.reserve(space, nb, 24)


def stage():
    ia = rt.register_host_buffer(hA, n * n, hf.ValueType.FLOAT32, "r")
    ib = rt.register_host_buffer(hB, n * n, hf.ValueType.FLOAT32, "r")
    ic = rt.register_host_buffer(hZ, n * n, hf.ValueType.FLOAT32, "w")
    rt.prefetch(ia, space)
    rt.prefetch(ib, space)
    return ia, ib, ic


dA = (torch.rand(n * n, device="cuda") + 1).view(torch.uint8)
dB = (torch.rand(n * n, device="cuda") + 1).view(torch.uint8)
dC = torch.zeros(nb, dtype=torch.uint8, device="cuda")


def run_device(steps, log):
    queue = []
    t_prev = time.perf_counter()
    with rt.task_stream(depth=args.depth) as ts:
        for i in range(steps):
            t0 = time.perf_counter()
            ia = rt.register_device_data(dA, n * n, hf.ValueType.FLOAT32, "r", space)
            ib = rt.register_device_data(dB, n * n, hf.ValueType.FLOAT32, "r", space)
            ic = rt.register_device_data(dC, n * n, hf.ValueType.FLOAT32, "w", space)
            t1 = time.perf_counter()
            queue.append((ts.submit(task, {"A": ia, "B": ib, "C": ic, "n": n}, strat), (ia, ib, ic)))
            t2 = time.perf_counter()
            popped = []
            while queue and queue[0][0].success:
                rep, areas = queue.pop(0)
                popped.append(rep.rounds)
                for x in areas:
                    rt.release(x)
            t3 = time.perf_counter()
            log.append({"i": i, "stage_ms": (t1 - t0) * 1e3, "submit_ms": (t2 - t1) * 1e3,
                        "pop_ms": (t3 - t2) * 1e3, "step_ms": (t3 - t_prev) * 1e3, "popped_rounds": popped})
            t_prev = t3
    for rep, areas in queue:
        for x in areas:
            rt.release(x)


def run(steps, log):
    if args.device:
        return run_device(steps, log)
    staged = [stage() for _ in range(min(args.lookahead, steps))]
    queue, retired, last = [], [], None
    t_prev = time.perf_counter()
    with rt.task_stream(depth=args.depth) as ts:
        for i in range(steps):
            ia, ib, ic = staged.pop(0)
            t0 = time.perf_counter()
            if i + args.lookahead < steps:
                staged.append(stage())
            t1 = time.perf_counter()
            queue.append((ts.submit(task, {"A": ia, "B": ib, "C": ic, "n": n}, strat), (ia, ib, ic)))
            t2 = time.perf_counter()
            popped = []
            while queue and queue[0][0].success:
                rep, areas = queue.pop(0)
                popped.append(rep.rounds)
                last = rt.read_into_async(areas[2], hC)
                for x in retired:
                    rt.release(x)
                retired = list(areas)
            t3 = time.perf_counter()
            log.append({"i": i, "stage_ms": (t1 - t0) * 1e3, "submit_ms": (t2 - t1) * 1e3,
                        "pop_ms": (t3 - t2) * 1e3, "step_ms": (t3 - t_prev) * 1e3, "popped_rounds": popped})
            t_prev = t3
    for rep, areas in queue:
        last = rt.read_into_async(areas[2], hC)
        retired += list(areas)
    if last is not None:
        last.synchronize()
    for x in retired:
        rt.release(x)


run(3, [])
torch.cuda.synchronize()
if args.nogc:
    gc.collect()
    gc.disable()
log = []
seg0 = torch.cuda.memory_stats().get("segment.all.allocated", 0)
if args.profile:
    import cProfile
    import pstats
    prof = cProfile.Profile()
    prof.enable()
kin = None
if args.kineto:
    from torch.profiler import ProfilerActivity, profile
    kin = profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA])
    kin.__enter__()
t0 = time.perf_counter()
run(args.steps, log)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
if kin is not None:
    kin.__exit__(None, None, None)
    kin.export_chrome_trace(args.kineto)
if args.profile:
    prof.disable()
    pstats.Stats(prof, stream=sys.stderr).sort_stats("tottime").print_stats(25)
ms = torch.cuda.memory_stats()
print("segments allocated during the run:", ms.get("segment.all.allocated", 0) - seg0,
      "retries:", ms.get("num_alloc_retries"), file=sys.stderr)
slow = [r for r in log if r["step_ms"] > 4]
print(json.dumps({"steps": args.steps, "tasks_per_s": args.steps / dt, "p": args.p, "nogc": args.nogc,
                  "median_step_ms": sorted(r["step_ms"] for r in log)[len(log) // 2],
                  "slow_steps": slow}, indent=None))
