"""Benchmark of the voted-task hot path (driver contract: one JSON line).

Workload (BASELINE.json configs[1], "C2"): dual-modular redundancy of a
4096x4096 fp32 matmul task on one B200 — the tcgen05 TF32 variant (unit
gpu0.tc) and the SIMT FP32 variant (unit gpu0.simt) run as replicas through
the drop-in Runtime (DMR strategy), protected attempts checkpoint their
device-resident inputs (hf_checkpoint into a reserve HBM space), seeded
bit-flip faults are injected at a fixed per-replica probability, hf_vote
decides, mismatches are re-run.  A "step" is one voted task.

  value  tasks/s with A, B already resident in HBM (sole device copies)
  e2e    tasks/s through the same public API with HOST buffers: per step the
         pinned inputs are copied host->device inside invoke() and the
         committed C is read back device->host (read_into)
N > 1: one process per GPU, each running its own independent task stream
(weak scaling, no data-path collective); timing is max over ranks.

--impl reference times the reference's own CPU implementation of the same
task (hetrt from baseline/_ref through its public Runtime API, numpy bodies,
its voting.compare) on the host cores; without baseline/_ref the oracle port
(oracle/: numpy matmul + restated voter) is timed instead.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("hetft", "reference"), default="hetft")
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--fault-prob", type=float, default=0.05, help="per-replica corrupt (bit flip) probability")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=None, help="default max(80, --steps)")
    ap.add_argument("--depth", type=int, default=1, help="TaskStream depth (tasks in flight beyond the one settling)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tmr", action="store_true", help="skip the HetTMR 4096^2 side measurement")
    ap.add_argument("--detect-probes", type=int, default=2000)
    ap.add_argument("--cpu-sample-s", type=float, default=12.0)
    ap.add_argument("--trace-steps", action="store_true", help="per-step host wall times to stderr")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---- clocks sampling -----------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self._t is not None:
            self._t.join(timeout=2)
        sm, smax, power, reasons = [], None, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
                power.append(float(f[3]))
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "power_w_max": max(power) if power else None, "samples": len(sm), "reasons": sorted(reasons)}


# ---- reference / CPU arm ------------------------------------------------------------------

def _reference_module():
    ref = ROOT / "baseline" / "_ref"
    if (ref / "hetrt").exists():
        sys.path.insert(0, str(ref))
        import hetrt  # noqa: F401
        return hetrt
    return None


def reference_tasks(n: int, count_or_seconds, seed: int, by_time: bool):
    """Run DMR n x n matmul tasks with the reference CPU implementation.
    Returns (tasks, seconds, kind, detail)."""
    hetrt = _reference_module()
    rng = np.random.default_rng(seed)
    a = rng.uniform(1, 2, (n, n)).astype(np.float32)
    b = rng.uniform(1, 2, (n, n)).astype(np.float32)
    if hetrt is not None:
        cfg = {"memory_spaces": [{"id": "host", "host": True}],
               "units": [{"id": "cpu0", "kind": "cpu", "memory_space": "host", "seed": 1},
                         {"id": "cpu1", "kind": "cpu", "memory_space": "host", "seed": 2}]}
        rt = hetrt.Runtime(hetrt.load_fleet(cfg), hetrt.RuntimeConfig(serial_replicas=True))
        task = rt.declare_task("matmul", (hetrt.Param.area("A", "r"), hetrt.Param.area("B", "r"),
                                          hetrt.Param.area("C", "w"), hetrt.Param.scalar("n")))

        def body(ctx):
            k = ctx.arg("n")
            A = ctx.request("A", "r").reshape(k, k)
            B = ctx.request("B", "r").reshape(k, k)
            C = ctx.request("C", "w").reshape(k, k)
            np.matmul(A, B, out=C)

        rt.attach_kernel(task, "mm_cpu", "cpu", body)
        zeros = bytes(4 * n * n)

        def one():
            ia = rt.register_data(a.tobytes(), n * n, hetrt.ValueType.FLOAT32, "r")
            ib = rt.register_data(b.tobytes(), n * n, hetrt.ValueType.FLOAT32, "r")
            ic = rt.register_data(zeros, n * n, hetrt.ValueType.FLOAT32, "w")
            rep = rt.invoke(task, {"A": ia, "B": ib, "C": ic, "n": n}, hetrt.Strategy(hetrt.StrategyKind.DMR))
            rt.read_area(ic)
            assert rep.success
        kind, detail = "reference", "hetrt (baseline/_ref) Runtime.invoke DMR: 2 numpy matmul bodies + voting.compare"
    else:
        from oracle import vote as ovote

        def one():
            c0 = a @ b
            c1 = a @ b
            ovote.vote([c0, c1], 1e-3)
        kind, detail = "port", "oracle port: 2 numpy matmuls + oracle.vote (reference absent)"
    # all host cores for the BLAS matmul bodies: torchrun exports
    # OMP_NUM_THREADS=1 to every rank, which would leave the reference arm
    # single-threaded under the driver's multi-GPU launch
    try:
        from threadpoolctl import threadpool_limits
        limiter = threadpool_limits(limits=host_cores(), user_api="blas")
    except Exception:  # noqa: BLE001 - threadpoolctl absent: numpy's own default
        limiter = None
    try:
        t0 = time.perf_counter()
        done = 0
        while True:
            one()
            done += 1
            el = time.perf_counter() - t0
            if by_time and el >= count_or_seconds and done >= 1:
                break
            if not by_time and done >= count_or_seconds:
                break
        return done, time.perf_counter() - t0, kind, detail
    finally:
        if limiter is not None:
            limiter.restore_original_limits()


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    n = args.n
    reference_tasks(n, max(1, args.warmup // 3), args.seed, by_time=False)   # warm caches/BLAS
    tasks, secs, kind, detail = reference_tasks(n, args.steps, args.seed, by_time=False)
    v = tasks / secs
    line = {"metric": "voted tasks/sec (DMR 4096^2 fp32 matmul, TC vs SIMT variants)", "value": v,
            "unit": "tasks/s", "n_gpus": args.gpus, "steps": tasks, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / tasks, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic U[1,2) fp32 operands",
            "config": {"workload": f"C2: DMR {n}x{n} fp32 matmul, detect-and-rerun", "n": n},
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "tasks/s", "cores": host_cores(), "kind": kind,
                             "sample": f"{tasks} tasks: {detail}"},
            "e2e": {"value": v, "unit": "tasks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---- B200 arm ---------------------------------------------------------------------------------

def build_runtime(device: int, fault_prob: float, seed: int):
    import paper_1405_2912_b200 as hf
    cfg = hf.gpu_fleet_config(devices=(device,), kinds=("gpu-tc", "gpu-simt"))
    cfg["memory_spaces"].append({"id": f"gpu{device}ckpt", "device": device, "label": "HBM checkpoint reserve"})
    for i, u in enumerate(cfg["units"]):
        u.update({"corrupt_prob": fault_prob, "corrupt_mode": "bitflip", "seed": seed * 1_000_003 + i * 101 + 17})
    fleet = hf.load_fleet(cfg)
    rt = hf.Runtime(fleet, hf.RuntimeConfig(checkpoint_space=f"gpu{device}ckpt", serial_replicas=True,
                                            attempt_limit=64))
    task = hf.get_workload("matmul").attach(rt, kinds=("gpu-tc", "gpu-simt"))
    return hf, rt, task


def run_hetft_arm(args, rank, world, local):
    import torch
    import torch.distributed as dist

    device = local if torch.cuda.device_count() > local else 0
    torch.cuda.set_device(device)
    # one GPU per rank: NCCL for the barrier and the max over ranks; more
    # ranks than GPUs (a code-path check on a small box) falls back to gloo
    shared_gpu = torch.cuda.device_count() < world
    if world > 1 and not dist.is_initialized():
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{device}"))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if shared_gpu else f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    hf, rt, task = build_runtime(device, args.fault_prob, args.seed + 7919 * rank)
    from paper_1405_2912_b200 import kernels
    n = args.n
    nb = n * n * 4
    space = f"gpu{device}mem"
    # pre-size the device heap for the stream's high-water mark (re-dispatched
    # rounds included): no cudaMalloc inside the timed regions
    rt.reserve(space, nb, 24)
    gen = torch.Generator(device=f"cuda:{device}")
    gen.manual_seed(args.seed * 7919 + rank)
    A = (torch.rand(n * n, device=f"cuda:{device}", generator=gen) + 1).view(torch.uint8)
    B = (torch.rand(n * n, device=f"cuda:{device}", generator=gen) + 1).view(torch.uint8)
    C0 = torch.zeros(nb, dtype=torch.uint8, device=f"cuda:{device}")
    strat = hf.Strategy(hf.StrategyKind.HET_DMR)
    stream = rt.backend.stream(device)

    stats = {"tasks": 0, "rounds": 0, "votes": {}, "injected": 0, "mismatch": 0, "vote_ns": 0,
             "attempt_ns": {}, "attempt_n": {}}

    def record(rep):
        stats["tasks"] += 1
        stats["rounds"] += rep.rounds
        for v in rep.votes:
            stats["votes"][v] = stats["votes"].get(v, 0) + 1
        stats["injected"] += len(rep.injected)
        stats["mismatch"] += rep.fault_counts["vote_mismatch"]
        stats["vote_ns"] += rep.voter_ns

    def device_stream(steps: int, recording: bool):
        """`steps` voted tasks on device-resident inputs through a TaskStream:
        task i+1's replicas are queued on the GPU before task i's verdict is
        read, so host-side settling overlaps kernels."""
        queue = []
        with rt.task_stream(depth=args.depth) as ts:
            for _ in range(steps):
                ia = rt.register_device_data(A, n * n, hf.ValueType.FLOAT32, "r", space)
                ib = rt.register_device_data(B, n * n, hf.ValueType.FLOAT32, "r", space)
                ic = rt.register_device_data(C0, n * n, hf.ValueType.FLOAT32, "w", space)
                queue.append((ts.submit(task, {"A": ia, "B": ib, "C": ic, "n": n}, strat), (ia, ib, ic)))
                while queue and queue[0][0].success:
                    rep, areas = queue.pop(0)
                    if recording:
                        record(rep)
                    for x in areas:
                        rt.release(x)
        for rep, areas in queue:
            if not rep.success:
                raise RuntimeError("task failed")
            if recording:
                record(rep)
            for x in areas:
                rt.release(x)

    # trace per-kernel durations via the executor's measured attempts
    def on_trace(line: str):
        if line.startswith("ATT") and "fault=none" in line:
            f = dict(kv.split("=", 1) for kv in line.split()[1:] if "=" in kv)
            k = f["kernel"]
            stats["attempt_ns"][k] = stats["attempt_ns"].get(k, 0) + int(f["duration_ns"])
            stats["attempt_n"][k] = stats["attempt_n"].get(k, 0) + 1

    # the clock sampler starts during warm-up (nvidia-smi needs ~0.5 s to
    # emit its first sample) and stops right after the timed region
    sampler = ClockSampler(device) if rank == 0 else None
    device_stream(1, False)
    if sampler:
        sampler.start()
    t_start = time.perf_counter()
    done = 1
    while done < args.warmup or time.perf_counter() - t_start < 0.8:
        device_stream(max(1, args.warmup), False)
        done += max(1, args.warmup)
    torch.cuda.synchronize()

    # ---- timed region: device-resident inputs ----
    rt.executor._trace = on_trace
    barrier()
    torch.cuda.synchronize()
    launches0 = kernels.LAUNCHES
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    device_stream(args.steps, True)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop() if sampler else None
    launches = kernels.LAUNCHES - launches0
    rt.executor._trace = None
    t_dev = ev0.elapsed_time(ev1) * 1e-3
    t_max = max_over_ranks(t_dev)

    # ---- e2e: host buffers through the same API (H2D inside invoke, D2H read) ----
    # at least 80 steps: the pipeline fill (first 128 MiB H2D before any
    # kernel can start) and drain (last D2H) are paid once per timed region
    e2e_steps = args.e2e_steps or max(80, args.steps)
    hA = torch.empty(nb, dtype=torch.uint8).pin_memory()
    hB = torch.empty(nb, dtype=torch.uint8).pin_memory()
    hC = torch.empty(nb, dtype=torch.uint8).pin_memory()
    hZ = torch.zeros(nb, dtype=torch.uint8).pin_memory()
    hA.copy_(A.cpu())
    hB.copy_(B.cpu())

    def stage(i):
        """Register step i's host inputs and start their H2D on the copy stream."""
        ia = rt.register_host_buffer(hA, n * n, hf.ValueType.FLOAT32, "r")
        ib = rt.register_host_buffer(hB, n * n, hf.ValueType.FLOAT32, "r")
        ic = rt.register_host_buffer(hZ, n * n, hf.ValueType.FLOAT32, "w")
        rt.prefetch(ia, space)
        rt.prefetch(ib, space)
        return ia, ib, ic

    LOOKAHEAD = 2

    def host_stream(steps):
        """Software pipeline over the public API: step i+1's inputs go H2D on
        the copy engine and step i-1's result goes D2H while step i computes;
        a TaskStream keeps the next task's kernels queued behind the current."""
        # inputs are staged LOOKAHEAD steps ahead, so the copy engine stays
        # busy while the host blocks on a re-dispatched (mismatching) task
        staged = [stage(i) for i in range(min(LOOKAHEAD, steps))]
        queue, retired, last = [], [], None
        reps = []
        with rt.task_stream(depth=args.depth) as ts:
            for i in range(steps):
                ia, ib, ic = staged.pop(0)
                if i + LOOKAHEAD < steps:
                    staged.append(stage(i + LOOKAHEAD))
                queue.append((ts.submit(task, {"A": ia, "B": ib, "C": ic, "n": n}, strat), (ia, ib, ic)))
                reps.append(queue[-1][0])
                if args.trace_steps:
                    print(f"e2e step {i} t={time.perf_counter():.6f} rounds={queue[-1][0].rounds}", file=sys.stderr)
                while queue and queue[0][0].success:
                    rep, areas = queue.pop(0)
                    last = rt.read_into_async(areas[2], hC)
                    for x in retired:     # released one step late: their D2H overlapped
                        rt.release(x)
                    retired = list(areas)
        for rep, areas in queue:
            last = rt.read_into_async(areas[2], hC)
            retired += list(areas)
        if last is not None:
            last.synchronize()
        for x in retired:
            rt.release(x)
        return sum(r.rounds for r in reps)

    host_stream(2)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_rounds = host_stream(e2e_steps)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    t_e2e = max_over_ranks(e0.elapsed_time(e1) * 1e-3)
    # the result of the last step really arrived: spot-check it against the device copy
    hC_check = hC.view(torch.float32)[:4].clone()

    # ---- kernel-level measurements (same process, after the timed regions) ----
    kern = kernel_rooflines(device, n, kernels, torch)
    # at least 30 timed tasks: a 20-task window swings with the fault draws
    tmr = tmr_rate(device, n, args.fault_prob, args.seed + 7919 * rank, max(30, args.steps),
                   max(5, args.warmup), torch) if not args.no_tmr else None
    detect = detect_rate(device, n, kernels, torch, args.seed, probes=args.detect_probes) if rank == 0 else None

    total_tasks = args.steps * world
    if rank != 0:
        return
    peaks, peak_src = load_peaks()
    simt_ns = stats["attempt_ns"].get("mm_simt", 0) / max(1, stats["attempt_n"].get("mm_simt", 1))
    tc_ns = stats["attempt_ns"].get("mm_tc", 0) / max(1, stats["attempt_n"].get("mm_tc", 1))
    flops = 2.0 * n ** 3
    simt_tflops = flops / (simt_ns * 1e-9) / 1e12 if simt_ns else None
    sm_max = (clocks or {}).get("sm_max_mhz") or 1965.0
    ffma_peak, ffma_src = fp32_peak(sm_max)
    traffic = ncu_traffic("sgemm_128x128", "transpose_a")
    vote_gbs = (stats["votes"] and stats["vote_ns"]) and \
        (2 * nb * sum(stats["votes"].values())) / (stats["vote_ns"] * 1e-9) / 1e9
    cpu = None
    if not args.no_cpu_baseline:
        tasks, secs, kind, detail = reference_tasks(n, args.cpu_sample_s, args.seed, by_time=True)
        cpu = {"value": tasks / secs, "unit": "tasks/s", "cores": host_cores(), "kind": kind,
               "sample": f"{tasks} tasks in {secs:.1f} s: {detail}"}
    line = {
        "metric": "voted tasks/sec (DMR 4096^2 fp32 matmul, TC vs SIMT variants)",
        "value": total_tasks / t_max,
        "unit": "tasks/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * t_max / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic U[1,2) fp32 operands generated on device (no dataset)",
        "config": {"workload": f"C2: DMR {n}x{n} fp32 matmul, tcgen05-TF32 vs SIMT-FP32 replicas, "
                               f"HBM checkpoint of inputs, bit-flip faults p={args.fault_prob}/replica, "
                               f"hf_vote detect-and-rerun", "n": n, "replicas": 2,
                   "strategy": "hetdmr", "parallelism": f"independent task streams x{world}",
                   "l2": "operands (3 x 64 MiB) exceed the 126 MB L2; no flush needed"},
        "e2e": {"value": (e2e_steps * world) / t_e2e, "unit": "tasks/s", "steps": e2e_steps,
                "rounds": e2e_rounds,
                "note": "own window of max(80, steps) tasks with their own fault draws; the H2D of "
                        "step i+2 and the D2H of step i-1 overlap step i, PCIe-bound (~2.56 ms/step)",
                "h2d_bytes_per_step": 2 * nb,
                "d2h_bytes_per_step": nb},
        "gpu_launches": launches,
        "clocks": clocks,
        "roofline": {"bound": "fp32-simt", "kernel": "hf_gemm_simt (incl. A^T pre-pass)",
                     "achieved": simt_tflops, "peak": ffma_peak, "unit": "TFLOP/s",
                     "frac": (simt_tflops / ffma_peak) if simt_tflops else None, "traffic": traffic,
                     "traffic_unit": "DRAM bytes per launch (ncu --set full, GEMM + A^T pre-pass; "
                                     f"operand bytes 3*{n}^2*4 = {3 * nb})",
                     "peak_source": ffma_src,
                     "algorithmic": f"2*{n}^3 flop per launch"},
        "rooflines": kern,
        "replica_ms": {"mm_simt": simt_ns * 1e-6, "mm_tc": tc_ns * 1e-6},
        "voter_gbs_in_task": vote_gbs,
        "tmr": tmr,
        "detect": detect,
        "faults": {"injected": stats["injected"], "detected_mismatch_votes": stats["mismatch"],
                   "votes": stats["votes"], "rounds": stats["rounds"]},
        "cpu_baseline": cpu,
        "peaks": {"source": peak_src, **peaks},
    }
    print(json.dumps(line), flush=True)


def fp32_peak(sm_max_mhz: float):
    """FP32 SIMT peak for the SIMT variant's roofline (MEASURED_PEAKS.json has
    none): the packed-FFMA2 probe tools/fp32_peak (built by build()) run live
    on this GPU, else the round's committed probe result, else nominal."""
    exe = ROOT / "tools" / "fp32_peak"
    if exe.exists():
        try:
            out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
            d = json.loads(out.stdout.strip().splitlines()[-1])
            if out.returncode != 0 or not d["ffma2_tflops"] > 0:
                raise ValueError(d.get("error"))
            return d["ffma2_tflops"], ("measured live: tools/fp32_peak (FFMA2 loop, 148x4 CTAs, best of 5; an 8x8 "
                                       "outer product issued b-pair-outer reaches it too, tools/ffma2_forms.cu); "
                                       f"issued a-scalar-outer it peaks at {d['ffma2_bcast_tflops']:.1f}, which is "
                                       "where ptxas's schedule of the GEMM lands")
        except (OSError, ValueError, KeyError, IndexError, subprocess.SubprocessError):
            pass
    for p in sorted((ROOT / "profiles").glob("r*_fp32_peak.json"), reverse=True):
        return json.loads(p.read_text())["ffma2_tflops"], f"measured: {p.relative_to(ROOT)} (FFMA2 probe)"
    return 148 * 128 * 2 * sm_max_mhz * 1e6 / 1e12, f"nominal FFMA 148 SM x 128 lanes x 2 flop x {sm_max_mhz:.0f} MHz"


def ncu_traffic(*kernels_):
    """DRAM bytes per launch of `kernels_` summed, from the newest committed
    ncu --set full capture summary (tools/ncu_traffic.py), or None."""
    for p in sorted((ROOT / "profiles").glob("r*_ncu_traffic*.json"), reverse=True):
        ks = json.loads(p.read_text())["kernels"]
        if all(k in ks for k in kernels_):
            return sum(ks[k]["traffic_bytes"] for k in kernels_)
    return None


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"]}, "MEASURED_PEAKS.json"
    return dict(PEAKS_FALLBACK), "fallback (B200_PROFILING.md)"


def detect_rate(device, n, kernels, torch, seed: int, probes: int = 2000):
    """Detect rate of the DMR voter on real diverse outputs: C_tc and C_simt
    of one n x n task; each probe flips one seeded (element, bit) of C_simt,
    votes on the GPU (hf_vote, K = 2, δ = 1e-3), flips it back.  Every GPU
    decision is checked against the oracle predicate on that element (the
    unflipped pair agrees everywhere, verified first).  Reports the detect
    rate overall and per bit class and the agreement with the oracle."""
    import random as _random
    from oracle import vote as ovote
    d = f"cuda:{device}"
    g = torch.Generator(device=d)
    g.manual_seed(seed)
    a = torch.rand(n, n, device=d, generator=g) + 1
    b = torch.rand(n, n, device=d, generator=g) + 1
    c_tc = torch.empty(n, n, device=d)
    c_si = torch.empty(n, n, device=d)
    kernels.gemm_tc(a, b, c_tc)
    kernels.gemm_simt(a, b, c_si)
    x, y = c_tc.view(-1), c_si.view(-1)
    base = kernels.vote([x, y], 1e-3)
    if base.verdict != "match":
        return {"error": f"unflipped TC/SIMT outputs disagree ({base.verdict}, first {base.first_div})"}
    hx, hy = x.cpu().numpy(), y.cpu().numpy()
    rng = _random.Random(seed * 1_000_003 + 17)
    classes = {"0-13": [0, 0], "14": [0, 0], "15-22": [0, 0], "23-30 (exponent)": [0, 0], "31 (sign)": [0, 0]}
    agree = detected = 0
    for _ in range(probes):
        e = rng.randrange(n * n)
        bit = rng.randrange(32)
        kernels.inject_bitflip(y, e, bit)
        res = kernels.vote([x, y], 1e-3)
        kernels.inject_bitflip(y, e, bit)
        flipped = hy[e:e + 1].copy()
        flipped.view("u4")[0] ^= 1 << bit
        oracle_detect = not bool(ovote.pair_ok(hx[e:e + 1], flipped, 1e-3)[0])
        gpu_detect = res.verdict == "mismatch"
        agree += int(gpu_detect == oracle_detect and (not gpu_detect or res.first_div == e))
        detected += int(gpu_detect)
        key = "0-13" if bit <= 13 else "14" if bit == 14 else "15-22" if bit <= 22 else \
            "23-30 (exponent)" if bit <= 30 else "31 (sign)"
        classes[key][0] += int(gpu_detect)
        classes[key][1] += 1
    return {"probes": probes, "detect_rate": detected / probes, "oracle_agreement": agree / probes,
            "per_bit_class": {k: (v[0] / v[1] if v[1] else None) for k, v in classes.items()},
            "note": "one seeded bit flip per probe in the SIMT replica of a real 4096^2 TC/SIMT pair; "
                    "known answer at δ=1e-3: bits 0-13 never, 14 ~96%, 15-31 always (uniform bit ≈ 56%)"}


def kernel_rooflines(device, n, kernels, torch):
    """Per-kernel rooflines: vote / checkpoint vs HBM, TC GEMM vs tensor, all
    CUDA-event timed on the launching stream over operands > L2."""
    peaks, _ = load_peaks()
    st = torch.cuda.Stream(device=device)
    d = f"cuda:{device}"
    out = {}

    def time_it(fn, iters=10):
        torch.cuda.synchronize()   # operands come from default-stream torch ops: finished before timing
        with torch.cuda.stream(st):
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(iters):
                fn()
            e1.record(st)
        st.synchronize()
        return e0.elapsed_time(e1) * 1e-3 / iters

    m = n * n
    base = torch.rand(m, device=d) + 1
    reps = [base * (1 + 1e-6 * torch.randn(m, device=d)) for _ in range(3)]
    kernels.inject_bitflip(reps[2], m // 3, 27, stream=st)
    ws = kernels.VoteWorkspace(device, stream=st)
    for K in (2, 3):
        t = time_it(lambda: kernels.vote_async(reps[:K], ws, 1e-3, voted=reps[0] if K >= 3 else None, stream=st))
        byts = K * m * 4      # replica reads; the in-place voted output stores only differing vectors
        out[f"hf_vote_K{K}"] = {"bound": "hbm", "achieved": byts / t / 1e9, "peak": peaks["hbm_gbs"],
                                "unit": "GB/s", "frac": byts / t / 1e9 / peaks["hbm_gbs"],
                                "us": t * 1e6, "algorithmic_bytes": byts,
                                "note": "voted output written in place over replica 0 (only differing "
                                        "vectors stored)" if K >= 3 else "no voted output (K = 2 verdict only)"}
    dst = torch.empty_like(base)
    t = time_it(lambda: kernels.checkpoint(dst, base, stream=st))
    out["hf_checkpoint"] = {"bound": "hbm", "achieved": 2 * m * 4 / t / 1e9, "peak": peaks["hbm_gbs"],
                            "unit": "GB/s", "frac": 2 * m * 4 / t / 1e9 / peaks["hbm_gbs"], "us": t * 1e6,
                            "algorithmic_bytes": 2 * m * 4}
    a = base.view(n, n)
    b = reps[1].view(n, n)
    c = torch.empty(n, n, device=d)
    t = time_it(lambda: kernels.gemm_tc(a, b, c, stream=st), iters=10)
    tf32_peak = peaks["bf16_tflops"] / 2
    out["hf_gemm_tc"] = {"bound": "tensor", "achieved": 2 * n ** 3 / t / 1e12, "peak": tf32_peak,
                         "unit": "TFLOP/s", "frac": 2 * n ** 3 / t / 1e12 / tf32_peak, "us": t * 1e6,
                         "peak_source": "measured bf16 dense / 2 (tf32 rate)", "includes": "B^T + RN pre-pass"}
    t = time_it(lambda: kernels.gemm_simt(a, b, c, stream=st), iters=5)
    out["hf_gemm_simt"] = {"bound": "fp32-simt", "achieved": 2 * n ** 3 / t / 1e12, "unit": "TFLOP/s",
                           "us": t * 1e6}
    return out


def tmr_rate(device, n, fault_prob, seed, steps, warmup, torch):
    """North-star headline shape on one GPU: HetTMR of the three diverse
    variants (tcgen05 TF32, SIMT FP32, tcgen05 3xBF16) on a 4096^2 fp32
    matmul, device-resident inputs checkpointed into HBM, bit-flip faults at
    the same per-replica probability, majority vote (K = 3) corrects a single
    faulty replica.  CUDA-event timed on the runtime's compute stream."""
    import paper_1405_2912_b200 as hf
    kinds = ("gpu-tc", "gpu-simt", "gpu-tc3")
    cfg = hf.gpu_fleet_config(devices=(device,), kinds=kinds)
    cfg["memory_spaces"].append({"id": f"gpu{device}ckpt", "device": device, "label": "HBM checkpoint reserve"})
    for i, u in enumerate(cfg["units"]):
        u.update({"corrupt_prob": fault_prob, "corrupt_mode": "bitflip", "seed": seed * 1_000_003 + i * 101 + 31})
    rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(checkpoint_space=f"gpu{device}ckpt",
                                                         serial_replicas=True, attempt_limit=64))
    task = hf.get_workload("matmul").attach(rt, kinds=kinds)
    space = f"gpu{device}mem"
    nb = n * n * 4
    rt.reserve(space, nb, 24)
    g = torch.Generator(device=f"cuda:{device}")
    g.manual_seed(seed * 7919 + 5)
    A = (torch.rand(n * n, device=f"cuda:{device}", generator=g) + 1).view(torch.uint8)
    B = (torch.rand(n * n, device=f"cuda:{device}", generator=g) + 1).view(torch.uint8)
    C0 = torch.zeros(nb, dtype=torch.uint8, device=f"cuda:{device}")
    strat = hf.Strategy(hf.StrategyKind.HET_TMR)
    votes, rounds = {}, 0

    def go(k, recording):
        nonlocal rounds
        queue = []
        with rt.task_stream(depth=1) as ts:
            for _ in range(k):
                areas = tuple(rt.register_device_data(x, n * n, hf.ValueType.FLOAT32, m, space)
                              for x, m in ((A, "r"), (B, "r"), (C0, "w")))
                queue.append((ts.submit(task, dict(zip("ABC", areas), n=n), strat), areas))
                while queue and queue[0][0].success:
                    rep, ar = queue.pop(0)
                    if recording:
                        rounds += rep.rounds
                        for v in rep.votes:
                            votes[v] = votes.get(v, 0) + 1
                    for x in ar:
                        rt.release(x)
        for rep, ar in queue:
            if recording:
                rounds += rep.rounds
                for v in rep.votes:
                    votes[v] = votes.get(v, 0) + 1
            for x in ar:
                rt.release(x)

    go(max(3, warmup), False)
    st = rt.backend.stream(device)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    go(steps, True)
    e1.record(st)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3
    return {"value": steps / t, "unit": "tasks/s", "ms_per_task": 1e3 * t / steps, "steps": steps,
            "workload": f"HetTMR {n}x{n} fp32 matmul (tcgen05 TF32 + SIMT FP32 + tcgen05 3xBF16 replicas "
                        f"on 1 GPU), HBM checkpoint of inputs, bit flips p={fault_prob}/replica, K=3 majority vote",
            "votes": votes, "rounds": rounds}


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    run_hetft_arm(args, rank, world, local)


if __name__ == "__main__":
    main()
