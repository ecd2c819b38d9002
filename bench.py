"""Benchmark of the voted-task hot path (driver contract: one JSON line).

Headline workload (BASELINE.json north_star / metric): HetTMR of a 4096x4096
fp32 matmul task on one B200 — three diverse replicas, the tcgen05 TF32
variant (unit gpu0.tc), the SIMT FP32 variant (gpu0.simt) and the tcgen05
3xBF16 variant (gpu0.tc3) — through the drop-in Runtime: protected attempts
checkpoint their device-resident inputs (hf_checkpoint into a reserve HBM
space), every replica draws seeded bit-flip faults at a fixed probability,
hf_vote (K = 3) commits the majority (a single faulty replica is corrected
in place), an element without a majority re-runs.  A "step" is one voted
task.

  value  tasks/s with A, B already resident in HBM (sole device copies)
  e2e    tasks/s through the same public API with HOST buffers: per step the
         pinned inputs are copied host->device inside the task and the
         committed C is read back device->host (read_into_async)
  dmr    BASELINE configs[1] (HetDMR, TC vs SIMT, detect-and-rerun), extra key
N > 1: one process per GPU, each running its own independent task stream
(weak scaling, no data-path collective); timing is max over ranks.  With
N >= 2, rank 0 also sweeps cross-GPU votes ("c4_cross_gpu": K replicas on K
GPUs, the vote sliced over them, NVLink ingress per GPU against a measured
P2P peak) and with N >= 3 runs configs[2] ("c3": the three replicas on GPUs
0/1/2, inputs pulled over NVLink, the sliced vote).

--impl reference times the reference's own CPU implementation of the same
task on the host cores: hetrt from baseline/_ref (its MemoryManager with a
protected checkpoint of the inputs, simulate_execution with the reference
fault model around three numpy fp32 matmul bodies, voting.compare on the
pairs (0,1), (0,2), (1,2), commit of an agreeing replica).  Without
baseline/_ref the oracle port (oracle/: numpy + restated voter) is timed.
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
    ap.add_argument("--e2e-steps", type=int, default=None, help="default max(160, --steps)")
    ap.add_argument("--depth", type=int, default=1, help="TaskStream depth (tasks in flight beyond the one settling)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dmr", action="store_true", help="skip the HetDMR (configs[1]) side measurement")
    ap.add_argument("--no-c3", action="store_true", help="skip the replicas-on-3-GPUs sub-measurement (N >= 3)")
    ap.add_argument("--c4-devices", default=None,
                    help="run the cross-GPU vote sweep on these GPUs at any N (e.g. 0,0,0: one-GPU code-path check)")
    ap.add_argument("--c3-devices", default=None,
                    help="run the c3 sub-measurement on these GPUs at any N (e.g. 0,0,0: one-GPU code-path check)")
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


METRIC = "voted tasks/sec (HetTMR 4096^2 fp32 matmul, 3 diverse replicas, majority vote)"


def bench_config(args, world: int) -> dict:
    """The workload both arms report (identical dict: the driver compares them)."""
    n = args.n
    return {"workload": f"HetTMR {n}x{n} fp32 matmul: 3 diverse replicas (tcgen05 TF32, SIMT FP32, "
                        f"tcgen05 3xBF16; reference arm: 3 numpy fp32 bodies), protected checkpoint of the "
                        f"inputs, per-replica fault p={args.fault_prob}, K=3 majority vote, re-run without "
                        f"majority",
            "n": n, "replicas": 3, "strategy": "hettmr", "fault_prob": args.fault_prob,
            "parallelism": f"independent task streams x{world}",
            "l2": "operands (4 x 64 MiB per task) exceed the 126 MB L2; no flush needed"}


def _ref_tmr_runner(hetrt, n, seed, fault_prob):
    """One HetTMR n x n task through the reference's own pieces (it has no
    TMR strategy; its Runtime only runs DMR, executor.py:225-285): the
    reference MemoryManager with the inputs as sole copies in a device space
    (so protected requests checkpoint them, memory.py:176-189), three units of
    its fault model (corrupt_prob = fault_prob, its CorruptionSpec) running
    numpy fp32 matmul bodies through simulate_execution (devices.py:223-259),
    voting.compare on every pair (voting.py:106-123) with the result bytes
    copied out as Executor._vote does (executor.py:319-325), commit of a
    replica that agrees with another, otherwise a re-run of all three.
    Returns (run_one, setup_one): setup registers a task's areas (untimed)."""
    from hetrt import memory as rmem
    from hetrt import voting as rvote
    from hetrt.devices import FaultClass, ValueType, simulate_execution
    f32 = ValueType.FLOAT32
    cfg = {"memory_spaces": [{"id": "host", "host": True}, {"id": "dev"}],
           "units": [{"id": f"cpu{i}", "kind": "cpu", "memory_space": "dev", "corrupt_prob": fault_prob,
                      "seed": seed * 1_000_003 + i * 101 + 31} for i in range(3)]}
    fleet = hetrt.load_fleet(cfg)
    units = [fleet.units[f"cpu{i}"] for i in range(3)]
    vcfg = rvote.VoterConfig()
    rng = np.random.default_rng(seed)
    a = rng.uniform(1, 2, (n, n)).astype(np.float32).tobytes()
    b = rng.uniform(1, 2, (n, n)).astype(np.float32).tobytes()
    zeros = bytes(4 * n * n)

    def setup():
        # a fresh manager per task: the reference has no area release, and the
        # areas of finished tasks would otherwise pile up (6 x 64 MiB each)
        mm = rmem.MemoryManager(fleet)
        ia = mm.register(a, n * n, f32, "r")
        ib = mm.register(b, n * n, f32, "r")
        ic = mm.register(zeros, n * n, f32, "w")
        for x in (ia, ib):            # device-resident sole copies (the GPU arm's register_device_data)
            h = mm.request(x, "dev", "rw")
            mm.commit_success([h])
        return mm, ia, ib, ic

    def run(areas):
        mm, ia, ib, ic = areas
        rounds = 0
        while True:
            rounds += 1
            hcs = []
            for u in units:
                while True:
                    ha = mm.request(ia, "dev", "r", protect=True)
                    hb = mm.request(ib, "dev", "r", protect=True)
                    hc = mm.request(ic, "dev", "w", protect=True)
                    A = np.frombuffer(ha.payload, np.float32).reshape(n, n)
                    B = np.frombuffer(hb.payload, np.float32).reshape(n, n)
                    C = np.frombuffer(hc.payload, np.float32).reshape(n, n)
                    out = simulate_execution(u, "mm_cpu", "cpu", n * n, body=lambda: np.matmul(A, B, out=C),
                                             write_views=[(C.reshape(-1), f32)])
                    if out.fault in (None, FaultClass.CORRUPT):
                        hcs.append(hc)
                        break
            res = [{ic: (bytes(h.payload), f32, 4)} for h in hcs]
            agree = [False] * 3
            for i, j in ((0, 1), (0, 2), (1, 2)):
                if rvote.compare(res[i], res[j], vcfg).verdict == "match":
                    agree[i] = agree[j] = True
            if any(agree):
                mm.commit_success([hcs[agree.index(True)]])
                return rounds
    return run, setup


def reference_tasks(n: int, count_or_seconds, seed: int, by_time: bool, fault_prob: float = 0.05,
                    max_seconds: float = 1e9):
    """Run HetTMR n x n matmul tasks with the reference CPU implementation.
    Returns (tasks, seconds, kind, detail); only the tasks are timed (the
    per-task area registration is not)."""
    hetrt = _reference_module()
    if hetrt is not None:
        run, setup = _ref_tmr_runner(hetrt, n, seed, fault_prob)
        kind = "reference"
        detail = ("hetrt (baseline/_ref): MemoryManager protected checkpoint, 3 numpy fp32 matmul bodies "
                  "via simulate_execution (reference fault model), voting.compare on pairs (0,1),(0,2),(1,2)")
    else:
        from oracle import vote as ovote
        rng = np.random.default_rng(seed)
        a = rng.uniform(1, 2, (n, n)).astype(np.float32)
        b = rng.uniform(1, 2, (n, n)).astype(np.float32)

        def setup():
            return None

        def run(_):
            ovote.vote([a @ b, a @ b, a @ b], 1e-3)
            return 1
        kind, detail = "port", "oracle port: 3 numpy matmuls + oracle.vote (reference absent)"
    # all host cores for the BLAS matmul bodies: torchrun exports
    # OMP_NUM_THREADS=1 to every rank, which would leave the reference arm
    # single-threaded under the driver's multi-GPU launch
    try:
        from threadpoolctl import threadpool_limits
        limiter = threadpool_limits(limits=host_cores(), user_api="blas")
    except Exception:  # noqa: BLE001 - threadpoolctl absent: numpy's own default
        limiter = None
    try:
        spent, done, rounds = 0.0, 0, 0
        while True:
            areas = setup()
            t0 = time.perf_counter()
            rounds += run(areas)
            spent += time.perf_counter() - t0
            done += 1
            if by_time and spent >= count_or_seconds:
                break
            if not by_time and (done >= count_or_seconds or spent >= max_seconds):
                break
        return done, spent, kind, f"{detail}; {rounds} rounds"
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
    reference_tasks(n, 1, args.seed, by_time=False, fault_prob=args.fault_prob)   # warm caches/BLAS
    # bounded: at most ~2 min of CPU work whatever --steps asks
    tasks, secs, kind, detail = reference_tasks(n, args.steps, args.seed, by_time=False,
                                                fault_prob=args.fault_prob, max_seconds=120.0)
    v = tasks / secs
    line = {"metric": METRIC, "value": v,
            "unit": "tasks/s", "n_gpus": args.gpus, "steps": tasks, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / tasks, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic U[1,2) fp32 operands",
            "config": bench_config(args, world),
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "tasks/s", "cores": host_cores(), "kind": kind,
                             "sample": f"{tasks} tasks: {detail}"},
            "e2e": {"value": v, "unit": "tasks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---- B200 arm ---------------------------------------------------------------------------------

TMR_KINDS = ("gpu-tc", "gpu-simt", "gpu-tc3")
DMR_KINDS = ("gpu-tc", "gpu-simt")


def build_runtime(device: int, fault_prob: float, seed: int, kinds=TMR_KINDS):
    import paper_1405_2912_b200 as hf
    cfg = hf.gpu_fleet_config(devices=(device,), kinds=kinds)
    cfg["memory_spaces"].append({"id": f"gpu{device}ckpt", "device": device, "label": "HBM checkpoint reserve"})
    for i, u in enumerate(cfg["units"]):
        u.update({"corrupt_prob": fault_prob, "corrupt_mode": "bitflip", "seed": seed * 1_000_003 + i * 101 + 17})
    fleet = hf.load_fleet(cfg)
    rt = hf.Runtime(fleet, hf.RuntimeConfig(checkpoint_space=f"gpu{device}ckpt", serial_replicas=True,
                                            attempt_limit=64))
    task = hf.get_workload("matmul").attach(rt, kinds=kinds)
    return hf, rt, task


class TaskStreamBench:
    """Voted n x n matmul tasks of one strategy through the drop-in Runtime's
    TaskStream on one GPU: device-resident inputs (`device_stream`) or host
    buffers with H2D/D2H inside the stream (`host_stream`)."""

    LOOKAHEAD = 2

    def __init__(self, args, device, rank, kinds, strategy, seed_salt=0, built=None, space=None):
        import torch
        self.torch = torch
        self.args, self.device, self.n = args, device, args.n
        self.hf, self.rt, self.task = built or build_runtime(device, args.fault_prob,
                                                             args.seed + 7919 * rank + seed_salt, kinds)
        hf, n = self.hf, self.n
        self.nb = n * n * 4
        self.space = space or f"gpu{device}mem"
        # pre-size the device heap for the stream's high-water mark (re-dispatched
        # rounds included): no cudaMalloc inside the timed regions
        for sp in self.rt.fleet.spaces.values():
            if sp.device is not None and sp.id != "ckpt" and not sp.id.endswith("ckpt"):
                self.rt.reserve(sp.id, self.nb, 32 if sp.id == self.space else 12)
        gen = torch.Generator(device=f"cuda:{device}")
        gen.manual_seed(args.seed * 7919 + rank)
        self.A = (torch.rand(n * n, device=f"cuda:{device}", generator=gen) + 1).view(torch.uint8)
        self.B = (torch.rand(n * n, device=f"cuda:{device}", generator=gen) + 1).view(torch.uint8)
        self.strat = strategy if isinstance(strategy, hf.Strategy) else hf.Strategy(strategy)
        self.stream = self.rt.backend.stream(device)
        self.stats = {"tasks": 0, "rounds": 0, "votes": {}, "injected": 0, "mismatch": 0, "corrected": 0,
                      "vote_ns": 0, "attempt_ns": {}, "attempt_n": {}}
        self._host = None

    def record(self, rep):
        st = self.stats
        st["tasks"] += 1
        st["rounds"] += rep.rounds
        for v in rep.votes:
            st["votes"][v] = st["votes"].get(v, 0) + 1
        st["injected"] += len(rep.injected)
        st["mismatch"] += rep.fault_counts["vote_mismatch"]
        st["corrected"] += rep.fault_counts["vote_corrected"]
        st["vote_ns"] += rep.voter_ns

    def on_trace(self, line: str):
        if line.startswith("ATT") and "fault=none" in line:
            f = dict(kv.split("=", 1) for kv in line.split()[1:] if "=" in kv)
            k = f["kernel"]
            self.stats["attempt_ns"][k] = self.stats["attempt_ns"].get(k, 0) + int(f["duration_ns"])
            self.stats["attempt_n"][k] = self.stats["attempt_n"].get(k, 0) + 1

    def device_stream(self, steps: int, recording: bool):
        """`steps` voted tasks on device-resident inputs through a TaskStream:
        task i+1's replicas are queued on the GPU before task i's verdict is
        read, so host-side settling overlaps kernels."""
        rt, hf, n = self.rt, self.hf, self.n
        hZ = self._host_buffers()[3]
        queue = []
        with rt.task_stream(depth=self.args.depth) as ts:
            for _ in range(steps):
                ia = rt.register_device_data(self.A, n * n, hf.ValueType.FLOAT32, "r", self.space)
                ib = rt.register_device_data(self.B, n * n, hf.ValueType.FLOAT32, "r", self.space)
                # the output area as reference programs register it (a host
                # payload of zeros; the reference arm does the same): a "w"
                # request never reads it, and with a host copy it is not a
                # sole device copy, so no checkpoint of C
                ic = rt.register_host_buffer(hZ, n * n, hf.ValueType.FLOAT32, "w")
                queue.append((ts.submit(self.task, {"A": ia, "B": ib, "C": ic, "n": n}, self.strat), (ia, ib, ic)))
                while queue and queue[0][0].success:
                    rep, areas = queue.pop(0)
                    if recording:
                        self.record(rep)
                    for x in areas:
                        rt.release(x)
        for rep, areas in queue:
            if not rep.success:
                raise RuntimeError("task failed")
            if recording:
                self.record(rep)
            for x in areas:
                rt.release(x)

    def _host_buffers(self):
        if self._host is None:
            torch, nb = self.torch, self.nb
            hA = torch.empty(nb, dtype=torch.uint8).pin_memory()
            hB = torch.empty(nb, dtype=torch.uint8).pin_memory()
            hC = torch.empty(nb, dtype=torch.uint8).pin_memory()
            hZ = torch.zeros(nb, dtype=torch.uint8).pin_memory()
            hA.copy_(self.A.cpu())
            hB.copy_(self.B.cpu())
            self._host = (hA, hB, hC, hZ)
        return self._host

    def host_stream(self, steps):
        """Software pipeline over the public API: step i+LOOKAHEAD's inputs go
        H2D on the copy engine and step i-1's result goes D2H while step i
        computes; a TaskStream keeps the next task's kernels queued behind the
        current.  Returns the rounds the tasks took."""
        rt, hf, n = self.rt, self.hf, self.n
        hA, hB, hC, hZ = self._host_buffers()

        def stage():
            ia = rt.register_host_buffer(hA, n * n, hf.ValueType.FLOAT32, "r")
            ib = rt.register_host_buffer(hB, n * n, hf.ValueType.FLOAT32, "r")
            ic = rt.register_host_buffer(hZ, n * n, hf.ValueType.FLOAT32, "w")
            rt.prefetch(ia, self.space)
            rt.prefetch(ib, self.space)
            return ia, ib, ic

        # inputs are staged LOOKAHEAD steps ahead, so the copy engine stays
        # busy while the host blocks on a re-dispatched (mismatching) task
        staged = [stage() for _ in range(min(self.LOOKAHEAD, steps))]
        queue, retired, last, reps = [], [], None, []
        with rt.task_stream(depth=self.args.depth) as ts:
            for i in range(steps):
                ia, ib, ic = staged.pop(0)
                if i + self.LOOKAHEAD < steps:
                    staged.append(stage())
                queue.append((ts.submit(self.task, {"A": ia, "B": ib, "C": ic, "n": n}, self.strat), (ia, ib, ic)))
                reps.append(queue[-1][0])
                if self.args.trace_steps:
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

    def warm(self):
        self.device_stream(1, False)
        t0 = time.perf_counter()
        done = 1
        while done < self.args.warmup or time.perf_counter() - t0 < 0.8:
            self.device_stream(max(1, self.args.warmup), False)
            done += max(1, self.args.warmup)
        self.torch.cuda.synchronize()

    def timed(self, fn, *a):
        """CUDA-event time of fn(*a) on the runtime's compute stream (seconds)."""
        torch = self.torch
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        out = fn(*a)
        e1.record(self.stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e-3, out

    def kernel_ms(self, kernel: str):
        c = self.stats["attempt_n"].get(kernel, 0)
        return self.stats["attempt_ns"].get(kernel, 0) / c * 1e-6 if c else None


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

    from paper_1405_2912_b200 import kernels
    n = args.n
    nb = n * n * 4
    import paper_1405_2912_b200 as hf
    tmr = TaskStreamBench(args, device, rank, TMR_KINDS, hf.StrategyKind.HET_TMR)

    # the clock sampler starts during warm-up (nvidia-smi needs ~0.5 s to
    # emit its first sample) and stops right after the timed region
    sampler = ClockSampler(device) if rank == 0 else None
    if sampler:
        sampler.start()
    tmr.warm()

    # ---- timed region: device-resident inputs ----
    tmr.rt.executor._trace = tmr.on_trace
    barrier()
    torch.cuda.synchronize()
    launches0 = kernels.LAUNCHES
    t_dev, _ = tmr.timed(tmr.device_stream, args.steps, True)
    barrier()
    clocks = sampler.stop() if sampler else None
    launches = kernels.LAUNCHES - launches0
    tmr.rt.executor._trace = None
    t_max = max_over_ranks(t_dev)

    # ---- e2e: host buffers through the same API (H2D inside the stream, D2H read) ----
    # at least 80 steps: the pipeline fill (first 128 MiB H2D before any
    # kernel can start) and drain (last D2H) are paid once per timed region
    e2e_steps = args.e2e_steps or max(160, args.steps)
    tmr.host_stream(2)
    torch.cuda.synchronize()
    barrier()
    t_e2e, e2e_rounds = tmr.timed(tmr.host_stream, e2e_steps)
    barrier()
    t_e2e = max_over_ranks(t_e2e)

    # ---- BASELINE configs[1]: HetDMR, TC vs SIMT, detect-and-rerun (extra key) ----
    dmr = None
    if not args.no_dmr:
        dmr_b = TaskStreamBench(args, device, rank, DMR_KINDS, tmr.hf.StrategyKind.HET_DMR, seed_salt=13)
        dmr_b.warm()
        dmr_steps = max(30, args.steps)
        t_d, _ = dmr_b.timed(dmr_b.device_stream, dmr_steps, True)
        dmr_b.host_stream(2)
        t_de, de_rounds = dmr_b.timed(dmr_b.host_stream, e2e_steps)
        dmr = {"value": dmr_steps / t_d, "unit": "tasks/s", "steps": dmr_steps, "ms_per_task": 1e3 * t_d / dmr_steps,
               "workload": f"C2 (BASELINE configs[1]): HetDMR {n}x{n} fp32 matmul, tcgen05-TF32 vs SIMT-FP32, "
                           f"bit flips p={args.fault_prob}/replica, detect-and-rerun",
               "e2e": {"value": e2e_steps / t_de, "unit": "tasks/s", "steps": e2e_steps, "rounds": de_rounds,
                       "h2d_bytes_per_step": 2 * nb, "d2h_bytes_per_step": nb},
               "votes": dmr_b.stats["votes"], "rounds": dmr_b.stats["rounds"],
               "voter_gbs_in_task": (2 * nb * sum(dmr_b.stats["votes"].values())) / (dmr_b.stats["vote_ns"] * 1e-9) / 1e9
               if dmr_b.stats["vote_ns"] else None}
        del dmr_b

    # ---- kernel-level measurements (rank 0, after the timed regions) ----
    # the other ranks stop here: C3/C4 below drive GPUs 1.. from rank 0, so
    # every rank's own work on its GPU must have drained first
    total_tasks = args.steps * world
    torch.cuda.synchronize()
    barrier()
    if rank != 0:
        return
    kern = kernel_rooflines(device, n, kernels, torch)
    detect = detect_rate(device, n, kernels, torch, args.seed, probes=args.detect_probes)
    def extra(fn, *a, **kw):
        # multi-GPU extras must never cost the headline line: a failure is
        # reported in its key instead of ending rank 0 before it prints
        try:
            return fn(*a, **kw)
        except Exception as exc:  # noqa: BLE001
            return {"error": f"{type(exc).__name__}: {exc}"[:400]}

    pcie = extra(pcie_step_bound, torch, nb, device)
    if dmr is not None and pcie and "tasks_per_s" in pcie:
        dmr["e2e"]["pcie_bound_frac"] = dmr["e2e"]["value"] / pcie["tasks_per_s"]

    c4x = None
    if not args.no_c3:
        if world >= 2 and not shared_gpu and torch.cuda.device_count() >= 2:
            c4x = extra(c4_cross, args, torch, tuple(range(min(5, world, torch.cuda.device_count()))))
        elif args.c4_devices:
            c4x = extra(c4_cross, args, torch, tuple(int(x) for x in args.c4_devices.split(",")))
    c3 = None
    if not args.no_c3:
        if world >= 3 and not shared_gpu and torch.cuda.device_count() >= 3:
            c3 = extra(c3_rate, args, torch, devices=(0, 1, 2))
        elif args.c3_devices:       # code-path check, e.g. 0,0,0 on a one-GPU box
            c3 = extra(c3_rate, args, torch, devices=tuple(int(x) for x in args.c3_devices.split(",")))

    peaks, peak_src = load_peaks()
    stats = tmr.stats
    simt_ms, tc_ms, tc3_ms = tmr.kernel_ms("mm_simt"), tmr.kernel_ms("mm_tc"), tmr.kernel_ms("mm_tc3x")
    flops = 2.0 * n ** 3
    simt_tflops = flops / (simt_ms * 1e-3) / 1e12 if simt_ms else None
    sm_max = (clocks or {}).get("sm_max_mhz") or 1965.0
    ffma_peak, ffma_src = fp32_peak(sm_max)
    traffic = ncu_traffic("sgemm_128x128<32>", "transpose_a")
    vote_gbs = (3 * nb * sum(stats["votes"].values())) / (stats["vote_ns"] * 1e-9) / 1e9 if stats["vote_ns"] else None
    cpu = None
    if not args.no_cpu_baseline:
        tasks, secs, kind, detail = reference_tasks(n, args.cpu_sample_s, args.seed, by_time=True,
                                                    fault_prob=args.fault_prob)
        cpu = {"value": tasks / secs, "unit": "tasks/s", "cores": host_cores(), "kind": kind,
               "sample": f"{tasks} tasks in {secs:.1f} s: {detail}"}
    line = {
        "metric": METRIC,
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
        "config": bench_config(args, world),
        "e2e": {"value": (e2e_steps * world) / t_e2e, "unit": "tasks/s", "steps": e2e_steps,
                "rounds": e2e_rounds,
                "note": "own window of max(160, steps) tasks with their own fault draws; the H2D of "
                        "step i+2 and the D2H of step i-1 overlap step i (PCIe: 192 MiB per step)",
                "h2d_bytes_per_step": 2 * nb,
                "d2h_bytes_per_step": nb,
                # the step's PCIe traffic alone, measured live: the e2e ceiling
                "pcie_bound": dict(pcie, frac=((e2e_steps * world) / t_e2e) / (pcie["tasks_per_s"] * world))
                if pcie and "tasks_per_s" in pcie else pcie},
        "gpu_launches": launches,
        "clocks": clocks,
        "roofline": {"bound": "fp32-simt", "kernel": "hf_gemm_simt (incl. A^T pre-pass), in-task",
                     "achieved": simt_tflops, "peak": ffma_peak, "unit": "TFLOP/s",
                     "frac": (simt_tflops / ffma_peak) if simt_tflops else None, "traffic": traffic,
                     "traffic_unit": "DRAM bytes per launch (ncu --set full, GEMM + A^T pre-pass; "
                                     f"operand bytes 3*{n}^2*4 = {3 * nb})",
                     "peak_source": ffma_src,
                     "algorithmic": f"2*{n}^3 flop per launch",
                     "step_bound": {"simt_alone_ms": 1e3 * flops / (ffma_peak * 1e12),
                                    "tasks_per_s_at_peak": ffma_peak * 1e12 / flops,
                                    "frac": (total_tasks / t_max) / world / (ffma_peak * 1e12 / flops)}},
        "rooflines": kern,
        "replica_ms": {"mm_simt": simt_ms, "mm_tc": tc_ms, "mm_tc3x": tc3_ms},
        "voter_gbs_in_task": vote_gbs,
        "dmr": dmr,
        "c3": c3,
        "c4_cross_gpu": c4x,
        "detect": detect,
        "faults": {"injected": stats["injected"], "corrected_votes": stats["corrected"],
                   "mismatch_votes": stats["mismatch"], "votes": stats["votes"], "rounds": stats["rounds"]},
        "cpu_baseline": cpu,
        "peaks": {"source": peak_src, **peaks},
    }
    print(json.dumps(line), flush=True)


def pcie_step_bound(torch, nb: int, device: int, iters: int = 5):
    """The e2e step's host traffic alone on the copy engines: 2 x nb H2D on one
    stream while nb D2H runs on another (pinned buffers), best of `iters`.
    1 / that time bounds the e2e rate whatever the GPU does (tools/pcie_bw.py)."""
    with torch.cuda.device(device):
        hin = torch.empty(2 * nb, dtype=torch.uint8).pin_memory()
        hout = torch.empty(nb, dtype=torch.uint8).pin_memory()
        din = torch.empty(2 * nb, dtype=torch.uint8, device=f"cuda:{device}")
        dout = torch.empty(nb, dtype=torch.uint8, device=f"cuda:{device}")
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        best = None
        for _ in range(iters + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            with torch.cuda.stream(s_in):
                din[:nb].copy_(hin[:nb], non_blocking=True)
                din[nb:].copy_(hin[nb:], non_blocking=True)
            with torch.cuda.stream(s_out):
                hout.copy_(dout, non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        del hin, hout, din, dout
    return {"step_ms": best * 1e3, "tasks_per_s": 1.0 / best,
            "shape": f"2 x {nb >> 20} MiB H2D + {nb >> 20} MiB D2H at once, pinned, copy engines"}


def p2p_peak(src_dev: int, dst_dev: int, torch, nbytes: int = 1 << 30):
    """NVLink P2P roofline denominator, measured: hf_copy of `nbytes` from
    src_dev's HBM into dst_dev's (the copy kernel on dst_dev pulling peer
    loads, the voter's access pattern), CUDA-event timed on dst_dev after
    warm-up; best of 5.  GB/s of NVLink ingress into dst_dev."""
    from paper_1405_2912_b200 import _lib, kernels
    _lib.enable_peers()
    if not _lib.peer_enabled(dst_dev, src_dev):
        return None
    src = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{src_dev}")
    dst = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{dst_dev}")
    src.fill_(1)
    torch.cuda.synchronize(src_dev)
    st = torch.cuda.Stream(device=dst_dev)
    best = None
    with torch.cuda.device(dst_dev):
        for it in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            kernels.copy(dst, src, stream=st)
            e1.record(st)
            st.synchronize()
            if it >= 2:
                t = e0.elapsed_time(e1) * 1e-3
                best = t if best is None else min(best, t)
    return nbytes / best / 1e9


def c4_cross(args, torch, devices):
    """BASELINE configs[3] across GPUs: K replicas of 64 MiB / 256 MiB / 1 GiB
    on `devices` (one per replica), voted sliced over them
    (CudaBackend._vote_sliced_start: each GPU votes 1/K of the elements,
    loading the other K-1 replicas' slices from their peers), K = 2..min(5,
    GPUs).  Reports the vote time (max of the slices' own kernel clocks and
    the CUDA events on the lead GPU) and each GPU's NVLink ingress rate,
    (K-1)/K * n * 4 bytes / time, against the measured P2P peak."""
    import paper_1405_2912_b200 as hf
    from paper_1405_2912_b200.backend import CudaBackend
    try:
        be = CudaBackend()
        peak = p2p_peak(devices[1], devices[0], torch) if len(set(devices)) > 1 else None
        rows = []
        for mib in (64, 256, 1024):
            for K in range(2, min(5, len(devices)) + 1):
                n = mib << 18
                devs = devices[:K]
                bufs = []
                for d in devs:
                    g = torch.Generator(device=f"cuda:{d}")
                    g.manual_seed(17)
                    bufs.append((torch.rand(n, device=f"cuda:{d}", generator=g) + 1).view(torch.uint8))
                for d in set(devs):
                    torch.cuda.synchronize(d)
                ts = []
                for it in range(6):
                    h = be.vote_start(bufs, hf.ValueType.FLOAT32, 4, [1e-3] * K)
                    res, ns = h.wait()
                    assert res.verdict == "match"
                    if it >= 2:
                        ts.append(ns)
                t = sorted(ts)[len(ts) // 2] * 1e-9
                ingress = (K - 1) / K * n * 4
                rows.append({"mib": mib, "K": K, "devices": list(devs), "vote_us": t * 1e6,
                             "nvlink_ingress_gbs_per_gpu": ingress / t / 1e9 if len(set(devs)) > 1 else None,
                             "frac_p2p_peak": (ingress / t / 1e9 / peak) if peak and len(set(devs)) > 1 else None,
                             "replica_read_gbs": K * n * 4 / t / 1e9})
                del bufs
        return {"p2p_peak_gbs": peak, "peak_source": "measured: hf_copy 1 GiB peer pull (bench.p2p_peak)",
                "rows": rows}
    except Exception as exc:  # noqa: BLE001 - reported, the headline line still prints
        return {"error": f"{type(exc).__name__}: {exc}"}


def c3_rate(args, torch, devices=(0, 1, 2)):
    """BASELINE configs[2]: HetTMR n x n with the three replicas on three
    distinct GPUs (fleets.b200_replica_fleet_config: SIMT FP32 on GPU 0 with
    the inputs, tcgen05 TF32 on GPU 1, tcgen05 3xBF16 on GPU 2;
    Strategy(spread="device")), inputs device-resident on GPU 0 and pulled by
    the other replicas over NVLink, the K = 3 vote sliced over the three GPUs
    (each votes a third, loading the other replicas' thirds from their
    peers), in-place into the SIMT replica.  CUDA-event timed on every GPU's
    compute stream; the max over the GPUs is the time.  Also reports the
    sliced vote's per-GPU NVLink ingress rate against a measured P2P peak."""
    import paper_1405_2912_b200 as hf
    n = args.n
    nb = n * n * 4
    try:
        cfg = hf.b200_replica_fleet_config(devices=devices)
        for u in cfg["units"]:
            u.update({"corrupt_prob": args.fault_prob, "corrupt_mode": "bitflip",
                      "seed": args.seed * 1_000_003 + u["seed"]})
        rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(checkpoint_space="ckpt", serial_replicas=True,
                                                             attempt_limit=64))
        task = hf.get_workload("matmul").attach(rt, kinds=TMR_KINDS)
        # one replica per GPU (on a box without three GPUs, devices may repeat:
        # the one-variant-per-space fleet still forces one replica per space)
        spread = "device" if len(set(devices)) == len(devices) else "unit"
        b = TaskStreamBench(args, devices[0], 0, TMR_KINDS, hf.Strategy(hf.StrategyKind.HET_TMR, spread=spread),
                            built=(hf, rt, task), space="r0mem")
        rt.executor._trace = b.on_trace
        b.warm()
        steps = max(30, args.steps)
        devs = sorted(set(devices))
        for d in devs:
            torch.cuda.synchronize(d)
        starts, ends = {}, {}
        for d in devs:
            starts[d] = torch.cuda.Event(enable_timing=True)
            starts[d].record(rt.backend.stream(d))
        b.device_stream(steps, True)
        for d in devs:
            ends[d] = torch.cuda.Event(enable_timing=True)
            ends[d].record(rt.backend.stream(d))
        for d in devs:
            torch.cuda.synchronize(d)
        t = max(starts[d].elapsed_time(ends[d]) for d in devs) * 1e-3
        st = b.stats
        votes = sum(st["votes"].values())
        vote_s = st["vote_ns"] * 1e-9 / votes if votes else None
        K = 3
        ingress = (K - 1) / K * nb            # NVLink bytes into each voting GPU per vote
        peak = p2p_peak(devices[1], devices[0], torch) if len(devs) > 1 else None
        vote_gbs = ingress / vote_s / 1e9 if vote_s and len(devs) > 1 else None
        return {"value": steps / t, "unit": "tasks/s", "steps": steps, "ms_per_task": 1e3 * t / steps,
                "devices": list(devices),
                "workload": f"HetTMR {n}x{n}, replicas on GPUs {list(devices)} (SIMT / TF32 / 3xBF16), inputs "
                            f"on GPU {devices[0]} pulled over NVLink, vote sliced over the replica GPUs",
                "votes": st["votes"], "rounds": st["rounds"],
                "replica_ms": {k: b.kernel_ms(k) for k in ("mm_simt", "mm_tc", "mm_tc3x")},
                "vote_us": vote_s * 1e6 if vote_s else None,
                "nvlink": {"bytes_per_gpu_per_vote": ingress, "achieved_gbs": vote_gbs,
                           "peak_gbs": peak, "frac": (vote_gbs / peak) if vote_gbs and peak else None,
                           "peak_source": f"measured: hf_copy GPU{devices[1]}->GPU{devices[0]} 1 GiB pull, "
                                          "best of 5 (bench.p2p_peak)",
                           "input_bytes_per_task": 2 * 2 * nb}}
    except Exception as exc:  # noqa: BLE001 - reported, the headline line still prints
        return {"error": f"{type(exc).__name__}: {exc}"}


_FP32_PEAK = None


def fp32_peak(sm_max_mhz: float):
    """Cached: the probe runs once per bench process."""
    global _FP32_PEAK
    if _FP32_PEAK is None:
        _FP32_PEAK = _fp32_peak(sm_max_mhz)
    return _FP32_PEAK


def _fp32_peak(sm_max_mhz: float):
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
                                       f"issued a-scalar-outer it peaks at {d['ffma2_bcast_tflops']:.1f}; the "
                                       "8x16 column-pair-outer GEMM loop reaches ~0.90 of the loop figure at "
                                       "exact-wave shapes, tools/simt_fullwave.py)")
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

    def vote_kernel_s(ws):
        # the vote kernel's own clock (hf_vote_result.kernel_ns) of the last launch
        return ws.read().kernel_ns * 1e-9

    m = n * n
    base = torch.rand(m, device=d) + 1
    reps = [base * (1 + 1e-6 * torch.randn(m, device=d)) for _ in range(3)]
    kernels.inject_bitflip(reps[2], m // 3, 27, stream=st)
    ws = kernels.VoteWorkspace(device, stream=st)
    for K in (2, 3):
        t = time_it(lambda: kernels.vote_async(reps[:K], ws, 1e-3, voted=reps[0] if K >= 3 else None, stream=st))
        byts = K * m * 4      # replica reads; the in-place voted output stores only differing vectors
        tk = vote_kernel_s(ws)
        out[f"hf_vote_K{K}"] = {"bound": "hbm", "achieved": byts / t / 1e9, "peak": peaks["hbm_gbs"],
                                "unit": "GB/s", "frac": byts / t / 1e9 / peaks["hbm_gbs"],
                                "us": t * 1e6, "algorithmic_bytes": byts,
                                "kernel_us": tk * 1e6, "frac_kernel_clock": byts / tk / 1e9 / peaks["hbm_gbs"]
                                if tk > 0 else None,
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
    ffma_peak, _src = fp32_peak(1965.0)
    out["hf_gemm_simt"] = {"bound": "fp32-simt", "achieved": 2 * n ** 3 / t / 1e12, "unit": "TFLOP/s",
                           "peak": ffma_peak, "frac": 2 * n ** 3 / t / 1e12 / ffma_peak, "us": t * 1e6,
                           "note": "standalone (alone on the GPU, incl. the A^T pre-pass); the headline "
                                   "roofline is the same kernel in-task, sharing SMs with two TC replicas"}
    return out


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    run_hetft_arm(args, rank, world, local)


if __name__ == "__main__":
    main()
