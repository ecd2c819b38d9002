"""BASELINE config C5: a batched stream of voted matmul tasks with random
fault injection and checkpoint rollback, sharded over the GPUs of one box.

Each rank (one process per GPU, launched by torchrun for N > 1) owns the
tasks t with t mod world == rank (sharding.tasks_for_rank) and runs them
through the drop-in Runtime's TaskStream on its own GPU: HetTMR of the three
diverse variants (tcgen05 TF32, SIMT FP32, tcgen05 3xBF16; one logical unit
each, sharing the GPU's memory space), protected attempts checkpoint their
device-resident inputs into an HBM reserve space, every unit draws faults
from its own seeded stream — bit-flip corruption (caught or masked by the
majority vote) and aborts (scribble + rollback: the attempt's siblings are
invalidated and the retry restores A and B from the checkpoint).

Every committed C is verified on the GPU against the binary64 product of its
inputs (an hf_vote K = 2 under the task's δ must return "match"), inside the
timed region, so the rate includes that check; the checks run asynchronously
on the compute stream (a ring of pinned result slots, read when a slot comes
round again and before the timed region closes).  There is no data-path
collective: ranks meet only for the barrier, the max of the device times and
the sum of the counters (NCCL).

    python tools/stream_c5.py --tasks 10000                   # 1 GPU
    torchrun --nproc-per-node 8 tools/stream_c5.py --tasks 10000

Writes one JSON line (rank 0) to stdout and, with --out, to a file.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tasks", type=int, default=10000, help="tasks in the whole job (all ranks)")
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--strategy", default="hettmr", choices=("hettmr", "hetdmr"))
    ap.add_argument("--corrupt-prob", type=float, default=0.05, help="per replica attempt, bit-flip mode")
    ap.add_argument("--abort-prob", type=float, default=0.01, help="per replica attempt (scribble + rollback)")
    ap.add_argument("--inputs", type=int, default=8, help="distinct (A, B) input pairs cycled over the tasks")
    ap.add_argument("--depth", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--gc", choices=("default", "freeze", "off"), default="default",
                    help="Python cyclic GC during the timed region: as is, gc.freeze() after warm-up, or disabled")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--out", default=None)
    return ap.parse_args()


def main():
    args = parse()
    import torch.distributed as dist
    import paper_1405_2912_b200 as hf
    from paper_1405_2912_b200 import _lib, kernels, sharding

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = local if torch.cuda.device_count() > local else 0
    torch.cuda.set_device(dev)
    shared_gpu = torch.cuda.device_count() < world      # code-path check: ranks share a GPU -> gloo
    if world > 1:
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))

    n, nn = args.n, args.n * args.n
    kinds = ("gpu-tc", "gpu-simt", "gpu-tc3") if args.strategy == "hettmr" else ("gpu-tc", "gpu-simt")
    cfg = hf.gpu_fleet_config(devices=(dev,), kinds=kinds)
    cfg["memory_spaces"].append({"id": f"gpu{dev}ckpt", "device": dev, "label": "HBM checkpoint reserve"})
    for i, u in enumerate(cfg["units"]):
        u.update({"corrupt_prob": args.corrupt_prob, "abort_prob": args.abort_prob, "corrupt_mode": "bitflip",
                  "seed": args.seed * 1_000_003 + rank * 10_007 + i * 101 + 17})
    rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(checkpoint_space=f"gpu{dev}ckpt", serial_replicas=True,
                                                         attempt_limit=64))
    task = hf.get_workload("matmul").attach(rt, kinds=kinds)
    strat = hf.Strategy(hf.StrategyKind.HET_TMR if args.strategy == "hettmr" else hf.StrategyKind.HET_DMR)
    space = f"gpu{dev}mem"
    d = f"cuda:{dev}"

    # inputs U[1,2) (reference distribution) and their binary64 products
    pairs, refs = [], []
    for j in range(args.inputs):
        g = np.random.default_rng(args.seed * 7919 + 131 * j)
        a = g.random((n, n), dtype=np.float32) + np.float32(1)
        b = g.random((n, n), dtype=np.float32) + np.float32(1)
        c = (a.astype(np.float64) @ b.astype(np.float64)).astype(np.float32)
        pairs.append((torch.from_numpy(a).view(-1).view(torch.uint8).to(d),
                      torch.from_numpy(b).view(-1).view(torch.uint8).to(d)))
        refs.append(torch.from_numpy(c).view(-1).to(d))
    hz = torch.zeros(nn * 4, dtype=torch.uint8).pin_memory()
    mine = sharding.tasks_for_rank(args.tasks, rank, world)

    cnt = {"tasks": 0, "rounds": 0, "attempts": 0, "injected_bitflips": 0, "aborts": 0, "api_errors": 0,
           "timeouts": 0, "vote_mismatch": 0, "votes_match": 0, "votes_corrected": 0, "votes_mismatch": 0,
           "verify_fail": 0}

    # verification of every committed C against its binary64 product, on the
    # GPU and asynchronous: hf_vote_async on the runtime's compute stream
    # (ordered after the task's vote; the caching allocator cannot reuse C
    # before it), results into a ring of pinned slots checked when a slot
    # comes round again and at the end — no host sync per task
    vstream = rt.backend.stream(dev)
    ring = [(kernels.VoteWorkspace(dev, stream=vstream),
             torch.empty(ctypes.sizeof(_lib.HfVoteResult), dtype=torch.uint8).pin_memory()) for _ in range(64)]
    pending = {}

    def check_slot(i):
        ev = pending.pop(i, None)
        if ev is not None:
            ev.synchronize()
            r = kernels.VoteResult.from_c(_lib.HfVoteResult.from_buffer_copy(ring[i][1].numpy().tobytes()))
            cnt["verify_fail"] += int(r.verdict != "match")

    def account(rep, j, ic):
        c = rt.read_tensor(ic).view(torch.float32)
        i = cnt["tasks"] % len(ring)
        check_slot(i)
        kernels.vote_async([c, refs[j]], ring[i][0], 1e-3, stream=vstream, result_into=ring[i][1])
        ev = torch.cuda.Event()
        ev.record(vstream)
        pending[i] = ev
        cnt["tasks"] += 1
        cnt["rounds"] += rep.rounds
        cnt["attempts"] += rep.attempts
        cnt["injected_bitflips"] += len(rep.injected)
        cnt["aborts"] += rep.fault_counts.get("abort", 0)
        cnt["api_errors"] += rep.fault_counts.get("api_error", 0)
        cnt["timeouts"] += rep.fault_counts.get("timeout", 0)
        cnt["vote_mismatch"] += rep.fault_counts.get("vote_mismatch", 0)
        for v in rep.votes:
            cnt["votes_" + v] = cnt.get("votes_" + v, 0) + 1

    def run(ts_ids, record):
        queue = []
        with rt.task_stream(depth=args.depth) as ts:
            for t in ts_ids:
                j = t % args.inputs
                ia = rt.register_device_data(pairs[j][0], nn, hf.ValueType.FLOAT32, "r", space)
                ib = rt.register_device_data(pairs[j][1], nn, hf.ValueType.FLOAT32, "r", space)
                # the output area as reference programs register it (host zeros,
                # never read by a "w" request; not a sole device copy, so no
                # checkpoint of C) — as bench.py does
                ic = rt.register_host_buffer(hz, nn, hf.ValueType.FLOAT32, "w")
                queue.append((ts.submit(task, {"A": ia, "B": ib, "C": ic, "n": n}, strat), j, (ia, ib, ic)))
                while queue and queue[0][0].success:
                    rep, jj, areas = queue.pop(0)
                    if record:
                        account(rep, jj, areas[2])
                    for x in areas:
                        rt.release(x)
        for rep, jj, areas in queue:
            if not rep.success:
                raise RuntimeError("task failed (attempt budget exhausted)")
            if record:
                account(rep, jj, areas[2])
            for x in areas:
                rt.release(x)

    run(range(args.warmup), False)
    for i in list(pending):
        check_slot(i)
    cnt["verify_fail"] = 0
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    st = rt.backend.stream(dev)
    import gc
    if args.gc == "freeze":
        gc.collect()
        gc.freeze()
    elif args.gc == "off":
        gc.collect()
        gc.disable()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record(st)
    run(mine, True)
    for i in list(pending):
        check_slot(i)
    e1.record(st)
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    gc.enable()
    t_dev = e0.elapsed_time(e1) * 1e-3
    keys = sorted(cnt)
    cd = "cpu" if shared_gpu else d
    vec = torch.tensor([cnt[k] for k in keys], dtype=torch.int64, device=cd)
    tmax = torch.tensor([t_dev], dtype=torch.float64, device=cd)
    if world > 1:
        dist.barrier()
        dist.all_reduce(vec)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    tot = dict(zip(keys, (int(x) for x in vec.tolist())))
    t_job = float(tmax.item())
    if rank == 0:
        line = {"metric": f"voted tasks/sec ({args.strategy.upper()} {n}^2 fp32 matmul task stream)",
                "value": tot["tasks"] / t_job, "unit": "tasks/s", "n_gpus": world, "tasks": tot["tasks"],
                "seconds": t_job, "wall_s_rank0": wall, "scaling": "weak (tasks sharded t mod world)",
                "config": {"workload": f"C5: {args.tasks} {args.strategy} tasks {n}x{n}, HBM checkpoint of "
                                       f"inputs, bit flips p={args.corrupt_prob}, aborts p={args.abort_prob} "
                                       f"per replica attempt", "inputs": args.inputs, "depth": args.depth, "gc": args.gc},
                "counts": tot,
                "verify": "every committed C == binary64 A·B under the voter predicate (δ=1e-3), "
                          f"{tot['tasks'] - tot['verify_fail']}/{tot['tasks']} pass"}
        print(json.dumps(line), flush=True)
        if args.out:
            Path(args.out).parent.mkdir(parents=True, exist_ok=True)
            Path(args.out).write_text(json.dumps(line, indent=1))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
