"""Lab (not product code): how much of a HetTMR 4096^2 task's serial prologue
(vote of the previous task -> input checkpoints -> pre-passes -> SIMT grid)
can overlap the previous task's tensor-core tail, by stream structure alone.
Raw libhetft kernels on the streams the runtime uses, a host that waits for
task i-1's vote before queueing task i+1 (TaskStream depth 1):

  serial     vote on the device's compute stream; the next task's
             checkpoints and replicas queue behind it (the runtime today)
  vote_side  vote on its own stream; replicas wait only for their own
             task's checkpoints (compute stream)
  no_ckpt    vote on its own stream and waits for the checkpoints; replicas
             wait for nothing of the compute stream

    python tools/pipeline_lab.py [tasks] [n]
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1405_2912_b200 import kernels  # noqa: E402
from paper_1405_2912_b200._lib import HF_GEMM_COSCHEDULE as CO, HF_GEMM_TF32, HF_GEMM_3XBF16  # noqa: E402

tasks = int(sys.argv[1]) if len(sys.argv) > 1 else 40
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
d = "cuda:0"
A = torch.rand(n, n, device=d) + 1
B = torch.rand(n, n, device=d) + 1
pool = [[torch.empty(n, n, device=d) for _ in range(3)] for _ in range(4)]
ck = [torch.empty(n * n * 4, dtype=torch.uint8, device=d) for _ in range(2)]
compute = torch.cuda.Stream(device=d)
s_simt = torch.cuda.Stream(device=d, priority=-1)
s_tc = torch.cuda.Stream(device=d)
s_tc3 = torch.cuda.Stream(device=d)
s_vote = torch.cuda.Stream(device=d)
ws = [kernels.VoteWorkspace(0) for _ in range(4)]


def one(i, mode):
    cs = pool[i % 4]
    # input checkpoints on the compute stream (memory.py _maybe_checkpoint)
    kernels.checkpoint(ck[0], A.view(torch.uint8).view(-1), stream=compute)
    kernels.checkpoint(ck[1], B.view(torch.uint8).view(-1), stream=compute)
    if mode != "no_ckpt":
        ev = torch.cuda.Event()
        ev.record(compute)
        for s in (s_simt, s_tc, s_tc3):
            s.wait_event(ev)
    kernels.gemm_simt(A, B, cs[0], mode=CO, stream=s_simt)
    kernels.gemm_tc(A, B, cs[1], mode=HF_GEMM_TF32 | CO, stream=s_tc)
    kernels.gemm_tc(A, B, cs[2], mode=HF_GEMM_3XBF16 | CO, stream=s_tc3)
    vs = compute if mode == "serial" else s_vote
    for s in (s_simt, s_tc, s_tc3) + ((compute,) if mode == "no_ckpt" else ()):
        vs.wait_stream(s)
    kernels.vote_async([cs[1], cs[0], cs[2]], ws[i % 4], 1e-3, voted=cs[0], stream=vs)
    ev = torch.cuda.Event(enable_timing=True)
    ev.record(vs)
    return ev


def run(mode):
    evs = []
    for i in range(4):
        evs.append(one(i, mode))
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(compute)
    wall = time.perf_counter()
    evs = []
    for i in range(tasks):
        evs.append(one(i, mode))
        if len(evs) >= 2:
            evs[-2].synchronize()       # depth 1: task i-1 settles after task i is queued
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall
    ms = t0.elapsed_time(evs[-1])
    return {"mode": mode, "tasks": tasks, "ms_per_task": ms / tasks, "tasks_per_s": tasks / (ms * 1e-3),
            "wall_tasks_per_s": tasks / wall}


if __name__ == "__main__":
    for rep in range(2):
        for mode in ("serial", "vote_side", "no_ckpt"):
            print(json.dumps(run(mode)), flush=True)
