"""Multi-GPU placement logic, CPU side.

* slicing + exact recombination of K-way votes equals the unsliced oracle vote
* task ownership / replica-group rotation
* world_size-2 gloo run of the N > 1 path: each rank votes its slice and runs
  its shard of a task stream; gathered results equal the single-process ones
"""

import os
import random

import numpy as np
import pytest

from oracle import inject as oinject
from oracle import vote as ovote
from paper_1405_2912_b200 import sharding


def _replicas(seed, K, n, faults):
    rng = np.random.default_rng(seed)
    base = rng.uniform(1, 2, n).astype(np.float32)
    reps = [base.copy() for _ in range(K)]
    for _ in range(faults):
        oinject.bitflip(reps[int(rng.integers(0, K))], int(rng.integers(0, n)), int(rng.integers(10, 32)))
    return reps


def _slice_vote(reps, parts, delta=1e-3):
    out = []
    for lo, hi in sharding.slice_bounds(reps[0].size, parts):
        if hi <= lo:
            continue
        r = ovote.vote([x[lo:hi] for x in reps], delta)
        out.append(sharding.SliceResult(lo, r.mismatch, r.unresolved, r.first_div))
    return out


@pytest.mark.parametrize("K", [2, 3, 5])
@pytest.mark.parametrize("parts", [1, 2, 3, 7])
@pytest.mark.parametrize("n", [1, 5, 1000, 4099])
def test_sliced_vote_recombines_exactly(K, parts, n):
    reps = _replicas(K * 100 + parts + n, K, n, max(1, n // 300))
    full = ovote.vote(reps, 1e-3)
    comb = sharding.combine_slices(_slice_vote(reps, parts), K)
    assert (comb.verdict, comb.mismatch, comb.unresolved, comb.first_div, comb.winner) == \
        (full.verdict, full.mismatch, full.unresolved, full.first_div, full.winner)


def test_slice_bounds_cover_and_align():
    for n in (0, 1, 3, 4, 17, 4096, 4099):
        for parts in (1, 2, 3, 8):
            b = sharding.slice_bounds(n, parts)
            assert len(b) == parts
            assert b[0][0] == 0 and b[-1][1] == n
            for (lo, hi), (lo2, _) in zip(b, b[1:]):
                assert hi == lo2 and (lo % 4 == 0 or lo == n)


def test_task_ownership_and_replica_rotation():
    world = 8
    owned = [sharding.tasks_for_rank(10_000, r, world) for r in range(world)]
    assert sorted(t for o in owned for t in o) == list(range(10_000))
    assert max(map(len, owned)) - min(map(len, owned)) <= 1
    load = [0] * world
    for t in range(10_000):
        g = sharding.replica_group(t, world, 3)
        assert len(set(g)) == 3
        for d in g:
            load[d] += 1
    assert max(load) - min(load) <= 3          # K/G of the replica load per GPU


# ---- world_size 2, gloo --------------------------------------------------------------

def _worker(rank, world, port, result_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path
        here = Path(__file__).resolve().parent
        sys.path[:0] = [str(here), str(here.parent)]
        import paper_1405_2912_b200 as hf
        from host_backend import HostBackend

        # (1) sliced vote: this rank votes its slice, all slices are gathered
        reps = _replicas(7, 3, 5000, 12)
        lo, hi = sharding.slice_bounds(5000, world)[rank]
        r = ovote.vote([x[lo:hi] for x in reps], 1e-3)
        mine = sharding.SliceResult(lo, r.mismatch, r.unresolved, r.first_div)
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        comb = sharding.combine_slices(gathered, 3)

        # (2) independent task stream shard (DMR, seeded corruption)
        cfg = {"default_ns_per_byte": 0.01, "memory_spaces": [{"id": "host", "host": True},
                                                               {"id": "g1"}, {"id": "g2"}],
               "units": [{"id": "u1", "kind": "gpu", "memory_space": "g1", "seed": 11 + rank,
                          "corrupt_prob": 0.3, "corrupt_rel_magnitude": 0.5},
                         {"id": "u2", "kind": "gpu", "memory_space": "g2", "seed": 23 + rank}]}
        rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(serial_replicas=True), backend=HostBackend())
        task = rt.declare_task("inc", (hf.Param.area("input", "r"), hf.Param.area("output", "w"),
                                       hf.Param.scalar("count")))

        def inc(ctx):
            n = ctx.arg("count")
            np.add(ctx.request("input", "r")[:n], np.float32(1.0), out=ctx.request("output", "w")[:n])

        rt.attach_kernel(task, "inc", "gpu", inc)
        mismatches = 0
        mine_tasks = sharding.tasks_for_rank(20, rank, world)
        for t in mine_tasks:
            data = np.full(64, t, dtype=np.float32)
            i = rt.register_data(data.tobytes(), 64, hf.ValueType.FLOAT32, "r")
            o = rt.register_data(bytes(256), 64, hf.ValueType.FLOAT32, "w")
            rep = rt.invoke(task, {"input": i, "output": o, "count": 64}, hf.Strategy(hf.StrategyKind.DMR))
            mismatches += rep.fault_counts["vote_mismatch"]
            assert np.array_equal(rt.read_array(o), data + 1)
        total_tasks = sharding.sum_over_ranks(float(len(mine_tasks)))
        t_max = sharding.max_over_ranks(float(rank + 1))
        result_q.put((rank, comb.verdict, comb.mismatch, comb.first_div, total_tasks, t_max, mismatches))
    finally:
        dist.destroy_process_group()


def test_world_size_two_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.Random(os.getpid()).randrange(2000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = sorted(q.get(timeout=5) for _ in range(2))
    full = ovote.vote(_replicas(7, 3, 5000, 12), 1e-3)
    for rank, verdict, mism, first, total, tmax, _ in res:
        assert (verdict, mism, first) == (full.verdict, full.mismatch, full.first_div)
        assert total == 20.0 and tmax == 2.0
