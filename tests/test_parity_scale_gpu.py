"""Parity at the sizes and shapes the benchmarks actually run.

1. C4 (BASELINE configs[3]) vote sizes: K = 2..5 replicas of 256 MiB, 1 GiB
   and 4 GiB + 64 KiB + 12 B fp32 buffers (the last one ragged, with element
   byte offsets beyond 2^32).  Replicas are diverse (1e-6 relative noise, as
   between TC and SIMT outputs, so the fp32 screen decides every element)
   with bit flips planted in the first vector, the last full vector, the
   scalar tail, just past byte 2^32, on both sides of a 2^31 element
   boundary and at random positions; for K = 4 a 2-vs-2 split makes one
   element unresolved.  The vote is element-wise, so
   the oracle (oracle/vote.py) runs on windows around every planted fault;
   every other element provably agrees (|noise| < 1e-5 << δ) and must keep
   replica 0's bytes.  Global counts, first divergence, winner, verdict and
   the voted bytes (windows on the host, the rest compared on the device
   against a saved copy) must equal the oracle's.
2. The benchmark's own task shape: HetDMR and HetTMR of a 4096^2 fp32 matmul
   through the Runtime with bit-flip faults at p = 0.05 per replica, >= 30
   tasks each.  Every round's fault coordinates equal the oracle's draw
   order (oracle/fault_schedule.py; reference devices.py:144-220), every
   faulty replica's bytes equal its variant's clean output with exactly
   that bit flipped, and every vote's verdict / counts / first divergence
   equal oracle.vote on D2H copies of the replicas taken right before the
   vote (reference voting.py:68-123 at K = 2).
"""

import random

import numpy as np
import pytest

from oracle import fault_schedule
from oracle import matmul as omatmul
from oracle import vote as ovote

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_1405_2912_b200 as hf  # noqa: E402
from paper_1405_2912_b200 import kernels  # noqa: E402

MiB = 1 << 20
WIN = 4096


def _plant(n, K, seed):
    """(replica, element, bit) flips; returns the list and the window starts."""
    rng = random.Random(seed)
    last_vec = (n // 4 - 1) * 4
    spots = [0, 3, last_vec, last_vec + 3, n - 1, n - 2, n // 2, (1 << 29) - 1, 1 << 29]
    if n * 4 > (1 << 32) + 64:
        spots += [(1 << 30) + 1, (1 << 30) + 4]          # byte offsets > 2^32
    spots += [rng.randrange(n) for _ in range(6)]
    flips = []
    for i, e in enumerate(s for s in spots if s < n):
        flips.append((i % K, e, rng.choice([23, 27, 30, 31, 25])))
    return flips


@pytest.mark.parametrize("nbytes", [256 * MiB, 1024 * MiB, 4096 * MiB + 64 * 1024 + 12],
                         ids=["256MiB", "1GiB", "4GiB+ragged"])
@pytest.mark.parametrize("K", [2, 3, 4, 5])
def test_c4_vote_parity(nbytes, K):
    n = nbytes // 4
    g = torch.Generator(device="cuda")
    g.manual_seed(K * 1000 + n % 997)
    base = torch.rand(n, device="cuda", generator=g) + 1
    reps = []
    for _ in range(K):
        noise = torch.randn(n, device="cuda", generator=g).clamp_(-6, 6)
        reps.append((base * (1 + 1e-6 * noise)).contiguous())
        del noise
    del base
    flips = _plant(n, K, seed=K + n)
    for r, e, bit in flips:
        kernels.inject_bitflip(reps[r], e, bit)
    unres_elem = None
    if K == 4:     # 2-vs-2 split: replicas 0,1 vs 2,3 (same flip in both) -> no majority
        unres_elem = n // 3
        kernels.inject_bitflip(reps[2], unres_elem, 30)
        kernels.inject_bitflip(reps[3], unres_elem, 30)
    torch.cuda.synchronize()
    # windows around every planted element, merged
    centers = sorted({e for _, e, _ in flips} | ({unres_elem} if unres_elem is not None else set()))
    wins = []
    for c in centers:
        lo, hi = max(0, c - WIN // 2), min(n, c + WIN // 2)
        if wins and lo <= wins[-1][1]:
            wins[-1] = (wins[-1][0], max(wins[-1][1], hi))
        else:
            wins.append((lo, hi))
    host = {(lo, hi): [r[lo:hi].cpu().numpy() for r in reps] for lo, hi in wins}
    saved0 = reps[0].clone() if K >= 3 else None
    voted = reps[0] if K >= 3 else None
    res = kernels.vote(reps, 1e-3, voted=voted)
    torch.cuda.synchronize()
    mism, unres, first = [0] * K, 0, -1
    for (lo, hi), xs in host.items():
        o = ovote.vote(xs, 1e-3)
        mism = [a + b for a, b in zip(mism, o.mismatch)]
        unres += o.unresolved
        if o.first_div >= 0 and first < 0:
            first = lo + o.first_div
        if voted is not None:
            assert voted[lo:hi].cpu().numpy().tobytes() == o.voted.tobytes()
            saved0[lo:hi] = voted[lo:hi]      # windows checked; the rest must be untouched
    winner = min(range(K), key=lambda r: (mism[r], r))
    verdict = "mismatch" if unres else ("corrected" if any(mism) else "match")
    if K == 2:
        verdict = "mismatch" if any(mism) else "match"
    assert (res.verdict, res.mismatch, res.unresolved, res.first_div, res.winner) == \
        (verdict, mism, unres, first, winner)
    assert sum(mism) >= len(flips)          # every planted flip is a detectable disagreement
    if voted is not None:
        assert torch.equal(voted, saved0)


# ---- the benchmark's task shape ------------------------------------------------------

N = 4096


@pytest.fixture(scope="module")
def mm_operands():
    a, b = omatmul.make_inputs(N, seed=21)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    clean = {}
    # launch shapes of replicas sharing one GPU (co-scheduling flag): these
    # are the exact bytes each variant produces inside a task
    co = hf._lib.HF_GEMM_COSCHEDULE
    for kernel, fn in (("mm_simt", lambda c: kernels.gemm_simt(ta, tb, c, mode=co)),
                       ("mm_tc", lambda c: kernels.gemm_tc(ta, tb, c, mode=hf._lib.HF_GEMM_TF32 | co)),
                       ("mm_tc3x", lambda c: kernels.gemm_tc(ta, tb, c, mode=hf._lib.HF_GEMM_3XBF16 | co))):
        c = torch.empty(N, N, device="cuda")
        fn(c)
        clean[kernel] = c.cpu().numpy().reshape(-1)
    return ta, tb, clean


@pytest.mark.parametrize("strategy,kinds,tasks,p", [
    (hf.StrategyKind.HET_DMR, ("gpu-tc", "gpu-simt"), 30, 0.05),
    (hf.StrategyKind.HET_TMR, ("gpu-tc", "gpu-simt", "gpu-tc3"), 30, 0.05),
    (hf.StrategyKind.HET_TMR, ("gpu-tc", "gpu-simt", "gpu-tc3"), 8, 0.4),
], ids=["hetdmr-p0.05", "hettmr-p0.05", "hettmr-p0.4"])
def test_bench_shape_runtime_replay(mm_operands, strategy, kinds, tasks, p):
    ta, tb, clean = mm_operands
    cfg = hf.gpu_fleet_config(devices=(0,), kinds=kinds)
    cfg["memory_spaces"].append({"id": "gpu0ckpt", "device": 0})
    for i, u in enumerate(cfg["units"]):
        u.update({"corrupt_prob": p, "corrupt_mode": "bitflip", "seed": 7_000_003 + i * 101})
    rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(checkpoint_space="gpu0ckpt", serial_replicas=True,
                                                         attempt_limit=64))
    task = hf.get_workload("matmul").attach(rt, kinds=kinds)
    kernel_of = {u["id"]: {"gpu-tc": "mm_tc", "gpu-simt": "mm_simt", "gpu-tc3": "mm_tc3x"}[u["kind"]]
                 for u in cfg["units"]}
    fid = hf.workloads.MATMUL_FIDELITY
    taps = {}

    def tap(log, areas):
        (bufs,) = areas.values()
        with torch.cuda.stream(rt.backend.stream(0)):
            taps[log["seq"]] = [b.view(torch.float32).cpu().numpy() for b in bufs]
    rt.executor.replica_tap = tap
    rngs = {u["id"]: random.Random(u["seed"]) for u in cfg["units"]}
    vt = hf.ValueType.FLOAT32
    reports = []
    with rt.task_stream(depth=1) as ts:
        for _ in range(tasks):
            ia = rt.register_device_data(ta.view(-1).view(torch.uint8), N * N, vt, "r", "gpu0mem")
            ib = rt.register_device_data(tb.view(-1).view(torch.uint8), N * N, vt, "r", "gpu0mem")
            ic = rt.register_device_data(torch.zeros(4 * N * N, dtype=torch.uint8, device="cuda"), N * N, vt, "w",
                                         "gpu0mem")
            reports.append((ts.submit(task, {"A": ia, "B": ib, "C": ic, "n": N}, hf.Strategy(strategy)), ic))
    rounds = sorted((log["seq"], log) for rep, _ in reports for log in rep.rounds_log)
    launched = {}
    n_votes = n_faults = 0
    for seq, log in rounds:
        for slot, unit in sorted(log["launched"].items()):
            view = clean[kernel_of[unit]].copy()
            ev = fault_schedule.apply_attempt(rngs[unit], (0, 0, 0, p), [view], [True], mode="bitflip")
            want = (ev["corrupt"][1], ev["corrupt"][2]) if ev["corrupt"] else None
            assert log["corrupt"].get(slot) == want, (seq, slot, unit)
            launched[(seq, slot)] = view
            n_faults += want is not None
        if "verdict" not in log:
            continue
        n_votes += 1
        reps = taps[seq]
        slots = log["slots"]
        # the replica bytes voted are the clean variant output with the drawn
        # flip (bit flips are the only fault drawn here, so every vote's slots
        # were all launched in its own round)
        assert sorted(log["launched"]) == list(range(len(slots)))
        for r, unit in enumerate(slots):
            assert reps[r].tobytes() == launched[(seq, r)].tobytes(), (seq, r, unit)
        order = sorted(range(len(slots)), key=lambda r: (fid[kernel_of[slots[r]]], r))
        ores = ovote.vote([reps[r] for r in order], 1e-3)
        mism = [0] * len(slots)
        for j, r in enumerate(order):
            mism[r] = ores.mismatch[j]
        want_verdict = ores.verdict if len(slots) > 2 else ("match" if ores.verdict == "match" else "mismatch")
        assert (log["verdict"], log["mismatch"], log["unresolved"]) == (want_verdict, mism, ores.unresolved)
        fd = log["first_divergence"]
        assert (fd[1] if fd else -1) == ores.first_div
    assert n_votes >= tasks
    for rep, ic in reports:
        assert rep.success
        got = rt.read_array(ic)
        assert got.tobytes() == clean["mm_simt"].tobytes() or \
            ovote.reference_first_divergence(got, clean["mm_simt"], 1e-3) is None
    if p >= 0.4:
        assert n_faults >= 5
