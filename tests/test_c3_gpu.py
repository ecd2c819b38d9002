"""Replicas that are not local HBM buffers, and replicas on distinct devices
(BASELINE configs[2]).

The load rule (csrc/common.cuh): every replica the vote kernel only reads is
loaded with ld.global.nc — local HBM, a peer GPU's memory over NVLink, or
mapped pinned host memory over UVA alike (each replica's producers are
ordered before the vote by events); the in-place target is loaded coherently.
On a one-GPU box the "non-local pointer" case is a pinned host replica (UVA);
the sliced multi-GPU vote and the replica-per-GPU runtime run with every
slice / replica space on device 0 (same code path, no NVLink), and for real
on GPUs 0/1/2 when the box has three.  Decisions, counts, first divergence
and voted bytes are checked against the oracle (oracle/vote.py, SURVEY.md
Appendix A; K = 2 reduction pinned to /root/reference voting.py:68-123).
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
from paper_1405_2912_b200.backend import CudaBackend  # noqa: E402


def _replicas(n, K, seed, faults):
    rng = np.random.default_rng(seed)
    base = rng.uniform(1, 2, n).astype(np.float32)
    reps = [(base * (1 + 1e-6 * rng.standard_normal(n))).astype(np.float32) for _ in range(K)]
    for r, i, bit in faults:
        reps[r].view(np.uint32)[i] ^= np.uint32(1 << bit)
    return reps


def _check(res, ores, voted_host=None):
    assert (res.verdict, res.mismatch, res.unresolved, res.first_div, res.winner) == \
        (ores.verdict, ores.mismatch, ores.unresolved, ores.first_div, ores.winner)
    if voted_host is not None:
        assert voted_host.tobytes() == ores.voted.tobytes()


@pytest.mark.parametrize("host_slot", [0, 1, 2])
@pytest.mark.parametrize("in_place", [False, True])
def test_vote_with_pinned_host_replica(host_slot, in_place):
    """One replica lives in pinned host memory (UVA loads over PCIe), the
    others in HBM; with in_place the voted output goes over replica 0, which
    may itself be the host replica (stores over UVA)."""
    n = (1 << 20) + 7
    faults = [(1, 5, 30), (2, n - 1, 29), (0, n // 2, 31), (1, n // 2 + 1, 23)]
    reps = _replicas(n, 3, 7 + host_slot, faults)
    ores = ovote.vote(reps, 1e-3)
    ts = []
    for r, x in enumerate(reps):
        t = torch.from_numpy(x.copy())
        ts.append(t.pin_memory() if r == host_slot else t.cuda())
    voted = ts[0] if in_place else torch.empty(n, device="cuda")
    res = kernels.vote(ts, 1e-3, voted=voted, device=0)
    torch.cuda.synchronize()
    _check(res, ores, voted.cpu().numpy())
    assert res.verdict == "corrected"


def test_vote_all_replicas_in_host_memory():
    n = 4099
    reps = _replicas(n, 3, 3, [(2, 4098, 30)])
    ts = [torch.from_numpy(x.copy()).pin_memory() for x in reps]
    voted = torch.empty(n).pin_memory()
    res = kernels.vote(ts, 1e-3, voted=voted, device=0)
    _check(res, ovote.vote(reps, 1e-3), voted.numpy())


@pytest.mark.parametrize("K", [2, 3, 5])
def test_backend_sliced_vote_on_one_device(K):
    """CudaBackend's asynchronous sliced vote (the multi-GPU path) with every
    slice on device 0, voting in place into replica 0 (K >= 3): combined
    slices must equal one unsliced oracle vote; faults sit on and next to
    slice boundaries."""
    n = 3 * 65536 + 13
    bnd = [65536 * i for i in range(1, 3)]
    faults = [(K - 1, bnd[0] - 1, 30), (0, bnd[0], 31), (1 % K, bnd[1], 27), (K - 1, n - 1, 24)]
    reps = _replicas(n, K, 40 + K, faults)
    ores = ovote.vote(reps, 1e-3)
    be = CudaBackend()
    bufs = [torch.from_numpy(x.copy()).cuda().view(torch.uint8) for x in reps]
    voted = bufs[0] if K >= 3 else None
    h = be._vote_sliced_start(bufs, hf.ValueType.FLOAT32, 4, [1e-3] * K, None, voted, [0, 0, 0])
    res, ns = h.wait()
    assert ns > 0
    _check(res, ores, bufs[0].view(torch.float32).cpu().numpy() if K >= 3 else None)


def _c3_runtime(devices, p, seed):
    cfg = hf.b200_replica_fleet_config(devices=devices)
    for u in cfg["units"]:
        u.update({"corrupt_prob": p, "corrupt_mode": "bitflip", "seed": seed + u["seed"]})
    rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(checkpoint_space="ckpt", attempt_limit=100))
    task = hf.get_workload("matmul").attach(rt)
    return rt, task, cfg


def _run_c3_replay(devices, n=512, tasks=12, p=0.3, seed=5, depth=None):
    """HetTMR with one variant kind per replica space: every round's fault
    placement equals the oracle draw order, the vote decision equals the
    oracle on the exact bytes voted (tapped before the vote), the commit is
    the SIMT replica's bytes (or the voted value where it was faulty)."""
    rt, task, cfg = _c3_runtime(devices, p, seed)
    st = hf.Strategy(hf.StrategyKind.HET_TMR, spread="device" if len(set(devices)) == 3 else "unit")
    taps = {}

    def tap(log, areas):
        (bufs,) = areas.values()
        outs = []
        for b in bufs:
            with torch.cuda.device(b.device), torch.cuda.stream(rt.backend.stream(b.device.index)):
                outs.append(b.view(torch.float32).cpu().numpy())
        taps[log["seq"]] = outs
    rt.executor.replica_tap = tap
    a, b = omatmul.make_inputs(n, seed=seed)
    ta = torch.from_numpy(a).to(f"cuda:{devices[0]}")
    tb = torch.from_numpy(b).to(f"cuda:{devices[0]}")
    rngs = {u["id"]: random.Random(u["seed"]) for u in cfg["units"]}
    reports, outs = [], []
    vt = hf.ValueType.FLOAT32
    for _ in range(tasks):
        ia = rt.register_device_data(ta.view(-1).view(torch.uint8).clone(), n * n, vt, "r", "r0mem")
        ib = rt.register_device_data(tb.view(-1).view(torch.uint8).clone(), n * n, vt, "r", "r0mem")
        ic = rt.register_data(bytes(4 * n * n), n * n, vt, "w")
        reports.append(rt.invoke(task, {"A": ia, "B": ib, "C": ic, "n": n}, st))
        outs.append(rt.read_array(ic))
    exact = omatmul.matmul(a, b).reshape(-1)
    for rep, out in zip(reports, outs):
        assert rep.success
        assert {s for log in rep.rounds_log for s in log.get("slots", [])} <= {u["id"] for u in cfg["units"]}
        for log in rep.rounds_log:
            for slot, unit in sorted(log["launched"].items()):
                ev = fault_schedule.apply_attempt(rngs[unit], (0, 0, 0, p), [np.zeros(n * n, np.float32)],
                                                  [True], mode="bitflip")
                want = (ev["corrupt"][1], ev["corrupt"][2]) if ev["corrupt"] else None
                assert log["corrupt"].get(slot) == want
            if "verdict" in log:
                reps = taps[log["seq"]]
                slots = log["slots"]
                order = sorted(range(3), key=lambda r: ({"r0.simt": 0, "r2.tc3": 1, "r1.tc": 2}[slots[r]], r))
                ores = ovote.vote([reps[r] for r in order], 1e-3)
                mism = [0] * 3
                for j, r in enumerate(order):
                    mism[r] = ores.mismatch[j]
                assert (log["verdict"], log["mismatch"], log["unresolved"]) == (ores.verdict, mism, ores.unresolved)
                fd = log["first_divergence"]
                assert (fd[1] if fd else -1) == ores.first_div
                if log["verdict"] != "mismatch":
                    assert out.tobytes() == ores.voted.tobytes()
        assert ovote.reference_first_divergence(out, exact, 1e-3) is None
    return reports


def test_replica_fleet_runtime_on_one_gpu():
    reports = _run_c3_replay((0, 0, 0))
    votes = [v for r in reports for v in r.votes]
    assert "corrected" in votes or "mismatch" in votes


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 3, reason="needs 3 GPUs")
def test_replicas_on_three_gpus_with_nvlink_sliced_vote():
    from paper_1405_2912_b200 import _lib
    _lib.enable_peers()
    if not all(_lib.peer_enabled(i, j) for i in range(3) for j in range(3) if i != j):
        pytest.skip("no peer access between GPUs 0-2")
    reports = _run_c3_replay((0, 1, 2), tasks=10)
    units = {s for r in reports for log in r.rounds_log for s in log.get("slots", [])}
    assert units == {"r0.simt", "r1.tc", "r2.tc3"}


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 3, reason="needs 3 GPUs")
@pytest.mark.parametrize("K", [2, 3])
def test_peer_replicas_sliced_vote_three_gpus(K):
    """Replicas on GPUs 0..K-1 (peer pointers), the vote sliced over them,
    voted in place into replica 0 through peer stores."""
    from paper_1405_2912_b200 import _lib
    _lib.enable_peers()
    n = (1 << 22) + 5
    faults = [(K - 1, 17, 30), (0, n - 2, 30), (1, n // 2, 28)]
    reps = _replicas(n, K, 90 + K, faults)
    ores = ovote.vote(reps, 1e-3)
    be = CudaBackend()
    bufs = [torch.from_numpy(x.copy()).to(f"cuda:{r}").view(torch.uint8) for r, x in enumerate(reps)]
    h = be.vote_start(bufs, hf.ValueType.FLOAT32, 4, [1e-3] * K, voted=bufs[0] if K >= 3 else None)
    res, _ = h.wait()
    _check(res, ores, bufs[0].view(torch.float32).cpu().numpy() if K >= 3 else None)
