"""End-to-end GPU tests of the drop-in Runtime: duplicated execution of the
matmul variants, K-way voting, device checkpoint/rollback and seeded fault
injection, checked against the CPU oracle.

The fault-schedule parity test replays every round the executor ran with
the oracle's restatement of the reference draw order (oracle/fault_schedule.py)
and the oracle voter, and requires identical verdicts, per-replica mismatch
counts and first divergences (bit-exact decisions)."""

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


def matmul_runtime(kinds=("gpu-tc", "gpu-simt"), overrides=None, **cfg_kw):
    cfg = hf.gpu_fleet_config(devices=(0,), kinds=kinds)
    cfg["memory_spaces"].append({"id": "gpu0ckpt", "device": 0})
    for u in cfg["units"]:
        u.update((overrides or {}).get(u["id"], {}))
    rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(**cfg_kw))
    task = hf.get_workload("matmul").attach(rt, kinds=kinds)
    return rt, task


def register_mm(rt, a, b, device_inputs=False):
    n = a.shape[0]
    vt = hf.ValueType.FLOAT32
    if device_inputs:
        ia = rt.register_device_data(torch.from_numpy(a).cuda().view(-1).view(torch.uint8), n * n, vt, "r", "gpu0mem")
        ib = rt.register_device_data(torch.from_numpy(b).cuda().view(-1).view(torch.uint8), n * n, vt, "r", "gpu0mem")
    else:
        ia = rt.register_data(a.tobytes(), n * n, vt, "r")
        ib = rt.register_data(b.tobytes(), n * n, vt, "r")
    ic = rt.register_data(bytes(4 * n * n), n * n, vt, "w")
    return ia, ib, ic, {"A": ia, "B": ib, "C": ic, "n": n}


def test_dmr_matmul_fault_free_matches_oracle():
    a, b = omatmul.make_inputs(512, seed=3)
    rt, task = matmul_runtime()
    _, _, ic, args = register_mm(rt, a, b)
    rep = rt.invoke(task, args, hf.Strategy(hf.StrategyKind.HET_DMR))
    assert rep.success and rep.votes == ["match"]
    got = rt.read_array(ic).reshape(512, 512)
    assert ovote.reference_first_divergence(got.reshape(-1), omatmul.matmul(a, b).reshape(-1), 1e-3) is None
    assert {s for s in rep.rounds_log[0]["slots"]} == {"gpu0.simt", "gpu0.tc"}


def test_dmr_detects_corruption_and_reruns():
    a, b = omatmul.make_inputs(256, seed=4)
    # find a seed whose first draw is corrupt and second is clean at p = 0.5
    seed = next(s for s in range(100) if random.Random(s).random() < 0.5 and
                (lambda r: (r.random(), r.randrange(1), r.randrange(256 * 256), r.random())[3])(random.Random(s)) >= 0.5)
    rt, task = matmul_runtime(overrides={"gpu0.tc": {"corrupt_prob": 0.5, "seed": seed,
                                                     "corrupt_rel_magnitude": 0.5}})
    _, _, ic, args = register_mm(rt, a, b)
    rep = rt.invoke(task, args, hf.Strategy(hf.StrategyKind.HET_DMR))
    assert rep.success
    assert rep.votes == ["mismatch", "match"]
    assert rep.fault_counts["vote_mismatch"] == 1
    got = rt.read_array(ic)
    assert ovote.reference_first_divergence(got, omatmul.matmul(a, b).reshape(-1), 1e-3) is None


def test_tmr_majority_corrects_single_faulty_variant():
    a, b = omatmul.make_inputs(256, seed=5)
    rt, task = matmul_runtime(kinds=("gpu-tc", "gpu-simt", "gpu-tc3"),
                              overrides={"gpu0.tc": {"corrupt_prob": 1.0, "corrupt_rel_magnitude": 0.5}})
    _, _, ic, args = register_mm(rt, a, b)
    rep = rt.invoke(task, args, hf.Strategy(hf.StrategyKind.HET_TMR))
    assert rep.success and rep.votes == ["corrected"]
    log = rep.rounds_log[0]
    faulty_slot = log["slots"].index("gpu0.tc")
    assert log["mismatch"][faulty_slot] == 1 and sum(log["mismatch"]) == 1
    # the committed result is the voted buffer: never the corrupted element
    got = rt.read_array(ic)
    ref = omatmul.matmul(a, b).reshape(-1)
    assert ovote.reference_first_divergence(got, ref, 1e-3) is None
    # the faulty unit's reliability rating was penalised
    rec = rt.profiles.record(rt.profiles.key_for("mm_tc", 256 * 256, "gpu0.tc"))
    assert rec.t - rec.v == 1


def test_perfcp_abort_rolls_back_to_hbm_checkpoint():
    a, b = omatmul.make_inputs(256, seed=6)
    rt, task = matmul_runtime(overrides={"gpu0.simt": {"abort_prob": 1.0}}, checkpoint_space="gpu0ckpt")
    ia, ib, ic, args = register_mm(rt, a, b, device_inputs=True)
    rep = rt.invoke(task, args, hf.Strategy(hf.StrategyKind.PERF_CP))
    assert rep.success and rep.fault_counts["abort"] >= 1
    # inputs were sole device copies: protected attempts snapshot them into HBM
    assert rt.memory.checkpoints >= 2
    table = rt.memory.sibling_table()
    assert (ia, "gpu0ckpt", 0, True) in table
    got = rt.read_array(ic)
    assert ovote.reference_first_divergence(got, omatmul.matmul(a, b).reshape(-1), 1e-3) is None


COPY_PARAMS = (hf.Param.area("input", "r"), hf.Param.area("output", "w"), hf.Param.scalar("count"))


def _copy_body(ctx):
    kernels.copy(ctx.request("output", "w"), ctx.request("input", "r"), stream=ctx.stream)


@pytest.mark.parametrize("K,strategy", [(2, hf.StrategyKind.HET_DMR), (3, hf.StrategyKind.HET_TMR)])
def test_fault_schedule_and_decisions_match_oracle(K, strategy):
    """Seeded random bit flips on bit-identical replicas: every round's fault
    placement and vote decision must equal the oracle replay."""
    n = 4099
    kinds = [f"gpu-v{i}" for i in range(K)]
    cfg = {"memory_spaces": [{"id": "host", "host": True}, {"id": "gpu0mem", "device": 0}],
           "units": [{"id": f"u{i}", "kind": kinds[i], "memory_space": "gpu0mem", "timing": "measured",
                      "corrupt_prob": 0.35, "corrupt_mode": "bitflip", "seed": 100 + 7 * i} for i in range(K)]}
    rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(serial_replicas=True, attempt_limit=200))
    task = rt.declare_task("copy", COPY_PARAMS)
    for i in range(K):
        rt.attach_kernel(task, f"copy{i}", kinds[i], _copy_body)
    rng = np.random.default_rng(0)
    oracle_rngs = {f"u{i}": random.Random(100 + 7 * i) for i in range(K)}
    rounds = 0
    for t in range(25):
        data = rng.uniform(1, 2, n).astype(np.float32)
        inp = rt.register_data(data.tobytes(), n, hf.ValueType.FLOAT32, "r")
        out = rt.register_data(bytes(4 * n), n, hf.ValueType.FLOAT32, "w")
        rep = rt.invoke(task, {"input": inp, "output": out, "count": n}, hf.Strategy(strategy))
        for log in rep.rounds_log:
            rounds += 1
            reps = []
            for slot, unit in sorted(log["launched"].items()):
                view = data.copy()
                ev = fault_schedule.apply_attempt(oracle_rngs[unit], (0, 0, 0, 0.35), [view], [True],
                                                  mode="bitflip")
                if ev["corrupt"] is not None:
                    assert log["corrupt"][slot] == (ev["corrupt"][1], ev["corrupt"][2])
                else:
                    assert slot not in log["corrupt"]
                reps.append(view)
            if "verdict" in log:
                ores = ovote.vote(reps, 1e-3)
                expect = ores.verdict if K > 2 else ("match" if ores.verdict == "match" else "mismatch")
                assert log["verdict"] == expect
                assert log["mismatch"] == ores.mismatch
                fd = log["first_divergence"]
                assert (fd[1] if fd else -1) == ores.first_div
        # committed output: exact unless an undetectable flip (within δ by
        # definition) survived the vote
        got = rt.read_array(out)
        assert ovote.reference_first_divergence(got, data, 1e-3) is None
    assert rounds >= 25


@pytest.mark.parametrize("depth", [1, 2])
def test_task_stream_decisions_match_oracle(depth):
    """Pipelined TaskStream: rounds of different tasks interleave; replaying
    every round in its launch sequence ("seq") with the oracle must reproduce
    each fault placement and vote decision bit-exactly."""
    K, n = 3, 2053
    kinds = [f"gpu-v{i}" for i in range(K)]
    cfg = {"memory_spaces": [{"id": "host", "host": True}, {"id": "gpu0mem", "device": 0}],
           "units": [{"id": f"u{i}", "kind": kinds[i], "memory_space": "gpu0mem", "timing": "measured",
                      "corrupt_prob": 0.4, "corrupt_mode": "bitflip", "seed": 500 + i} for i in range(K)]}
    rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(serial_replicas=True, attempt_limit=200))
    task = rt.declare_task("copy", COPY_PARAMS)
    for i in range(K):
        rt.attach_kernel(task, f"copy{i}", kinds[i], _copy_body)
    rng = np.random.default_rng(1)
    datas, reports, outs = [], [], []
    with rt.task_stream(depth=depth) as ts:
        for t in range(20):
            data = rng.uniform(1, 2, n).astype(np.float32)
            inp = rt.register_data(data.tobytes(), n, hf.ValueType.FLOAT32, "r")
            out = rt.register_data(bytes(4 * n), n, hf.ValueType.FLOAT32, "w")
            reports.append(ts.submit(task, {"input": inp, "output": out, "count": n}, hf.Strategy(hf.StrategyKind.HET_TMR)))
            datas.append(data)
            outs.append(out)
    rounds = sorted((log["seq"], t, log) for t, r in enumerate(reports) for log in r.rounds_log)
    rngs = {f"u{i}": random.Random(500 + i) for i in range(K)}
    for _, t, log in rounds:
        reps = []
        for slot, unit in sorted(log["launched"].items()):
            view = datas[t].copy()
            ev = fault_schedule.apply_attempt(rngs[unit], (0, 0, 0, 0.4), [view], [True], mode="bitflip")
            assert (log["corrupt"].get(slot) == (ev["corrupt"][1], ev["corrupt"][2])) if ev["corrupt"] \
                else slot not in log["corrupt"]
            reps.append(view)
        if "verdict" in log:
            ores = ovote.vote(reps, 1e-3)
            assert (log["verdict"], log["mismatch"]) == (ores.verdict, ores.mismatch)
    for t, out in enumerate(outs):
        assert reports[t].success
        assert ovote.reference_first_divergence(rt.read_array(out), datas[t], 1e-3) is None


@pytest.mark.parametrize("seed", range(0, 300, 3))
def test_memory_protocol_on_device_matches_model(seed):
    """The sibling/version protocol over real HBM buffers (hf_copy,
    hf_checkpoint, pinned host) against the flat model, as on the host
    double in test_runtime_host.py."""
    from oracle import memory_model
    cfg = {"default_ns_per_byte": 0.01,
           "memory_spaces": [{"id": "host", "host": True}, {"id": "gpu1mem", "device": 0},
                             {"id": "gpu2mem", "device": 0}],
           "units": [{"id": "g", "kind": "gpu", "memory_space": "gpu1mem"}]}
    fleet = hf.load_fleet(cfg)
    from paper_1405_2912_b200.backend import CudaBackend
    m = hf.MemoryManager(fleet, CudaBackend())
    ref = memory_model.SiblingModel("host")
    rng = random.Random(seed)
    spaces = ["host", "gpu1mem", "gpu2mem"]
    areas = []
    for _ in range(30):
        op = rng.choice(["reg", "read", "read", "write", "write", "fault", "inval"])
        if op == "reg" or not areas:
            if len(areas) < 3:
                size = rng.randint(1, 8) * 4
                payload = bytes(rng.randrange(256) for _ in range(size))
                areas.append((m.register(payload, size // 4, hf.ValueType.INT, "rw"), ref.register(payload), size))
            continue
        ia, ra, size = rng.choice(areas)
        sp = rng.choice(spaces)
        prot = rng.random() < 0.5
        if op == "read":
            try:
                h = m.request(ia, sp, "r", prot)
                got = (h.base_version, m.payload_bytes(h))
            except hf.DataLossError:
                got = "loss"
            try:
                exp = ref.read(ra, sp, prot)
            except memory_model.ModelDataLoss:
                exp = "loss"
            assert got == exp
        elif op == "write":
            acc = rng.choice(["w", "rw"])
            new = bytes(rng.randrange(256) for _ in range(rng.randint(0, size)))
            try:
                h = m.request(ia, sp, acc, prot)
                if new:
                    kernels.scribble(h.payload, new[:64]) if len(new) <= 64 else None
                    new = new[:64]
                m.commit_success([h])
                got = h.target_version
            except hf.DataLossError:
                got = "loss"
            try:
                tok = ref.write(ra, sp, acc, prot)
                tok[3][:len(new)] = new
                ref.commit(tok)
                exp = tok[2]
            except memory_model.ModelDataLoss:
                exp = "loss"
            assert got == exp
        elif op == "fault":
            try:
                m.request(ia, sp, "r", True)
                m.request(ia, sp, "w", True)
                if sp != "host":
                    m.invalidate(ia, sp)
                got = "ok"
            except hf.DataLossError:
                got = "loss"
            try:
                ref.read(ra, sp, True)
                ref.write(ra, sp, "w", True)
                ref.rollback([ra], sp)
                exp = "ok"
            except memory_model.ModelDataLoss:
                exp = "loss"
            assert got == exp
        else:
            if (ia, sp) in {(a, s) for a, s, _, _ in m.sibling_table()}:
                m.invalidate(ia, sp)
                ref.invalidate(ra, sp)
        amap = {x: y for x, y, _ in areas}
        assert {(amap[a], s): (v, ok) for a, s, v, ok in m.sibling_table()} == \
            {k: (e[0], e[1]) for k, e in ref.t.items()}
        for (a, s), (v, ok, data) in m.payload_snapshot().items():
            if ok:
                assert data == ref.t[(amap[a], s)][2]


def test_watchdog_times_out_hung_replica_and_quarantines_unit():
    """A replica whose kernel never returns within its deadline is a timeout
    (classified while it still runs, clocked from when it started on the
    GPU); the task re-dispatches to another unit and the hung unit is held
    out of selection until its stream drains."""
    import time as _time

    cfg = {"memory_spaces": [{"id": "host", "host": True}, {"id": "gpu0mem", "device": 0},
                             {"id": "gpu0ckpt", "device": 0}],
           "units": [{"id": "ua", "kind": "gpu-a", "memory_space": "gpu0mem", "timing": "measured"},
                     {"id": "ub", "kind": "gpu-b", "memory_space": "gpu0mem", "timing": "measured"}]}
    rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(default_deadline_ns=50_000_000,
                                                         checkpoint_space="gpu0ckpt"))
    task = rt.declare_task("copy", COPY_PARAMS)
    calls = []

    def body(ctx):
        if not calls:
            kernels.debug_spin(1_500_000_000, stream=ctx.stream, device=ctx.device)   # a 1.5 s hang
        calls.append(ctx.stream)
        _copy_body(ctx)

    rt.attach_kernel(task, "ka", "gpu-a", body)
    rt.attach_kernel(task, "kb", "gpu-b", body)
    n = 1 << 20
    data = np.random.default_rng(1).uniform(1, 2, n).astype(np.float32)
    inp = rt.register_data(data.tobytes(), n, hf.ValueType.FLOAT32, "r")
    out = rt.register_data(bytes(4 * n), n, hf.ValueType.FLOAT32, "w")
    torch.cuda.synchronize()
    t0 = _time.perf_counter()
    rep = rt.invoke(task, {"input": inp, "output": out, "count": n}, hf.Strategy(hf.StrategyKind.PERF_CP))
    got = rt.read_array(out)
    wall = _time.perf_counter() - t0
    assert rep.success and rep.fault_counts["timeout"] == 1 and rep.attempts == 2
    assert np.array_equal(got, data)
    assert wall < 1.0, f"the hang was waited out ({wall:.2f} s)"
    hung = set(rt.executor._hung)
    assert len(hung) == 1
    t1 = _time.perf_counter()
    mid = rt.invoke(task, {"input": inp, "output": out, "count": n}, hf.Strategy(hf.StrategyKind.PERF_CP))
    assert _time.perf_counter() - t1 < 0.5 and mid.success and mid.committed.unit_id not in hung
    assert np.array_equal(rt.read_array(out), data)
    torch.cuda.synchronize()        # the spin ends (<= 1.5 s); the unit returns to service
    rt.executor._reap_hung()
    assert not rt.executor._hung
    rep2 = rt.invoke(task, {"input": inp, "output": out, "count": n}, hf.Strategy(hf.StrategyKind.PERF_CP))
    assert rep2.success and rep2.fault_counts["timeout"] == 0


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6])
def test_c1_tmr_1024_single_seeded_bitflip(seed):
    """BASELINE config C1: TMR of a 1024^2 fp32 matmul (tcgen05, SIMT and
    3xTF32 replicas) with one seeded bit flip in the tensor-core replica.
    The fault coordinates follow the reference draw order (Appendix B, via
    the oracle); the vote corrects it exactly when the flip moves the value
    by more than δ — bits >= 15 always, bits <= 13 never."""
    n = 1024
    a, b = omatmul.make_inputs(n, seed=100 + seed)
    rt, task = matmul_runtime(kinds=("gpu-tc", "gpu-simt", "gpu-tc3"),
                              overrides={"gpu0.tc": {"corrupt_prob": 1.0, "corrupt_mode": "bitflip",
                                                     "seed": seed}})
    _, _, ic, args = register_mm(rt, a, b)
    rep = rt.invoke(task, args, hf.Strategy(hf.StrategyKind.HET_TMR))
    assert rep.success and len(rep.votes) == 1
    rng = random.Random(seed)
    assert fault_schedule.draw_class(rng, 0.0, 0.0, 0.0, 1.0) == "corrupt"
    rng.randrange(1)
    idx, bit = rng.randrange(n * n), rng.randrange(32)
    log = rep.rounds_log[0]
    slot = log["slots"].index("gpu0.tc")
    assert rep.injected == [(slot, "gpu0.tc", idx, bit)]
    if bit >= 15:
        assert rep.votes == ["corrected"] and log["mismatch"][slot] == 1 and sum(log["mismatch"]) == 1
        assert log["first_divergence"][1] == idx
    elif bit <= 13:
        assert rep.votes == ["match"]
    got = rt.read_array(ic)
    assert ovote.reference_first_divergence(got, omatmul.matmul(a, b).reshape(-1), 1e-3) is None


@pytest.mark.gpu
def test_reserve_presizes_the_device_heap():
    """Runtime.reserve(space, nbytes, count): the caching allocator then holds
    count free blocks, so count buffers of that size for the space's compute
    stream allocate no new device segment (no cudaMalloc inside a stream)."""
    cfg = hf.gpu_fleet_config(devices=(0,), kinds=("gpu-tc", "gpu-simt"))
    rt = hf.Runtime(hf.load_fleet(cfg))
    nb = 48 << 20
    torch.cuda.synchronize()
    rt.reserve("gpu0mem", nb, 6)
    stats = torch.cuda.memory_stats()
    # (the reserved total need not grow: earlier tests in the process may
    # have left enough cached blocks; what matters is the next check)
    seg0 = stats.get("segment.all.allocated", 0)
    sp = rt.fleet.spaces["gpu0mem"]
    bufs = [rt.backend.alloc(sp, nb, zero=False) for _ in range(6)]
    assert torch.cuda.memory_stats().get("segment.all.allocated", 0) == seg0
    del bufs
    with pytest.raises(hf.UnknownSpaceError):
        rt.reserve("nowhere", nb, 1)


def _hang_runtime(devices, deadline_ns=50_000_000):
    spaces = [{"id": "host", "host": True}] + [{"id": f"g{d}mem", "device": d} for d in devices]
    units = []
    for d in devices:
        # two units per kind: after the hung unit's timeout quarantines it
        # (reference rating rule), HetDMR still finds a diverse pair
        units += [{"id": f"g{d}.{k}{i}", "kind": f"gpu-{k}", "memory_space": f"g{d}mem", "timing": "measured"}
                  for k in "ab" for i in (1, 2)]
    rt = hf.Runtime(hf.load_fleet({"memory_spaces": spaces, "units": units}),
                    hf.RuntimeConfig(default_deadline_ns=deadline_ns, attempt_limit=20))
    task = rt.declare_task("copy", COPY_PARAMS)
    calls = []

    def body(ctx):
        if not calls:
            kernels.debug_spin(1_500_000_000, stream=ctx.stream, device=ctx.device)   # a 1.5 s hang
        calls.append(ctx.device)
        _copy_body(ctx)

    rt.attach_kernel(task, "ka", "gpu-a", body)
    rt.attach_kernel(task, "kb", "gpu-b", body)
    return rt, task


def test_task_stream_hang_is_bounded_on_one_gpu():
    """TaskStream (deferred timing, vote launched before the replicas are
    known to finish): a hung replica must not block the host.  Its vote
    already joined GPU 0's compute stream to the hung stream, so GPU 0 is
    wedged; with no other device the re-dispatch has no candidate and the
    task fails fast with the mapper's error instead of waiting out the hang.
    Once the spin drains, the device returns to service."""
    import time as _time
    rt, task = _hang_runtime([0])
    n = 1 << 20
    data = np.random.default_rng(2).uniform(1, 2, n).astype(np.float32)
    inp = rt.register_data(data.tobytes(), n, hf.ValueType.FLOAT32, "r")
    out = rt.register_data(bytes(4 * n), n, hf.ValueType.FLOAT32, "w")
    torch.cuda.synchronize()
    t0 = _time.perf_counter()
    with pytest.raises((hf.StrategyInfeasibleError, hf.UnrecoverableTaskError)):
        with rt.task_stream(depth=1) as ts:
            ts.submit(task, {"input": inp, "output": out, "count": n}, hf.Strategy(hf.StrategyKind.HET_DMR))
    assert _time.perf_counter() - t0 < 1.0, "the host waited out the hang"
    assert rt.executor._wedged and any(not k.endswith("#stranded") for k in rt.executor._hung)
    torch.cuda.synchronize()          # the spin ends (<= 1.5 s)
    rt.executor._reap_hung()
    assert not rt.executor._wedged
    out2 = rt.register_data(bytes(4 * n), n, hf.ValueType.FLOAT32, "w")
    with rt.task_stream(depth=1) as ts:
        rep = ts.submit(task, {"input": inp, "output": out2, "count": n}, hf.Strategy(hf.StrategyKind.HET_DMR))
    assert rep.success and rep.votes == ["match"]
    assert np.array_equal(rt.read_array(out2), data)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_task_stream_hang_redispatches_to_another_gpu():
    import time as _time
    rt, task = _hang_runtime([0, 1])
    n = 1 << 20
    data = np.random.default_rng(3).uniform(1, 2, n).astype(np.float32)
    inp = rt.register_data(data.tobytes(), n, hf.ValueType.FLOAT32, "r")
    out = rt.register_data(bytes(4 * n), n, hf.ValueType.FLOAT32, "w")
    torch.cuda.synchronize()
    t0 = _time.perf_counter()
    with rt.task_stream(depth=1) as ts:
        rep = ts.submit(task, {"input": inp, "output": out, "count": n}, hf.Strategy(hf.StrategyKind.HET_DMR))
    assert _time.perf_counter() - t0 < 1.0
    assert rep.success and rep.fault_counts["timeout"] == 1
    assert np.array_equal(rt.read_array(out), data)
    assert rep.committed.unit_id.startswith("g1.")


TWO_OUT_PARAMS = (hf.Param.area("input", "r"), hf.Param.area("out_a", "w"), hf.Param.area("out_b", "w"),
                  hf.Param.scalar("count"))


def _two_out_body(ctx):
    src = ctx.request("input", "r")
    kernels.copy(ctx.request("out_a", "w"), src, stream=ctx.stream)
    kernels.vec_inc(src, ctx.request("out_b", "w"), stream=ctx.stream)


def test_multi_area_task_votes_in_one_batch_launch():
    """A task with two output areas: the executor votes both in one
    hf_vote_batch launch (CudaBackend.vote_start_batch).  Every round's
    fault placement (which write view, element, bit: reference draw order)
    and the combined decision — sorted-area order, counts summed over areas,
    first divergence from the first diverging area (voting.py:106-123) —
    equal the oracle replay."""
    K, n = 3, 5003
    kinds = [f"gpu-v{i}" for i in range(K)]
    cfg = {"memory_spaces": [{"id": "host", "host": True}, {"id": "gpu0mem", "device": 0}],
           "units": [{"id": f"u{i}", "kind": kinds[i], "memory_space": "gpu0mem", "timing": "measured",
                      "corrupt_prob": 0.4, "corrupt_mode": "bitflip", "seed": 900 + i} for i in range(K)]}
    rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(serial_replicas=True, attempt_limit=200))
    task = rt.declare_task("two", TWO_OUT_PARAMS)
    for i in range(K):
        rt.attach_kernel(task, f"k{i}", kinds[i], _two_out_body)
    launches = []
    orig = rt.backend.vote_start_batch

    def spy(specs, rel, device=None):
        launches.append(len(specs))
        return orig(specs, rel, device=device)
    rt.backend.vote_start_batch = spy
    rng = np.random.default_rng(4)
    rngs = {f"u{i}": random.Random(900 + i) for i in range(K)}
    for t in range(12):
        data = rng.uniform(1, 2, n).astype(np.float32)
        inp = rt.register_data(data.tobytes(), n, hf.ValueType.FLOAT32, "r")
        oa = rt.register_data(bytes(4 * n), n, hf.ValueType.FLOAT32, "w")
        ob = rt.register_data(bytes(4 * n), n, hf.ValueType.FLOAT32, "w")
        rep = rt.invoke(task, {"input": inp, "out_a": oa, "out_b": ob, "count": n}, hf.Strategy(hf.StrategyKind.HET_TMR))
        assert rep.success
        for log in rep.rounds_log:
            views = {}
            for slot, unit in sorted(log["launched"].items()):
                va, vb = data.copy(), (data + np.float32(1)).astype(np.float32)
                fault_schedule.apply_attempt(rngs[unit], (0, 0, 0, 0.4), [va, vb], [True, True], mode="bitflip")
                views[slot] = (va, vb)
            if "verdict" not in log:
                continue
            per = {}
            for ai, area in enumerate((oa, ob)):
                per[area] = ovote.vote([views[s][ai] for s in range(K)], 1e-3)
            mism = [sum(per[a].mismatch[r] for a in per) for r in range(K)]
            unres = sum(per[a].unresolved for a in per)
            verdict = "mismatch" if unres else ("corrected" if any(mism) else "match")
            assert (log["verdict"], log["mismatch"], log["unresolved"]) == (verdict, mism, unres)
            firsts = [(a, per[a].first_div) for a in sorted(per) if per[a].first_div >= 0]
            fd = log["first_divergence"]
            assert (fd[:2] if fd else None) == (firsts[0] if firsts else None)
        assert np.array_equal(rt.read_array(oa), data) or ovote.reference_first_divergence(rt.read_array(oa), data,
                                                                                           1e-3) is None
        assert ovote.reference_first_divergence(rt.read_array(ob), data + np.float32(1), 1e-3) is None
    assert launches and all(c == 2 for c in launches)


def test_voter_placement_costs_are_learnt_from_measured_votes():
    """VoterConfig.learn_costs: every measured vote's kernel time refits the
    hf_vote profiles place_voter ranks by (reference placement: voting.py:
    146-174, calibrated constants voting.py:37-42).  After votes at two
    sizes the fitted rate is the device's, not the prior constant."""
    rt, task = matmul_runtime(kinds=("gpu-tc", "gpu-simt", "gpu-tc3"))
    # sizes where the votes' kernel time is bandwidth- rather than
    # latency-dominated (K = 3 reads of 12 and 48 MiB): at 1-4 MiB the slope
    # between two sizes is noise on a few-microsecond fixed cost
    for n in (1024, 2048, 1024, 2048):
        a, b = omatmul.make_inputs(n, seed=n)
        _, _, _, args = register_mm(rt, a, b)
        assert rt.invoke(task, args, hf.Strategy(hf.StrategyKind.HET_TMR)).success
    profs = [p for p in rt.config.voter.profiles if p.kernel == "hf_vote" and p.unit_kind == "*"]
    assert profs
    per = profs[0].per_byte_ns
    gbs = 1.0 / per           # bytes per ns = GB/s
    assert 200 < gbs < 20_000, gbs     # 12 MiB reads can be partly L2-resident
    assert profs[0].base_ns >= 0



def test_empty_areas_are_rejected_at_registration():
    """The reference refuses zero-element areas (memory.py:92-93), so no task
    ever votes an empty output; the drop-in raises the same error for host
    and device-resident registrations (empty payloads still vote as a match
    at the kernel level, test_kernels_gpu.py::test_empty_votes_async_and_batched)."""
    rt, _task = matmul_runtime()
    with pytest.raises(hf.RegistrationError):
        rt.register_data(b"", 0, hf.ValueType.FLOAT32, "r")
    with pytest.raises(hf.RegistrationError):
        rt.register_device_data(torch.empty(0, dtype=torch.uint8, device="cuda"), 0, hf.ValueType.FLOAT32, "r",
                                "gpu0mem")


def test_shared_gpu_lead_is_the_declared_costliest_variant_and_reads_wait_for_votes():
    """Replicas sharing one GPU: the lead (LEAD_PRIORITY stream) is the variant
    with the largest declared cost (the SIMT GEMM) on every round, whatever
    the measured in-task timings say (r2b).  Votes run on the vote
    stream; committed outputs read back right after each task of a pipelined
    stream equal the SIMT kernel's own bytes (the reads wait on the vote)."""
    from paper_1405_2912_b200.executor import LEAD_PRIORITY
    rt, task = matmul_runtime(kinds=("gpu-tc", "gpu-simt", "gpu-tc3"), serial_replicas=True)
    leads = []
    orig = rt.backend.unit_stream

    def spy(unit_id, device, priority=0, sync=True):
        if priority == LEAD_PRIORITY:
            leads.append(unit_id)
        return orig(unit_id, device, priority=priority, sync=sync)
    rt.backend.unit_stream = spy
    n = 512
    a, b = omatmul.make_inputs(n, seed=11)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    want = torch.empty(n, n, device="cuda")
    kernels.gemm_simt(ta, tb, want)
    want = want.cpu().numpy().tobytes()
    outs = []
    with rt.task_stream(depth=2) as ts:
        for _ in range(8):
            _, _, ic, args = register_mm(rt, a, b, device_inputs=True)
            outs.append((ts.submit(task, args, hf.Strategy(hf.StrategyKind.HET_TMR)), ic))
    assert len(leads) == 8 and set(leads) == {"gpu0.simt"}, leads
    for rep, ic in outs:
        assert rep.success and rep.votes == ["match"]
        host = torch.empty(4 * n * n, dtype=torch.uint8).pin_memory()
        rt.read_into(ic, host)
        assert host.numpy().tobytes() == want


@pytest.mark.parametrize("depth", [None, 1])
def test_nmr5_two_faulty_units_majority_commits_clean_simt_bytes(depth):
    """K = 5 (Strategy(DMR, replicas=5): distinct units, variants may repeat)
    on one GPU: two units flip one bit of every output they produce.  Every
    element keeps a 3-of-5 majority, so the vote corrects; per-replica counts
    are 1 for the two faulty slots and 0 elsewhere; the committed bytes equal
    the clean SIMT kernel's output bit for bit (the vote lands in the lowest
    fidelity-rank replica's buffer, and where that replica is faulty the
    majority value comes from the clean SIMT replica)."""
    cfg = hf.gpu_fleet_config(devices=(0,), kinds=("gpu-tc", "gpu-simt", "gpu-tc3"))
    cfg["memory_spaces"].append({"id": "gpu0ckpt", "device": 0})
    extra = [("gpu0.simt2", "gpu-simt"), ("gpu0.tc2", "gpu-tc")]
    for uid, kind in extra:
        cfg["units"].append({"id": uid, "kind": kind, "memory_space": "gpu0mem", "timing": "measured",
                             "seed": 4242 + len(cfg["units"])})
    faulty = {"gpu0.tc3": 27, "gpu0.simt2": 29}
    for u in cfg["units"]:
        if u["id"] in faulty:
            u.update({"corrupt_prob": 1.0, "corrupt_mode": "bitflip", "corrupt_bit": faulty[u["id"]]})
    rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(checkpoint_space="gpu0ckpt", serial_replicas=True))
    task = hf.get_workload("matmul").attach(rt)
    n = 512
    a, b = omatmul.make_inputs(n, seed=21)
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    want = torch.empty(n, n, device="cuda")
    kernels.gemm_simt(ta, tb, want)
    want = want.cpu().numpy().tobytes()
    strat = hf.Strategy(hf.StrategyKind.DMR, replicas=5)
    reps = []
    if depth is None:
        for _ in range(3):
            _, _, ic, args = register_mm(rt, a, b, device_inputs=True)
            reps.append((rt.invoke(task, args, strat), ic))
    else:
        with rt.task_stream(depth=depth) as ts:
            for _ in range(3):
                _, _, ic, args = register_mm(rt, a, b, device_inputs=True)
                reps.append((ts.submit(task, args, strat), ic))
    for rep, ic in reps:
        assert rep.success and rep.votes == ["corrected"], rep.votes
        log = rep.rounds_log[-1]
        assert len(log["slots"]) == 5
        for slot, unit in enumerate(log["slots"]):
            assert log["mismatch"][slot] == (1 if unit in faulty else 0), (unit, log["mismatch"])
        assert rt.read_area(ic) == want
