"""Control-plane behaviour of the drop-in (reference semantics of
/root/reference/pkg/tests/test_executor.py, test_memory.py, test_mapper.py,
test_devices.py, test_voter.py placement) on a simulated fleet, run on the
CPU through the tests-only HostBackend double.  The same code paths run on
the B200 with CudaBackend in tests/test_runtime_gpu.py."""

import math
import random
from fractions import Fraction

import numpy as np
import pytest

import paper_1405_2912_b200 as hf
from host_backend import HostBackend
from oracle import memory_model

N = 16
DATA = np.arange(1, N + 1, dtype=np.float32)
PERF = hf.Strategy(hf.StrategyKind.PERF)
PERFCP = hf.Strategy(hf.StrategyKind.PERF_CP)
DMR = hf.Strategy(hf.StrategyKind.DMR)
TMR = hf.Strategy(hf.StrategyKind.TMR)
IO = (hf.Param.area("input", "r"), hf.Param.area("output", "w"), hf.Param.scalar("count"))


def fleet_cfg(units, rate=0.01):
    spaces = [{"id": "host", "host": True}]
    for u in units:
        sp = u.get("memory_space", "host")
        if sp not in [s["id"] for s in spaces]:
            spaces.append({"id": sp})
    return {"default_ns_per_byte": rate, "memory_spaces": spaces, "units": list(units)}


def three_units(**over):
    cfg = fleet_cfg([
        {"id": "cpu0", "kind": "cpu", "memory_space": "host", "base_latency_us": 100.0, "per_elem_cost_ns": 10.0, "seed": 1},
        {"id": "gpu1", "kind": "gpu", "memory_space": "gpu1mem", "base_latency_us": 20.0, "per_elem_cost_ns": 1.0, "seed": 2},
        {"id": "gpu2", "kind": "gpu", "memory_space": "gpu2mem", "base_latency_us": 30.0, "per_elem_cost_ns": 2.0, "seed": 3},
    ])
    for u in cfg["units"]:
        u.update(over.get(u["id"], {}))
    return cfg


def inc(ctx):
    n = ctx.arg("count")
    np.add(ctx.request("input", "r")[:n], np.float32(1.0), out=ctx.request("output", "w")[:n])


def runtime(cfg, rtc=None, kinds=("cpu", "gpu")):
    rt = hf.Runtime(hf.load_fleet(cfg), rtc or hf.RuntimeConfig(), backend=HostBackend())
    task = rt.declare_task("inc", IO)
    for k in kinds:
        rt.attach_kernel(task, f"inc_{k}", k, inc)
    return rt, task


def args_for(rt, data=DATA):
    n = len(data)
    i = rt.register_data(data.astype(np.float32).tobytes(), n, hf.ValueType.FLOAT32, "r")
    o = rt.register_data(bytes(4 * n), n, hf.ValueType.FLOAT32, "w")
    return i, o, {"input": i, "output": o, "count": n}


def clean_bytes():
    rt, task = runtime(three_units())
    _, o, a = args_for(rt)
    rt.invoke(task, a, PERF)
    return rt.read_area(o)


# ---- executor ----------------------------------------------------------------------

class TestTransparency:
    @pytest.mark.parametrize("over", [{"cpu0": {"abort_prob": 1.0}}, {"cpu0": {"api_error_prob": 1.0}},
                                      {"cpu0": {"hang_prob": 1.0}},
                                      {"cpu0": {"abort_prob": 0.5, "seed": 3}, "gpu1": {"api_error_prob": 0.5, "seed": 5}}])
    def test_perfcp_result_equals_fault_free_run(self, over):
        rt, task = runtime(three_units(**over))
        _, o, a = args_for(rt)
        rep = rt.invoke(task, a, PERFCP)
        assert rep.success
        assert rt.read_area(o) == clean_bytes()

    def test_certain_abort_costs_one_retry(self):
        rt, task = runtime(three_units(cpu0={"abort_prob": 1.0}))
        _, _, a = args_for(rt)
        rep = rt.invoke(task, a, PERFCP)
        assert rep.attempts == 2 and rep.fault_counts["abort"] == 1


class TestPerf:
    def test_direct_fault_surfaces(self):
        rt, task = runtime(three_units(cpu0={"abort_prob": 1.0}))
        _, _, a = args_for(rt)
        with pytest.raises(hf.TaskFaultError) as e:
            rt.invoke(task, a, PERF)
        assert e.value.fault_class == "abort"

    def test_corruption_commits_silently(self):
        rt, task = runtime(three_units(cpu0={"corrupt_prob": 1.0}))
        _, o, a = args_for(rt)
        assert rt.invoke(task, a, PERF).success
        assert np.count_nonzero(rt.read_array(o) != DATA + 1) == 1


class TestTimeouts:
    def test_hang_charged_r_times_factor(self):
        rt, task = runtime(three_units(cpu0={"hang_prob": 1.0}))
        for k, u, r in (("inc_cpu", "cpu0", 200_000), ("inc_gpu", "gpu1", 400_000), ("inc_gpu", "gpu2", 401_000)):
            rt.profiles.record_outcome(rt.profiles.key_for(k, N, u), True, r)
        _, o, a = args_for(rt)
        rep = rt.invoke(task, a, hf.Strategy(hf.StrategyKind.PERF_CP, timeout_factor=3.0))
        assert rep.fault_counts["timeout"] == 1
        assert rep.compute_ns == 3 * 200_000 + rt.fleet.units["gpu1"].speed.runtime_ns(N)
        assert rt.read_area(o) == clean_bytes()

    def test_underestimated_deadline_is_a_spurious_timeout(self):
        rt, task = runtime(three_units())
        rt.profiles.record_outcome(rt.profiles.key_for("inc_cpu", N, "cpu0"), True, 1_000)
        for u in ("gpu1", "gpu2"):
            rt.profiles.record_outcome(rt.profiles.key_for("inc_gpu", N, u), True, 400_000)
        _, o, a = args_for(rt)
        rep = rt.invoke(task, a, PERFCP)
        assert rep.success and rep.fault_counts["timeout"] == 1
        assert rt.read_area(o) == clean_bytes()


class TestAccounting:
    def test_total_is_sum_of_parts(self):
        rt, task = runtime(three_units(cpu0={"abort_prob": 0.5}))
        for _ in range(8):
            _, _, a = args_for(rt)
            rep = rt.invoke(task, a, PERFCP)
            assert rep.total_ns == sum(rep.breakdown().values())

    def test_dmr_round_costs_slowest_replica(self):
        rt, task = runtime(three_units())
        for k, u, r in (("inc_cpu", "cpu0", 10_000_000), ("inc_gpu", "gpu1", 20_000), ("inc_gpu", "gpu2", 30_000)):
            rt.profiles.record_outcome(rt.profiles.key_for(k, N, u), True, r)
        _, _, a = args_for(rt)
        rep = rt.invoke(task, a, DMR)
        units = rt.fleet.units
        assert rep.compute_ns == max(units["gpu1"].speed.runtime_ns(N), units["gpu2"].speed.runtime_ns(N))
        assert rep.voter_ns > 0


class TestRedundancy:
    def test_dmr_catches_corruption_and_revotes(self):
        rt, task = runtime(three_units(gpu1={"corrupt_prob": 1.0}))
        _, o, a = args_for(rt)
        rep = rt.invoke(task, a, DMR)
        assert rep.success and rep.votes == ["mismatch", "match"]
        assert rep.fault_counts["vote_mismatch"] == 1
        assert np.array_equal(rt.read_array(o), DATA + 1)
        for k, u in (("inc_cpu", "cpu0"), ("inc_gpu", "gpu1")):
            rec = rt.profiles.record(rt.profiles.key_for(k, N, u))
            assert rec.t - rec.v == 1       # both replicas of the mismatching pair penalised

    def test_direct_fault_refills_one_slot(self):
        rt, task = runtime(three_units(cpu0={"abort_prob": 1.0}))
        _, o, a = args_for(rt)
        rep = rt.invoke(task, a, DMR)
        assert rep.success and rep.votes[-1] == "match" and rep.fault_counts["abort"] >= 1
        assert np.array_equal(rt.read_array(o), DATA + 1)

    def test_serial_and_threaded_replicas_agree(self):
        def run(serial):
            rt, task = runtime(three_units(gpu1={"corrupt_prob": 1.0}), hf.RuntimeConfig(serial_replicas=serial))
            _, o, a = args_for(rt)
            rep = rt.invoke(task, a, DMR)
            rt.close()
            return rt.read_area(o), rep.total_ns, rep.attempts, tuple(rep.votes)
        assert run(True) == run(False)

    def test_tmr_corrects_a_minority_without_rerun(self):
        rt, task = runtime(three_units(gpu1={"corrupt_prob": 1.0, "corrupt_rel_magnitude": 0.5}))
        _, o, a = args_for(rt)
        rep = rt.invoke(task, a, TMR)
        assert rep.success and rep.votes == ["corrected"] and rep.rounds == 1
        log = rep.rounds_log[0]
        assert log["mismatch"][log["slots"].index("gpu1")] == 1
        assert np.array_equal(rt.read_array(o), DATA + 1)

    def test_het_dmr_requires_distinct_kernels(self):
        cfg = fleet_cfg([{"id": "g1", "kind": "gpu", "memory_space": "m1"},
                         {"id": "g2", "kind": "gpu", "memory_space": "m2"}])
        rt, task = runtime(cfg, kinds=("gpu",))
        _, _, a = args_for(rt)
        with pytest.raises(hf.StrategyInfeasibleError):
            rt.invoke(task, a, hf.Strategy(hf.StrategyKind.HET_DMR))


class TestIsolation:
    def all_abort(self):
        return three_units(cpu0={"abort_prob": 1.0}, gpu1={"abort_prob": 1.0}, gpu2={"abort_prob": 1.0})

    def test_faulty_attempts_never_touch_committed_state(self):
        rt, task = runtime(self.all_abort(), hf.RuntimeConfig(attempt_limit=6))
        i, o, a = args_for(rt)
        before = rt.memory.payload_snapshot()
        with pytest.raises(hf.UnrecoverableTaskError):
            rt.invoke(task, a, PERFCP)
        after = rt.memory.payload_snapshot()
        for key, (v0, ok0, d0) in before.items():
            v1, ok1, d1 = after[key]
            assert v1 == v0 and (not ok1 or d1 == d0)
        assert rt.read_area(i) == DATA.tobytes() and rt.read_area(o) == bytes(4 * N)

    def test_attempt_budget(self):
        rt, task = runtime(self.all_abort(), hf.RuntimeConfig(attempt_limit=5))
        _, _, a = args_for(rt)
        with pytest.raises(hf.UnrecoverableTaskError):
            rt.invoke(task, a, PERFCP)
        assert sum(r.t for _, r in rt.profiles.items()) == 5

    def test_read_views_are_frozen(self):
        rt, _ = runtime(three_units())

        def hostile(ctx):
            ctx.request("input", "r")[0] = 99.0

        task = rt.declare_task("hostile", (hf.Param.area("input", "r"), hf.Param.scalar("count")))
        rt.attach_kernel(task, "h", "cpu", hostile)
        data = np.ones(4, dtype=np.float32)
        i = rt.register_data(data.tobytes(), 4, hf.ValueType.FLOAT32, "r")
        with pytest.raises(hf.UnrecoverableTaskError):
            rt.invoke(task, {"input": i, "count": 4}, PERFCP)
        assert rt.read_area(i) == data.tobytes()


def test_trace_kinds():
    lines = []
    rt, task = runtime(three_units(), hf.RuntimeConfig(trace=lines.append))
    _, _, a = args_for(rt)
    rt.invoke(task, a, DMR)
    assert {ln.split()[0] for ln in lines} == {"ATT", "VOTE", "DONE"}
    assert any("verdict=match" in ln for ln in lines)


# ---- memory protocol -------------------------------------------------------------------

@pytest.fixture
def mm():
    return hf.MemoryManager(hf.load_fleet(three_units()), HostBackend())


def test_register_buffer_checks_like_register(mm):
    """Zero-copy registration (register_host_buffer / register_device_data)
    applies register()'s checks (reference memory.py:88-101): no empty
    areas, known value type and mode, a buffer large enough for the
    elements."""
    from host_backend import _HostBytes
    buf = _HostBytes(16)
    assert mm.register_buffer(buf, 4, hf.ValueType.FLOAT32, "r")
    for args in ((0, hf.ValueType.FLOAT32, "r"), (5, hf.ValueType.FLOAT32, "r"), (4, "float32", "r"),
                 (4, hf.ValueType.FLOAT32, "x"), (17, hf.ValueType.INT, "r")):
        with pytest.raises(hf.RegistrationError):
            mm.register_buffer(buf, *args)


def floats(n, start=0.0):
    return np.arange(start, start + n, dtype=np.float32).tobytes()


class _WaitRecorder(HostBackend):
    """Host double that records every (stream, event) wait."""

    def __init__(self):
        super().__init__()
        self.waits = []

    def wait(self, stream, event):
        self.waits.append((stream, event))


def test_readers_of_a_voted_area_wait_on_its_vote_once():
    """Votes run on their own stream (CudaBackend.vote_stream), so the memory
    manager orders the compute stream after a committed sibling's `ready`
    event before the first copy-in, checkpoint or read of it, and only once
    per commit (Sibling.ready_seen)."""
    be = _WaitRecorder()
    m = hf.MemoryManager(hf.load_fleet(three_units()), be)
    a = m.register(floats(8), 8, hf.ValueType.FLOAT32, "w")
    h = m.request(a, "gpu1mem", "w")
    h.ready_event = "vote-event-1"
    m.commit_success([h])
    be.waits.clear()
    m.request(a, "gpu1mem", "r")
    m.request(a, "gpu1mem", "r", protect=True)      # sole copy: checkpointed, no second wait
    m.request(a, "host", "r")
    assert [e for _, e in be.waits] == ["vote-event-1"], be.waits
    h2 = m.request(a, "gpu1mem", "w")
    h2.ready_event = "vote-event-2"
    m.commit_success([h2])
    be.waits.clear()
    m.request(a, "host", "r")
    assert [e for _, e in be.waits] == ["vote-event-2"], be.waits


class TestMemory:
    def test_sole_device_copy_backed_up_before_protected_write(self, mm):
        a = mm.register(floats(1000), 1000, hf.ValueType.FLOAT32, "w")
        h = mm.request(a, "gpu1mem", "w")
        h.payload[:] = np.frombuffer(floats(1000, 9.0), np.uint8)
        mm.commit_success([h])
        h2 = mm.request(a, "gpu1mem", "w", protect=True)
        assert h2.checkpoint_ns == round(4 * 1000 * 0.01)
        assert (a, "host", 1, True) in mm.sibling_table()
        mm.invalidate(a, "gpu1mem")
        r = mm.request(a, "host", "r")
        assert r.base_version == 1 and mm.payload_bytes(r) == floats(1000, 9.0)

    def test_no_backup_when_a_copy_survives(self, mm):
        a = mm.register(floats(8), 8, hf.ValueType.FLOAT32, "w")
        assert mm.request(a, "gpu1mem", "w", protect=True).checkpoint_ns == 0
        assert mm.request(a, "host", "w", protect=True).checkpoint_ns == 0

    def test_fig1_replay(self, mm):
        i = mm.register(floats(8), 8, hf.ValueType.FLOAT32, "r")
        o = mm.register(floats(8), 8, hf.ValueType.FLOAT32, "w")
        mm.request(i, "gpu1mem", "r", protect=True)
        mm.request(o, "gpu1mem", "w", protect=True)
        mm.invalidate(i, "gpu1mem")
        mm.invalidate(o, "gpu1mem")
        hi = mm.request(i, "gpu2mem", "r", protect=True)
        ho = mm.request(o, "gpu2mem", "w", protect=True)
        ho.payload[:] = np.frombuffer(floats(8, 1.0), np.uint8)
        mm.commit_success([hi, ho])
        assert mm.request(o, "host", "r").source_space == "gpu2mem"
        assert mm.sibling_table() == [(i, "gpu1mem", 0, False), (i, "gpu2mem", 0, True), (i, "host", 0, True),
                                      (o, "gpu1mem", 0, False), (o, "gpu2mem", 1, True), (o, "host", 1, True)]

    def test_errors(self, mm):
        with pytest.raises(hf.UnknownAreaError):
            mm.request("nope", "host", "r")
        a = mm.register(floats(4), 4, hf.ValueType.FLOAT32, "r")
        with pytest.raises(hf.UnknownSpaceError):
            mm.request(a, "mars", "r")
        with pytest.raises(hf.UnknownSiblingError):
            mm.invalidate(a, "gpu1mem")
        mm.invalidate(a, "host")
        with pytest.raises(hf.DataLossError):
            mm.request(a, "host", "r")
        with pytest.raises(hf.RegistrationError):
            mm.register(b"123", 1, hf.ValueType.FLOAT32, "r")

    @pytest.mark.parametrize("seed", range(300))
    def test_random_sequences_match_model(self, seed):
        fleet = hf.load_fleet(three_units())
        m = hf.MemoryManager(fleet, HostBackend())
        ref = memory_model.SiblingModel("host")
        rng = random.Random(seed)
        spaces = ["host", "gpu1mem", "gpu2mem"]
        areas = []
        for _ in range(40):
            op = rng.choice(["reg", "read", "read", "write", "write", "fault", "inval"])
            if op == "reg" or not areas:
                if len(areas) < 3:
                    size = rng.randint(1, 8)
                    payload = bytes(rng.randrange(256) for _ in range(size))
                    areas.append((m.register(payload, size, hf.ValueType.INT, "rw"), ref.register(payload), size))
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
                    h.payload[:len(new)] = np.frombuffer(new, np.uint8)
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


# ---- mapper ------------------------------------------------------------------------------

class TestMapper:
    def test_fault_aware_estimate_exact(self):
        est = hf.fault_aware_estimate(1.0, 1, 4)
        assert est.p_exact == Fraction(3, 4) and est.F_exact == 4 and est.F == 4.0
        assert math.isinf(hf.fault_aware_estimate(5.0, 0, 3).F)

    def test_crossover_at_two_thirds(self):
        # fast-but-flaky (R = 1) vs 3x slower clean unit: equal F at p = 2/3
        fast = hf.fault_aware_estimate(1.0, 1, 3)
        slow = hf.fault_aware_estimate(3.0, 1, 1)
        assert fast.F_exact == slow.F_exact

    def test_quarantined_everything_still_spends_the_budget(self):
        cfg = three_units(cpu0={"abort_prob": 1.0}, gpu1={"abort_prob": 1.0}, gpu2={"abort_prob": 1.0})
        rt, task = runtime(cfg, hf.RuntimeConfig(attempt_limit=9, check_interval=50))
        _, _, a = args_for(rt)
        with pytest.raises(hf.UnrecoverableTaskError):
            rt.invoke(task, a, PERFCP)
        assert sum(r.t for _, r in rt.profiles.items()) == 9

    def test_nmr_groups_use_distinct_units(self):
        cfg = fleet_cfg([{"id": f"g{i}", "kind": "gpu", "memory_space": f"m{i}"} for i in range(5)])
        fleet = hf.load_fleet(cfg)
        mapper = hf.Mapper(fleet, hf.ProfileDB())
        cands = [hf.Selection("k", f"g{i}") for i in range(5)]
        d = mapper.select(hf.Strategy(hf.StrategyKind.DMR, replicas=5), 10, cands)
        assert len({s.unit_id for s in d.selections}) == 5
        with pytest.raises(hf.StrategyInfeasibleError):
            mapper.select(hf.Strategy(hf.StrategyKind.DMR, replicas=6), 10, cands)


# ---- devices / fleets ------------------------------------------------------------------------

class TestFleet:
    def test_loader_validation_names_fields(self):
        cfg = three_units()
        cfg["units"][1]["memory_space"] = "nowhere"
        with pytest.raises(hf.ConfigError, match=r"units\[1\].memory_space"):
            hf.load_fleet(cfg)
        cfg = three_units()
        cfg["memory_spaces"][0]["host"] = False
        with pytest.raises(hf.ConfigError, match="host"):
            hf.load_fleet(cfg)
        with pytest.raises(hf.ConfigError, match="device"):
            hf.load_fleet({"memory_spaces": [{"id": "h", "host": True}, {"id": "g", "device": -1}],
                           "units": [{"id": "u", "kind": "k", "memory_space": "g"}]})

    def test_gpu_fleet_units_share_one_space_per_device(self):
        fleet = hf.load_fleet(hf.gpu_fleet_config(devices=(0, 1)))
        assert sorted(fleet.units) == ["gpu0.simt", "gpu0.tc", "gpu1.simt", "gpu1.tc"]
        assert fleet.units["gpu1.tc"].device == 1 and fleet.units["gpu1.tc"].memory_space == "gpu1mem"
        assert fleet.units["gpu0.simt"].timing == "measured"

    def test_fault_frequencies_three_sigma(self):
        probs = dict(abort_prob=0.10, api_error_prob=0.05, hang_prob=0.05, corrupt_prob=0.10)
        u = hf.ProcessingUnit("u", "cpu", "host", hf.SpeedProfile(1000), hf.FaultModel(rng_seed=7, **probs))
        n = 20_000
        counts = {c: 0 for c in hf.FaultClass}
        for _ in range(n):
            f = u.draw_fault()
            if f is not None:
                counts[f] += 1
        for cls, p in zip(hf.FaultClass, probs.values()):
            assert abs(counts[cls] / n - p) <= 3 * math.sqrt(p * (1 - p) / n)


def test_voter_placement_follows_cost_model():
    fleet = hf.load_fleet(three_units())
    cfg = hf.VoterConfig()
    assert hf.place_voter(fleet, cfg, [(1_000, "host", "host")]).kernel == "voter_single"
    assert hf.place_voter(fleet, cfg, [(50_000, "host", "host")]).kernel == "voter_parallel"
    assert hf.place_voter(fleet, cfg, [(1_000_000, "host", "host")]).kernel == "voter_gpu"
    avoid = hf.VoterConfig(placement="avoid-task-units")
    assert hf.place_voter(fleet, avoid, [(1_000_000, "gpu1mem", "gpu2mem")], task_units=["gpu1", "gpu2"]).unit_id == "cpu0"


# ---- pipelined task stream ------------------------------------------------------------------

class TestTaskStream:
    def _run(self, depth, over):
        rt, task = runtime(three_units(**over), hf.RuntimeConfig(serial_replicas=True))
        outs = []
        with rt.task_stream(depth=depth) as ts:
            for t in range(12):
                data = np.full(N, t, dtype=np.float32)
                i = rt.register_data(data.tobytes(), N, hf.ValueType.FLOAT32, "r")
                o = rt.register_data(bytes(4 * N), N, hf.ValueType.FLOAT32, "w")
                ts.submit(task, {"input": i, "output": o, "count": N}, DMR)
                outs.append((o, data))
        return rt, [rt.read_array(o) for o, _ in outs], [d + 1 for _, d in outs]

    @pytest.mark.parametrize("depth", [0, 1, 3])
    def test_stream_commits_every_task(self, depth):
        rt, got, want = self._run(depth, {"gpu1": {"corrupt_prob": 0.4, "corrupt_rel_magnitude": 0.5}})
        for g, w in zip(got, want):
            assert np.array_equal(g, w)

    def test_stream_respects_data_dependencies(self):
        rt, _ = runtime(three_units())
        task = rt.declare_task("bump", (hf.Param.area("data", "rw"), hf.Param.scalar("count")))

        def bump(ctx):
            d = ctx.request("data", "rw")
            d[:ctx.arg("count")] += np.float32(1.0)

        for k in ("cpu", "gpu"):
            rt.attach_kernel(task, f"bump_{k}", k, bump)
        area = rt.register_data(np.zeros(N, dtype=np.float32).tobytes(), N, hf.ValueType.FLOAT32, "rw")
        with rt.task_stream(depth=3) as ts:
            for _ in range(5):      # each task reads what the previous one committed
                ts.submit(task, {"data": area, "count": N}, DMR)
        assert np.array_equal(rt.read_array(area), np.full(N, 5.0, dtype=np.float32))

    def test_rounds_log_carries_launch_order(self):
        rt, task = runtime(three_units())
        with rt.task_stream(depth=1) as ts:
            reps = []
            for t in range(4):
                i, o, a = args_for(rt)
                reps.append(ts.submit(task, a, DMR))
        seqs = [log["seq"] for r in reps for log in r.rounds_log]
        assert seqs == sorted(seqs) and len(set(seqs)) == len(seqs)


def test_overwrite_area_skips_zero_fill_only_when_declared():
    """Param.area(..., overwrites=True) (new) leaves a "w" provisional buffer
    uninitialised; plain "w" keeps the reference's zeroed buffer
    (memory.py:168), and overwrites is rejected for r/rw areas."""
    with pytest.raises(hf.DeclarationError):
        hf.Param.area("x", "rw", overwrites=True)
    calls = []

    class Spy(HostBackend):
        def alloc(self, space, nbytes, zero=True):
            calls.append(zero)
            return super().alloc(space, nbytes, zero)

    m = hf.MemoryManager(hf.load_fleet(three_units()), Spy())
    a = m.register(bytes(16), 4, hf.ValueType.FLOAT32, "w")
    m.request(a, "host", "w", protect=False)
    m.request(a, "host", "w", protect=False, zero_fill=False)
    assert calls == [True, False]


def test_overwrite_flag_reaches_the_bound_task():
    rt = hf.Runtime(hf.load_fleet(three_units()), backend=HostBackend())
    t = rt.declare_task("t", (hf.Param.area("x", "r"), hf.Param.area("y", "w", overwrites=True),
                              hf.Param.scalar("count")))
    rt.attach_kernel(t, "k", "cpu", lambda ctx: None)
    bound, _ = rt._bind(t, {"x": rt.register_data(bytes(16), 4, hf.ValueType.FLOAT32, "r"),
                            "y": rt.register_data(bytes(16), 4, hf.ValueType.FLOAT32, "w"), "count": 4},
                        None, None)
    assert [p.overwrites for p in bound.params] == [False, True, False]


# ---- commit preference (attach_kernel fidelity) ------------------------------------

def _scaled_inc(scale):
    def body(ctx):
        n = ctx.arg("count")
        src = ctx.request("input", "r")[:n]
        ctx.request("output", "w")[:n] = (src + np.float32(1.0)) * np.float32(scale)
    return body


class TestCommitFidelity:
    """A passing vote commits the agreeing replica of the best (lowest)
    fidelity rank; K >= 3 votes prefer its values.  Default ranks keep the
    reference's slot-0 commit (executor.py:268-274)."""

    def _rt(self, fid, kinds=("cpu", "gpu")):
        rt = hf.Runtime(hf.load_fleet(three_units()), hf.RuntimeConfig(), backend=HostBackend())
        task = rt.declare_task("inc", IO)
        # the variants agree within δ = 1e-3 but are bitwise distinct
        scale = {"cpu": 1.0, "gpu": 1.0 + 2 ** -12}
        for k in kinds:
            rt.attach_kernel(task, f"inc_{k}", k, _scaled_inc(scale[k]), fidelity=fid.get(k, 0))
        return rt, task

    def test_default_ranks_commit_slot_zero(self):
        rt, task = self._rt({})
        _, o, a = args_for(rt)
        rep = rt.invoke(task, a, DMR)
        assert rep.votes == ["match"]
        slot0 = rep.rounds_log[0]["slots"][0]
        assert rep.committed.unit_id == slot0

    @pytest.mark.parametrize("best", ["cpu", "gpu"], ids=["best-host", "best-accel"])
    def test_dmr_commits_best_fidelity_replica_bitwise(self, best):
        rt, task = self._rt({best: 0, ("gpu" if best == "cpu" else "cpu"): 5})
        _, o, a = args_for(rt)
        rep = rt.invoke(task, a, DMR)
        assert rep.votes == ["match"] and rep.committed.kernel == f"inc_{best}"
        scale = 1.0 if best == "cpu" else 1.0 + 2 ** -12
        want = ((DATA + np.float32(1.0)) * np.float32(scale)).astype(np.float32)
        assert rt.read_area(o) == want.tobytes()

    def test_tmr_corrected_lands_in_best_replica_slot_order_counts(self):
        cfg = three_units(gpu2={"corrupt_prob": 1.0, "corrupt_rel_magnitude": 0.5, "corrupt_element": 3})
        rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(), backend=HostBackend())
        task = rt.declare_task("inc", IO)
        rt.attach_kernel(task, "inc_cpu", "cpu", _scaled_inc(1.0), fidelity=1)
        rt.attach_kernel(task, "inc_gpu", "gpu", _scaled_inc(1.0 + 2 ** -12), fidelity=0)
        _, o, a = args_for(rt)
        rep = rt.invoke(task, a, TMR)
        assert rep.votes == ["corrected"]
        log = rep.rounds_log[0]
        # counts stay in slot order: only gpu2's slot mismatches
        assert log["mismatch"][log["slots"].index("gpu2")] == 1 and sum(log["mismatch"]) == 1
        assert rep.committed.unit_id == "gpu1"
        got = np.frombuffer(rt.read_area(o), dtype=np.float32)
        want = ((DATA + np.float32(1.0)) * np.float32(1.0 + 2 ** -12)).astype(np.float32)
        assert got.tobytes() == want.tobytes()


class TestDispatchCost:
    """attach_kernel(cost=...) orders a round's launches longest first (the
    lead replica on a shared GPU); without a cost on every variant the
    measured mean runtimes order them, as before."""

    def _rt(self, costs):
        rt = hf.Runtime(hf.load_fleet(three_units()), hf.RuntimeConfig(serial_replicas=True),
                        backend=HostBackend())
        task = rt.declare_task("inc", IO)
        calls = []

        def body_of(k):
            inner = _scaled_inc(1.0)

            def body(ctx):
                calls.append(k)
                inner(ctx)
            return body
        for k in ("cpu", "gpu"):
            rt.attach_kernel(task, f"inc_{k}", k, body_of(k), cost=costs.get(k, 0.0))
        return rt, task, calls

    @pytest.mark.parametrize("heavy", ["cpu", "gpu"])
    def test_cost_orders_launches(self, heavy):
        rt, task, calls = self._rt({heavy: 5.0, ("gpu" if heavy == "cpu" else "cpu"): 1.0})
        _, o, a = args_for(rt)
        for _ in range(3):
            rep = rt.invoke(task, a, hf.Strategy(hf.StrategyKind.HET_DMR))
            assert rep.success
            assert calls[-2] == heavy, calls
        assert len(calls) == 6

    def test_negative_cost_rejected(self):
        rt = hf.Runtime(hf.load_fleet(three_units()), hf.RuntimeConfig(), backend=HostBackend())
        task = rt.declare_task("inc", IO)
        with pytest.raises(hf.DeclarationError):
            rt.attach_kernel(task, "inc_cpu", "cpu", _scaled_inc(1.0), cost=-1.0)

    def test_matmul_workload_declares_costs(self):
        from paper_1405_2912_b200 import workloads
        assert max(workloads.MATMUL_COST, key=workloads.MATMUL_COST.get) == "mm_simt"


# ---- learnt voter cost (VoterCostModel) ---------------------------------------------

def test_voter_cost_model_fits_measured_line():
    m = hf.voting.VoterCostModel()
    for nbytes in (1 << 20, 1 << 24, 1 << 26, 1 << 24):
        m.observe("hf_vote", "gpu-simt", nbytes, round(2_000 + nbytes / 800))    # 800 B/ns = 0.8 TB/s
    base, per = m.fit("hf_vote", "gpu-simt")
    assert abs(base - 2_000) < 2 and abs(per * 800 - 1) < 1e-4
    prof = hf.VoterKernelProfile("hf_vote", "gpu-simt", 10_000, 1.0)
    m.apply([prof])
    assert prof.base_ns == round(base) and prof.per_byte_ns == per


def test_voter_cost_model_single_size_uses_mean_rate_and_keeps_base():
    m = hf.voting.VoterCostModel()
    assert m.observe("hf_vote", "*", 1000, 500)          # first observation: refit
    assert m.fit("hf_vote", "*") == (None, 0.5)
    prof = hf.VoterKernelProfile("hf_vote", "*", 7, 9.0)
    m.apply([prof])
    assert (prof.base_ns, prof.per_byte_ns) == (7, 0.5)
    assert m.fit("hf_vote", "cpu") is None


def test_nvtx_ranges_are_noops_unless_enabled():
    from paper_1405_2912_b200 import nvtx
    assert nvtx.ENABLED is False            # HETFT_NVTX unset in the test environment
    with nvtx.range("x"):
        pass


def test_nvtx_enabled_pushes_and_pops(monkeypatch):
    from paper_1405_2912_b200 import nvtx
    calls = []
    monkeypatch.setattr(nvtx, "ENABLED", True)
    monkeypatch.setattr(nvtx, "_push", lambda name: calls.append(("push", name)))
    monkeypatch.setattr(nvtx, "_pop", lambda: calls.append(("pop",)))
    rt, task = runtime(three_units())
    _, _, a = args_for(rt)
    assert rt.invoke(task, a, DMR).success
    names = [c[1] for c in calls if c[0] == "push"]
    assert calls.count(("pop",)) == len(names)
    assert any(n.startswith("hetft.vote") for n in names) and any(n.startswith("hetft.replica") for n in names)
    assert any(n.startswith("hetft.settle") for n in names) and any(n.startswith("hetft.advance") for n in names)
