"""Replica placement across GPUs (BASELINE configs[2]):
Strategy(spread="device") keeps the reference's distinct-unit (and, for
heterogeneous strategies, distinct-kernel) pair search
(/root/reference/pkg/src/hetrt/mapping.py:239-260) and additionally requires
the K replicas to sit on pairwise distinct CUDA devices; invoke/submit
``devices=`` restricts a task to a GPU group, which sharding.replica_group
rotates over a box.  Mapper-level tests need no GPU (load_fleet of a B200
fleet config only builds host objects)."""

import pytest

import paper_1405_2912_b200 as hf
from paper_1405_2912_b200 import sharding
from paper_1405_2912_b200.mapping import Mapper, Selection, TaskRetryState
from paper_1405_2912_b200.profiles import ProfileDB

KINDS = ("gpu-tc", "gpu-simt", "gpu-tc3")
KERNELS = {"gpu-tc": "mm_tc", "gpu-simt": "mm_simt", "gpu-tc3": "mm_tc3x"}


def fleet(n_gpus):
    return hf.load_fleet(hf.gpu_fleet_config(devices=tuple(range(n_gpus)), kinds=KINDS))


def candidates(fl, devices=None):
    out = []
    for kind in KINDS:
        out += [Selection(KERNELS[kind], uid) for uid in sorted(fl.units)
                if fl.units[uid].kind == kind and (devices is None or fl.units[uid].device in devices)]
    return out


def devs(fl, group):
    return [fl.units[s.unit_id].device for s in group]


def test_default_spread_may_stack_replicas_on_one_gpu():
    fl = fleet(3)
    m = Mapper(fl, ProfileDB())
    d = m.select(hf.Strategy(hf.StrategyKind.HET_TMR), 1 << 24, candidates(fl))
    # the reference rule only asks for distinct units: all three on GPU 0
    assert len({s.unit_id for s in d.selections}) == 3
    assert len(set(devs(fl, d.selections))) == 1


@pytest.mark.parametrize("kind", [hf.StrategyKind.HET_TMR, hf.StrategyKind.TMR, hf.StrategyKind.HET_DMR])
def test_spread_device_puts_each_replica_on_its_own_gpu(kind):
    fl = fleet(3)
    m = Mapper(fl, ProfileDB())
    st = hf.Strategy(kind, spread="device")
    d = m.select(st, 1 << 24, candidates(fl))
    k = st.n_replicas
    assert len(d.selections) == k
    assert len(set(devs(fl, d.selections))) == k
    if kind.heterogeneous:
        assert len({s.kernel for s in d.selections}) == k


def test_spread_device_infeasible_on_one_gpu_and_degrades_to_unit_spread():
    fl = fleet(1)
    m = Mapper(fl, ProfileDB())
    with pytest.raises(hf.StrategyInfeasibleError, match="distinct devices"):
        m.select(hf.Strategy(hf.StrategyKind.HET_TMR, spread="device"), 1 << 24, candidates(fl))
    d = m.select(hf.Strategy(hf.StrategyKind.HET_TMR, spread="device", degrade_on_infeasible=True),
                 1 << 24, candidates(fl))
    assert len(d.selections) == 3 and set(devs(fl, d.selections)) == {0}


def test_replace_replica_keeps_devices_distinct():
    fl = fleet(3)
    m = Mapper(fl, ProfileDB())
    st = hf.Strategy(hf.StrategyKind.HET_TMR, spread="device")
    d = m.select(st, 1 << 24, candidates(fl))
    state = TaskRetryState(attempt_limit=10)
    failed = d.selections[1]
    keep = [d.selections[0], d.selections[2]]
    new = m.replace_replica(st, 1 << 24, candidates(fl), state, failed, keep=keep)
    assert new != failed
    assert len(set(devs(fl, keep + [new]))) == 3


@pytest.mark.parametrize("world", [3, 4, 8])
def test_replica_group_rotation_places_task_t_on_its_gpu_group(world):
    fl = fleet(world)
    m = Mapper(fl, ProfileDB())
    st = hf.Strategy(hf.StrategyKind.HET_TMR, spread="device")
    load = [0] * world
    for t in range(2 * world):
        group = sharding.replica_group(t, world, 3)
        d = m.select(st, 1 << 22, candidates(fl, devices=group))
        got = devs(fl, d.selections)
        assert sorted(got) == sorted(group)
        for g in got:
            load[g] += 1
    # rotation balances the replica load: every GPU hosts K/G of it
    assert len(set(load)) == 1


def test_executor_candidates_honour_device_affinity():
    """Runtime.invoke/submit(devices=...) reaches the executor's candidate
    list (CPU check through the host test double)."""
    from host_backend import HostBackend
    rt = hf.Runtime(fleet(4), backend=HostBackend())
    task = hf.get_workload("matmul").attach(rt)
    bound, _ = rt._bind(task, {"A": rt.register_data(bytes(16), 4, hf.ValueType.FLOAT32, "r"),
                               "B": rt.register_data(bytes(16), 4, hf.ValueType.FLOAT32, "r"),
                               "C": rt.register_data(bytes(16), 4, hf.ValueType.FLOAT32, "w"), "n": 2},
                        None, None, devices=(1, 3))
    cands = rt.executor.candidates_for(bound)
    assert {rt.fleet.units[s.unit_id].device for s in cands} == {1, 3}
    assert len(cands) == 6


def test_spread_must_be_known():
    with pytest.raises(ValueError):
        hf.Strategy(hf.StrategyKind.TMR, spread="rack")
