"""Built-in fleet configurations (reference fleets.py).

"default" and "pathfinder" are the reference's modelled presets — one CPU and
two GPUs with dedicated memories, virtual time from the speed profiles —
kept value for value so the reference's experiments replay here exactly
(tests/test_experiments.py).  The "b200*" presets are real devices: one
memory space per GPU and one measured logical unit per (GPU, kernel kind),
see devices.gpu_fleet_config.
"""

from __future__ import annotations

import copy
from pathlib import Path

from .devices import Fleet, gpu_fleet_config, load_fleet
from .errors import ConfigError

_MODEL_SPACES = [
    {"id": "host", "label": "host RAM", "host": True},
    {"id": "gpu1mem", "label": "GPU1 memory"},
    {"id": "gpu2mem", "label": "GPU2 memory"},
]


def _modelled(cpu, gpu1, gpu2, seeds) -> dict:
    """cpu/gpu1/gpu2 = (base latency us, per-element ns) — reference fleets.py:24-54."""
    units = []
    for (uid, kind, space), (base, per), seed in zip(
            (("cpu0", "cpu", "host"), ("gpu1", "gpu", "gpu1mem"), ("gpu2", "gpu", "gpu2mem")),
            (cpu, gpu1, gpu2), seeds):
        units.append({"id": uid, "kind": kind, "memory_space": space,
                      "base_latency_us": base, "per_elem_cost_ns": per, "seed": seed})
    return {"default_ns_per_byte": 0.005, "memory_spaces": copy.deepcopy(_MODEL_SPACES), "units": units}


def default_fleet_config() -> dict:
    """GPUs are the fast units."""
    return _modelled((100.0, 10.0), (20.0, 1.0), (30.0, 2.0), (11, 12, 13))


def pathfinder_fleet_config() -> dict:
    """The CPU kernel runs 3x faster than the best GPU: the fault-aware
    switchover sits at p = 1 - 1/3."""
    return _modelled((100.0, 10.0), (300.0, 30.0), (400.0, 40.0), (21, 22, 23))


def b200_fleet_config() -> dict:
    """One B200, three diverse matmul units (tcgen05 TF32, SIMT FP32,
    tcgen05 3xBF16) sharing its HBM, plus an HBM checkpoint space."""
    cfg = gpu_fleet_config(devices=(0,), kinds=("gpu-tc", "gpu-simt", "gpu-tc3"))
    cfg["memory_spaces"].append({"id": "gpu0ckpt", "label": "HBM checkpoint reserve", "device": 0})
    return cfg


def b200_replica_fleet_config(devices=(0, 1, 2), kinds=("gpu-simt", "gpu-tc", "gpu-tc3"),
                              checkpoint_device: int = None) -> dict:
    """BASELINE configs[2]: one variant kind per GPU — replica i's kernel
    kind runs only on GPU devices[i] (unit "r<i>.<kind>" in space "r<i>mem"),
    so a heterogeneous strategy (distinct kernels) necessarily places its
    replicas on distinct GPUs.  The SIMT variant, the long pole of a round,
    sits on devices[0] next to the inputs; the tensor-core variants pull the
    inputs over NVLink and finish long before it.  Optional HBM checkpoint
    space "ckpt" on `checkpoint_device` (default devices[0]).  `devices` may
    repeat an ordinal: (0, 0, 0) keeps the per-replica spaces and the copies
    between them on one GPU (the code path of this preset on a 1-GPU box)."""
    if len(devices) != len(kinds):
        raise ConfigError(f"b200 replica fleet: {len(devices)} devices for {len(kinds)} kinds")
    spaces = [{"id": "host", "label": "pinned host RAM", "host": True}]
    units = []
    for i, (d, kind) in enumerate(zip(devices, kinds)):
        spaces.append({"id": f"r{i}mem", "device": int(d), "label": f"replica {i} HBM (GPU {d})"})
        units.append({"id": f"r{i}.{kind.split('-', 1)[-1]}", "kind": kind, "memory_space": f"r{i}mem",
                      "timing": "measured", "seed": 2000 + 17 * i})
    cd = devices[0] if checkpoint_device is None else checkpoint_device
    spaces.append({"id": "ckpt", "device": int(cd), "label": f"HBM checkpoint reserve (GPU {cd})"})
    return {"memory_spaces": spaces, "units": units, "default_ns_per_byte": 0.0}


def b200_multi_fleet_config(n_gpus: int) -> dict:
    """n B200s, one memory space each; the same three kinds on every GPU."""
    return gpu_fleet_config(devices=tuple(range(n_gpus)), kinds=("gpu-tc", "gpu-simt", "gpu-tc3"))


BUILTIN_FLEETS = {
    "default": default_fleet_config,
    "pathfinder": pathfinder_fleet_config,
    "b200": b200_fleet_config,
    **{f"b200x{n}": (lambda n=n: b200_multi_fleet_config(n)) for n in (2, 3, 4, 8)},
    "b200-replicas3": b200_replica_fleet_config,
}


def fleet_config_from(source) -> dict:
    """Resolve a fleet argument: builtin name, config dict, or YAML path."""
    if isinstance(source, dict):
        return copy.deepcopy(source)
    name = str(source)
    if name in BUILTIN_FLEETS:
        return BUILTIN_FLEETS[name]()
    if Path(name).exists():
        import yaml
        with open(name, "r", encoding="utf-8") as fh:
            return yaml.safe_load(fh)
    raise ConfigError(f"unknown fleet {name!r}: not a builtin ({', '.join(sorted(BUILTIN_FLEETS))}) "
                      f"and no such file")


def build_fleet(source) -> Fleet:
    return load_fleet(fleet_config_from(source))
