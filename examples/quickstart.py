"""A `hetrt` program switched to the B200 hot path: one HetTMR voted matmul
task on GPU 0 (tcgen05 TF32, SIMT FP32 and tcgen05 3xBF16 replicas), with the
tensor-core unit flipping one bit of its output, then a task stream.

    python examples/quickstart.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1405_2912_b200 as hetrt  # noqa: E402  (was: import hetrt)

n = 1024
rng = np.random.default_rng(0)
a = rng.uniform(1, 2, (n, n)).astype(np.float32)
b = rng.uniform(1, 2, (n, n)).astype(np.float32)

# one memory space per GPU and one logical unit per kernel variant; the
# tensor-core unit corrupts its output with a seeded single-bit flip
cfg = hetrt.gpu_fleet_config(devices=(0,), kinds=("gpu-tc", "gpu-simt", "gpu-tc3"),
                             **{"gpu0.tc": {"corrupt_prob": 1.0, "corrupt_mode": "bitflip", "corrupt_bit": 30}})
rt = hetrt.Runtime(hetrt.load_fleet(cfg))
task = hetrt.get_workload("matmul").attach(rt)          # declare_task + attach_kernel x 3

A = rt.register_data(a.tobytes(), n * n, hetrt.ValueType.FLOAT32, "r")
B = rt.register_data(b.tobytes(), n * n, hetrt.ValueType.FLOAT32, "r")
C = rt.register_data(bytes(4 * n * n), n * n, hetrt.ValueType.FLOAT32, "w")
report = rt.invoke(task, {"A": A, "B": B, "C": C, "n": n}, hetrt.Strategy(hetrt.StrategyKind.HET_TMR))
c = rt.read_array(C).reshape(n, n)
ref = a.astype(np.float64) @ b.astype(np.float64)
print("votes:", report.votes, "faulty replicas:", report.vote_outcomes[0].faulty,
      "rounds:", report.rounds, "max rel err:", float(np.max(np.abs(c - ref) / ref)))

# many tasks: keep the next task's kernels queued while the host settles one
with rt.task_stream(depth=1) as ts:
    reports = [ts.submit(task, {"A": A, "B": B, "C": C, "n": n}, hetrt.Strategy(hetrt.StrategyKind.HET_TMR))
               for _ in range(8)]
print("stream:", [r.votes[-1] for r in reports])
