"""What the third TMR replica costs: the bench's HetTMR stream (TF32, SIMT,
3xBF16) against a TMR stream whose third replica is a second TF32 unit
(distinct units, repeated kernel), same shape and fault rate.  Quantifies
DESIGN §8's "cheaper third variant" lever; not a product configuration."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402

sys.argv = [sys.argv[0], "--steps", "60"]
args = bench.parse()
out = {}
for name, kinds, strat in (("hettmr tf32+simt+3xbf16", bench.TMR_KINDS, "HET_TMR"),
                           ("tmr tf32+simt+tf32", ("gpu-tc", "gpu-simt", "gpu-tc"), "TMR")):
    import paper_1405_2912_b200 as hf
    cfg = hf.gpu_fleet_config(devices=(0,), kinds=("gpu-tc", "gpu-simt", "gpu-tc3"))
    if strat == "TMR":
        cfg["units"] = [u for u in cfg["units"] if u["kind"] != "gpu-tc3"]
        cfg["units"].append({"id": "gpu0.tc2", "kind": "gpu-tc", "memory_space": "gpu0mem", "timing": "measured",
                             "seed": 9001})
    cfg["memory_spaces"].append({"id": "gpu0ckpt", "device": 0})
    for i, u in enumerate(cfg["units"]):
        u.update({"corrupt_prob": 0.05, "corrupt_mode": "bitflip", "seed": 1_000_003 + i * 101 + 17})
    rt = hf.Runtime(hf.load_fleet(cfg), hf.RuntimeConfig(checkpoint_space="gpu0ckpt", serial_replicas=True,
                                                         attempt_limit=64))
    task = hf.get_workload("matmul").attach(rt)
    tb = bench.TaskStreamBench(args, 0, 0, None, hf.Strategy(getattr(hf.StrategyKind, strat)), built=(hf, rt, task))
    tb.warm()
    dt, _ = tb.timed(tb.device_stream, 60, True)
    out[name] = {"tasks_per_s": 60 / dt, "ms_per_task": dt / 60 * 1e3, "votes": tb.stats["votes"]}
    del tb, rt
    torch.cuda.synchronize()
print(json.dumps(out))
