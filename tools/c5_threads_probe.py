"""Lab: C5-shaped HetTMR 2048^2 task streams driven by T host threads in one
process, each thread with its own Runtime / TaskStream on the same GPU (the
GIL serialises the Python protocol; libhetft and most torch calls release
it).  Total tasks/s for T = 1, 2, 3."""
import json
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402

sys.argv = [sys.argv[0], "--n", "2048"]
args = bench.parse()
per = 1200
for T in (1, 2, 3):
    import paper_1405_2912_b200 as hf
    benches = [bench.TaskStreamBench(args, 0, 0, bench.TMR_KINDS, hf.Strategy(hf.StrategyKind.HET_TMR), seed_salt=w)
               for w in range(T)]
    for b in benches:
        b.warm()
    torch.cuda.synchronize()
    ths = [threading.Thread(target=b.device_stream, args=(per, False)) for b in benches]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"threads": T, "tasks": T * per, "tasks_per_s": T * per / dt}), flush=True)
    del benches
