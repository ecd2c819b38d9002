"""Lab (not product code): can a lean HBM-bound kernel (128-thread CTAs,
<= 32 registers, no smem) run beside the SIMT GEMM grid, or does it wait
for the grid's tail?  A long SIMT GEMM (8192^2, ~17 ms) on one stream, then,
once it is running, a 64 MiB checkpoint on another stream: the checkpoint's
own event-timed duration shows whether it ran at once (~30 us) or waited.

    HF_LEAN_STREAMS=0|1 python tools/coresidency_probe.py
"""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1405_2912_b200 import kernels  # noqa: E402
from paper_1405_2912_b200._lib import HF_GEMM_COSCHEDULE as CO  # noqa: E402

d = "cuda:0"
n = 8192
a = torch.rand(n, n, device=d) + 1
b = torch.rand(n, n, device=d) + 1
c = torch.empty(n, n, device=d)
src = torch.empty(64 << 20, dtype=torch.uint8, device=d)
dst = torch.empty_like(src)
s1 = torch.cuda.Stream(priority=-1)
s2 = torch.cuda.Stream(priority=int(os.environ.get("PROBE_PRIO", "0")))
out = {"lean": os.environ.get("HF_LEAN_STREAMS", "1"), "ckpt_stream_priority": os.environ.get("PROBE_PRIO", "0")}
for trial in range(3):
    torch.cuda.synchronize()
    e0, e1, e2, e3 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
    e0.record(s1)
    kernels.gemm_simt(a, b, c, mode=int(os.environ.get("PROBE_MODE", CO)), stream=s1)
    e1.record(s1)
    time.sleep(0.004)            # the grid is resident by now
    e2.record(s2)
    kernels.checkpoint(dst, src, stream=s2)
    e3.record(s2)
    torch.cuda.synchronize()
    out[f"t{trial}"] = {"simt_ms": e0.elapsed_time(e1), "ckpt_ms": e2.elapsed_time(e3),
                        "ckpt_end_before_simt_end_ms": e3.elapsed_time(e1)}
print(json.dumps(out))
