"""Standalone times of the tensor-core variants at 4096^3: CTA-pair TF32
(standalone shape) and the co-scheduling TF32 / 3xBF16 shapes, median of 20
CUDA-event timings each (pre-passes included)."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1405_2912_b200 import kernels  # noqa: E402
from paper_1405_2912_b200._lib import HF_GEMM_COSCHEDULE as CO, HF_GEMM_TF32, HF_GEMM_3XBF16  # noqa: E402

n = 4096
a = torch.rand(n, n, device="cuda") + 1
b = torch.rand(n, n, device="cuda") + 1
c = torch.empty(n, n, device="cuda")
out = {}
for name, mode in (("pair_tf32", HF_GEMM_TF32), ("cosched_tf32", HF_GEMM_TF32 | CO),
                   ("cosched_3xbf16", HF_GEMM_3XBF16 | CO), ("pair_3xbf16", HF_GEMM_3XBF16)):
    ts = []
    for i in range(25):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        kernels.gemm_tc(a, b, c, mode=mode)
        e1.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(e0.elapsed_time(e1))
    out[name] = round(statistics.median(ts), 4)
print(json.dumps(out))
