"""SIMT GEMM rate at shapes whose CTA count is an exact number of waves
(296 slots = 148 SMs x 2 CTAs) versus the 4096^3 task shape (3.46 waves):
separates the main loop's efficiency from the last partial wave."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1405_2912_b200 import kernels  # noqa: E402

out = []
for (m, k, n) in [(4096, 4096, 4096), (4736, 4096, 2048), (4736, 4096, 4096), (9472, 4096, 4096)]:
    a = torch.rand(m, k, device="cuda") + 1
    b = torch.rand(k, n, device="cuda") + 1
    c = torch.empty(m, n, device="cuda")
    ts = []
    for i in range(25):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        kernels.gemm_simt(a, b, c)
        e1.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    ctas = (m // 128) * (n // 128)
    out.append({"m": m, "k": k, "n": n, "ctas": ctas, "waves": ctas / 296, "ms": ms,
                "tflops": 2.0 * m * n * k / (ms * 1e-3) / 1e12})
    print(json.dumps(out[-1]), flush=True)
