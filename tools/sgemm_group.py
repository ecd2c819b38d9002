"""SIMT GEMM at 4096^3 under the HF_SGEMM_GROUP tile-row grouping in the
environment: CUDA-event time (for the DRAM traffic run it under ncu)."""
import json, os, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import kernels
n = 4096
a = torch.rand(n, n, device="cuda") + 1
b = torch.rand(n, n, device="cuda") + 1
c = torch.empty(n, n, device="cuda")
for _ in range(3):
    kernels.gemm_simt(a, b, c)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    kernels.gemm_simt(a, b, c)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 10
print(json.dumps({"group": os.environ.get("HF_SGEMM_GROUP", "8"), "ms": t, "tflops": 2 * n ** 3 / t / 1e9}))
