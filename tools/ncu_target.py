"""Minimal driver for ncu captures: each hot kernel at the bench size, 3x."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import kernels  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
d = "cuda:0"
m = n * n
base = torch.rand(m, device=d) + 1
reps = [base * (1 + 1e-6 * torch.randn(m, device=d)) for _ in range(3)]
kernels.inject_bitflip(reps[2], m // 3, 27)
a, b = base.view(n, n), reps[1].view(n, n)
c = torch.empty(n, n, device=d)
dst = torch.empty_like(base)
for _ in range(3):
    kernels.gemm_simt(a, b, c)
    kernels.gemm_tc(a, b, c)                 # CTA-pair tf32
    kernels.gemm_tc(a, b, c, mode=2)         # CTA-pair 3xBF16 (kind::f16)
    kernels.gemm_tc(a, b, c, mode=0x100)     # single-CTA co-scheduling shape, tf32
    kernels.vote(reps[:2], 1e-3)
    kernels.vote(reps, 1e-3, voted=reps[0])
    kernels.checkpoint(dst, base)
torch.cuda.synchronize()
print("ok")
