"""Minimal driver for ncu captures: each hot kernel once at the bench size,
in the launch shapes a one-GPU HetTMR task uses (co-scheduling flag) and the
standalone shapes of the roofline measurements."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import kernels  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps_ = int(sys.argv[2]) if len(sys.argv) > 2 else 1
d = "cuda:0"
m = n * n
base = torch.rand(m, device=d) + 1
reps = [base * (1 + 1e-6 * torch.randn(m, device=d)) for _ in range(3)]
kernels.inject_bitflip(reps[2], m // 3, 27)
a, b = base.view(n, n), reps[1].view(n, n)
c = torch.empty(n, n, device=d)
dst = torch.empty_like(base)
CO = 0x100
for _ in range(reps_):
    kernels.gemm_simt(a, b, c, mode=CO)      # in-task SIMT shape (blocked accumulation)
    kernels.gemm_tc(a, b, c, mode=CO)        # single-CTA co-scheduling shape, tf32
    kernels.gemm_tc(a, b, c, mode=2 | CO)    # co-scheduling shape, 3xBF16
    kernels.gemm_tc(a, b, c)                 # CTA-pair tf32 (standalone)
    kernels.vote(reps[:2], 1e-3)
    kernels.vote(reps, 1e-3, voted=reps[0])
    kernels.checkpoint(dst, base)
torch.cuda.synchronize()
print("ok")
