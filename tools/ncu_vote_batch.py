"""ncu driver for the batched voter: one hf_vote_batch launch of 32 K = 3
votes at 1 MiB, 4 MiB and 16 MiB each (diverse replicas), plus the same
16 MiB vote as one hf_vote_async for comparison."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import kernels  # noqa: E402

for mib in (1, 4, 16):
    n = mib << 18
    sets = []
    for _ in range(32):
        base = torch.rand(n, device="cuda") + 1
        sets.append([base * (1 + 1e-6 * torch.randn(n, device="cuda")) for _ in range(3)])
    wss = [kernels.VoteWorkspace(0) for _ in range(32)]
    kernels.VoteBatch([(r, None, w, None) for r, w in zip(sets, wss)], 1e-3).launch()
    if mib == 16:
        kernels.vote_async(sets[0], wss[0], 1e-3)
    torch.cuda.synchronize()
    del sets, wss
print("ok")
