"""Multi-GPU placement of the voted-task path.

Two ways the path spreads over the GPUs of one box, neither needing a
data-path collective:

* independent task streams (C5, weak scaling): rank r of a world of G owns
  tasks t with t mod G == r, or — when replicas live on distinct GPUs — task
  t uses the GPU group {(t + j) mod G : j < K}, rotating so every GPU hosts
  K/G of the replica load;
* replicas on distinct GPUs (C3): the vote of an n-element output is sliced:
  replica GPU i votes elements [lo_i, hi_i) reading the other K-1 replicas'
  slices over NVLink, so each GPU's ingress is (K-1)/K·n·s instead of
  (K-1)·n·s on one voter GPU.  Slice results combine exactly on the host:
  counts add, the first divergence is the minimum over slices (offset by the
  slice start), the winner is recomputed from the combined counts.

Only the timing uses a collective (barrier + max over ranks).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence


def task_owner(task_index: int, world: int) -> int:
    return task_index % world


def tasks_for_rank(n_tasks: int, rank: int, world: int) -> list:
    return [t for t in range(n_tasks) if task_owner(t, world) == rank]


def replica_group(task_index: int, world: int, k: int) -> list:
    """GPUs hosting the K replicas of task t (distinct when K <= world)."""
    return [(task_index + j) % world for j in range(k)]


def slice_bounds(n: int, parts: int, align: int = 4) -> list:
    """[lo, hi) element ranges, one per part, boundaries multiples of `align`
    elements so every slice keeps 16-byte vector alignment for fp32."""
    if parts <= 0:
        raise ValueError("parts must be positive")
    step = -(-n // parts)
    step = -(-step // align) * align
    out = []
    for i in range(parts):
        lo = min(n, i * step)
        hi = min(n, (i + 1) * step)
        out.append((lo, hi))
    return out


@dataclass
class SliceResult:
    """Per-slice vote outcome (indices relative to the slice)."""

    lo: int
    mismatch: list
    unresolved: int
    first_div: int          # -1 when the slice agrees everywhere
    first_raw0: Optional[int] = None   # replica 0's raw bits at first_div


@dataclass
class CombinedVote:
    verdict: str
    mismatch: list
    unresolved: int
    first_div: int
    winner: int
    first_raw0: Optional[int] = None

    @property
    def faulty(self) -> list:
        return [r for r, m in enumerate(self.mismatch) if m > 0]


def combine_slices(parts: Sequence[SliceResult], k: int) -> CombinedVote:
    """Exact combination of per-slice K-way votes (Appendix A is element-wise,
    so slicing cannot change any per-element decision)."""
    mism = [0] * k
    unres = 0
    first: Optional[int] = None
    raw0 = None
    for p in parts:
        for r in range(k):
            mism[r] += int(p.mismatch[r])
        unres += int(p.unresolved)
        if p.first_div >= 0:
            g = p.lo + int(p.first_div)
            if first is None or g < first:
                first, raw0 = g, p.first_raw0
    winner = min(range(k), key=lambda r: (mism[r], r))
    verdict = "mismatch" if unres else ("corrected" if any(mism) else "match")
    return CombinedVote(verdict, mism, unres, -1 if first is None else first, winner, raw0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a float over the default process group (gloo or nccl)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
