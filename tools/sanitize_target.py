"""Small-shape driver that launches every libhetft kernel once, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python tools/sanitize_target.py
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import kernels as K  # noqa: E402
from paper_1405_2912_b200._lib import HF_GEMM_COSCHEDULE as CS  # noqa: E402

d = "cuda:0"
g = torch.Generator(device=d).manual_seed(5)
# GEMM variants: ragged, square, pair-kernel shapes with a tail split
for (m, n, k) in [(300, 520, 264), (512, 768, 256), (1024, 512, 128)]:
    a = torch.rand(m, k, device=d, generator=g) + 1
    b = torch.rand(k, n, device=d, generator=g) + 1
    c = torch.empty(m, n, device=d)
    for mode in (0, 1, 2, CS, CS | 1, CS | 2):
        K.gemm_tc(a, b, c, mode=mode)
    K.gemm_simt(a, b, c)
    K.gemm_simt(a, b, c, mode=CS)
# 2560 x 4096: 160 pair tiles -> deterministic tail split (4 k-ranges)
a = torch.rand(2560, 256, device=d, generator=g) + 1
b = torch.rand(256, 4096, device=d, generator=g) + 1
c = torch.empty(2560, 4096, device=d)
K.gemm_tc(a, b, c)
# voter: K = 2..5, aligned / unaligned / ragged, in-place voted output, ints
n = (1 << 20) + 3
base = torch.rand(n, device=d, generator=g) + 1
for k in (2, 3, 5):
    reps = [base.clone() for _ in range(k)]
    K.inject_bitflip(reps[-1], 1234, 27)
    K.vote(reps, 1e-3)
    K.vote(reps, 1e-3, voted=reps[0])
    K.vote([r[1:] for r in reps], 1e-3)
ints = [torch.randint(0, 1 << 30, (n,), device=d, dtype=torch.int32, generator=g) for _ in range(3)]
K.vote(ints, 0.0)
K.vote_bytes([x.view(torch.uint8)[: 12 * 1000] for x in ints], 12)
ws = K.VoteWorkspace(0)
K.vote_async([base, base.clone()], ws, 1e-3)
ws.read()
# round 2: K = 3 in place with the divergence in replica 0 (first-divergence
# records + leader epilogue), and a batched launch of mixed sizes
reps = [base.clone() for _ in range(3)]
K.inject_bitflip(reps[0], 777, 30)
K.inject_bitflip(reps[2], 70_000, 29)
r3 = K.vote(reps, 1e-3, voted=reps[0])
assert r3.first_div == 777 and r3.first_raw0 is not None
items = []
for m_ in (1, 17, 5000, 1 << 16, (1 << 18) + 5):
    rr = [base[:m_].clone() for _ in range(3)]
    K.inject_bitflip(rr[1], m_ // 2, 30)
    items.append((rr, rr[0], K.VoteWorkspace(0), None))
K.vote_batch(items, 1e-3)
for it in items:
    it[2].read()
# empty votes (r2): async n = 0, and a batch mixing empty and non-empty items
empty = [torch.empty(0, device=d) for _ in range(3)]
ws_e = K.VoteWorkspace(0)
K.vote_async(empty, ws_e, 1e-3)
assert ws_e.read().verdict == "match"
items = [(empty, None, K.VoteWorkspace(0), None), ([base[:999].clone() for _ in range(3)], None, K.VoteWorkspace(0), None),
         (empty, None, K.VoteWorkspace(0), None)]
K.vote_batch(items, 1e-3)
assert all(it[2].read().verdict == "match" for it in items)
# copies, checkpoint + checksum, restore, fill, scribble, scale injection
dst = torch.empty_like(base)
cs = K.checkpoint(dst, base, with_checksum=True)
K.restore(base, dst, expect=cs)
K.copy(dst[1:], base[:-1])
K.fill(dst.view(torch.uint8), 7)
K.inject_scale(dst, 99, 0.01)
K.scribble(dst.view(torch.uint8), bytes(range(8)))
# 1-D workload bodies
K.vec_inc(base, dst)
K.vec_path(base, dst)
torch.cuda.synchronize()
print("sanitize target ok")
