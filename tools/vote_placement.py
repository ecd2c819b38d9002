"""K = 2 vote time against the distance between the two replica buffers.

The 64 MiB K = 2 vote runs at 0.84-0.95 of the HBM copy peak depending on
where the allocator put the two replicas.  This carves both
replicas out of one allocation at base offsets 0 and 64 MiB + delta and
times back-to-back votes (CUDA events, 30 iterations after 3 warm-up) for a
range of deltas, then times every pair of six separately allocated 64 MiB
replicas.  Both parts use identical and diverse (1e-6 relative noise, the
fp32-screen path) replica values.  Prints one JSON line per case.
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1405_2912_b200 import kernels  # noqa: E402

MIB = 1 << 20
n = 16 * MIB  # fp32 elements: 64 MiB per replica
deltas_kib = [0, 1, 4, 16, 64, 256, 512, 1024, 2048, 4096, 8192, 32768, 65536]
arena = torch.empty((2 * n * 4 + max(deltas_kib) * 1024) // 4 + 1024, device="cuda")
src = torch.rand(n, device="cuda") + 1
noisy = src * (1 + 1e-6 * torch.randn(n, device="cuda"))
st = torch.cuda.Stream()
ws = kernels.VoteWorkspace(0, stream=st)
iters = 30


def time_pair(r0, r1):
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        for _ in range(3):
            kernels.vote_async([r0, r1], ws, 1e-3, stream=st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(iters):
            kernels.vote_async([r0, r1], ws, 1e-3, stream=st)
        e1.record(st)
    st.synchronize()
    assert ws.read().verdict == "match"
    return e0.elapsed_time(e1) / iters * 1e-3


for values in ("identical", "diverse"):
    for d in deltas_kib:
        off1 = n + d * 256  # elements
        r0 = arena[:n]
        r1 = arena[off1:off1 + n]
        r0.copy_(src)
        r1.copy_(src if values == "identical" else noisy)
        t = time_pair(r0, r1)
        print(json.dumps({"layout": "arena", "values": values, "delta_kib": d,
                          "distance_mib": round(off1 * 4 / MIB, 4), "us": round(t * 1e6, 2),
                          "read_GBps": round(2 * n * 4 / t / 1e9, 1)}), flush=True)
del arena
bufs = [torch.empty(n, device="cuda") for _ in range(6)]
for values in ("identical", "diverse"):
    for i in range(6):
        for j in range(i + 1, 6):
            bufs[i].copy_(src)
            bufs[j].copy_(src if values == "identical" else noisy)
            t = time_pair(bufs[i], bufs[j])
            print(json.dumps({"layout": "separate", "values": values, "pair": [i, j],
                              "distance_mib": round((bufs[j].data_ptr() - bufs[i].data_ptr()) / MIB, 2),
                              "us": round(t * 1e6, 2), "read_GBps": round(2 * n * 4 / t / 1e9, 1)}), flush=True)
